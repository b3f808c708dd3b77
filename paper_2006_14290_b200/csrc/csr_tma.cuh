// CSR "stream" SpMV with TMA bulk-copy staging (load-balanced, bitwise for
// rows of <= kCsrChunk entries).
//
// Work items come from the nnz-chunk plan (`first[c]` = first row whose entries
// start in chunk c of kCsrChunk entries): item c owns the rows starting in
// chunk c, so its short rows span < 2*kCsrChunk contiguous entries. Persistent
// grid, W independent warp pipelines per CTA; warp w takes items w, w + Wtot,
// ... For each item lane 0 streams the item's value and column ranges with
// cp.async.bulk into an S-deep per-warp shared-memory ring (mbarrier
// complete_tx); the 32 lanes then form the products v*x[col] in place
// (coalesced shared reads, L1/L2 gathers of x) and fold whole rows
// sequentially from shared memory — the reference fold, bit for bit.
// A row longer than kCsrChunk entries ("long") is split across the items its
// entries fall into: each part is reduced by its warp (direct loads), written
// to a partial slot, and the last-arriving part (atomic ticket) adds the
// partials in chunk order (deterministic; reassociated, so long rows are
// checked with the 1e-12 tolerance).
#pragma once

#include "common.cuh"

namespace wk {

constexpr int kCsrChunk = 256;
constexpr int kCsrCap = 2 * kCsrChunk;

template <int W, int S, int B = 1>
struct CsrTmaCfg {
    static constexpr int kW = W, kS = S, kMinBlocks = B;
    static constexpr int kValSlots = kCsrCap + 2;   // 16-byte alignment slack
    static constexpr int kColSlots = kCsrCap + 4;
    static constexpr size_t kStageBytes = size_t(kValSlots) * 8 + size_t(kColSlots) * 4;
    static constexpr size_t kSmem = size_t(W) * S * kStageBytes + W * S * 8 + W * S * 64 + 256;
};

// Item geometry shared by producer and consumer (warp-uniform).
struct CsrItem {
    int64_t rb, re, rs_end;  // rows starting in the chunk; short rows [rb, rs_end)
    int64_t base, cnt;       // entry range of the short rows
    bool tail_long;          // part of a long row started in an earlier chunk
    bool head_long;          // the last row (re-1) is long and starts here
};

__device__ __forceinline__ CsrItem csr_item(int64_t c, const int* __restrict__ ptrs, const int* __restrict__ first) {
    CsrItem it;
    it.rb = __ldg(first + c);
    it.re = __ldg(first + c + 1);
    const int64_t chunk_lo = c * kCsrChunk;
    it.tail_long = false;
    if (it.rb > 0) {
        const int64_t Ls = __ldg(ptrs + it.rb - 1), Le = __ldg(ptrs + it.rb);
        it.tail_long = (Le - Ls > kCsrChunk) && (Le > chunk_lo);
    }
    it.head_long = false;
    it.rs_end = it.re;
    if (it.rb < it.re) {
        const int64_t Ls = __ldg(ptrs + it.re - 1), Le = __ldg(ptrs + it.re);
        if (Le - Ls > kCsrChunk) {
            it.head_long = true;
            it.rs_end = it.re - 1;
        }
    }
    it.base = 0;
    it.cnt = 0;
    if (it.rb < it.rs_end) {
        it.base = __ldg(ptrs + it.rb);
        it.cnt = int64_t(__ldg(ptrs + it.rs_end)) - it.base;
    }
    return it;
}

// Packed per-item descriptor stored in the plan (built once per matrix by
// csr_items_kernel): {rb, rs_end, base, cnt | tail_long << 30 | head_long << 29}.
constexpr int kTailBit = 1 << 30, kHeadBit = 1 << 29, kCntMask = (1 << 29) - 1;

__device__ __forceinline__ int4 csr_item_pack(const CsrItem& it) {
    return make_int4(int(it.rb), int(it.rs_end), int(it.base),
                     int(it.cnt) | (it.tail_long ? kTailBit : 0) | (it.head_long ? kHeadBit : 0));
}

__global__ void csr_items_kernel(int64_t nchunks, const int* __restrict__ ptrs, const int* __restrict__ first,
                                 int4* __restrict__ items) {
    const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c < nchunks) items[c] = csr_item_pack(csr_item(c, ptrs, first));
}

__host__ __device__ inline int64_t csr_first_slots(int64_t nchunks) { return ((nchunks + 1 + 3) / 4) * 4; }

// one part of a long row: entries [lo, hi) reduced by the warp; the last part
// to arrive publishes y[L] (partials summed in chunk order)
__device__ __forceinline__ void csr_long_part(int64_t L, int64_t lo, int64_t hi, int64_t slot, int64_t c_head,
                                              int64_t c_last, const int* __restrict__ col,
                                              const double* __restrict__ val, const double* __restrict__ x,
                                              double* __restrict__ partials, unsigned* __restrict__ tickets,
                                              double* __restrict__ y, int lane) {
    constexpr int U = 8;  // 8 independent loads + gathers in flight per lane
    double acc = 0.0;
    for (int64_t k0 = lo; k0 < hi; k0 += 32 * U) {
        double v[U], xv[U];
        int c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t k = k0 + u * 32 + lane;
            v[u] = 0.0;
            c[u] = 0;
            if (k < hi) {
                v[u] = ld_stream(val + k);
                c[u] = ld_stream(col + k);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) xv[u] = (k0 + u * 32 + lane < hi) ? ld_x(x, c[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u) acc += __dmul_rn(v[u], xv[u]);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
    if (lane == 0) {
        partials[slot] = acc;
        __threadfence();
        const unsigned parts = unsigned(c_last - c_head + 1);
        const unsigned t = atomicAdd(tickets + c_head, 1u);
        if (t == parts - 1) {
            __threadfence();
            double s = __ldcg(partials + 2 * c_head + 1);
            for (int64_t cc = c_head + 1; cc <= c_last; ++cc) s += __ldcg(partials + 2 * cc);
            y[L] = s;
            tickets[c_head] = 0;
        }
    }
    __syncwarp();
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::kW * 32, Cfg::kMinBlocks)
csr_tma_kernel(int64_t nrows, int64_t nnz, int64_t nchunks, const int* __restrict__ ptrs,
               const int* __restrict__ col, const double* __restrict__ val, const double* __restrict__ x,
               double* __restrict__ y, const int* __restrict__ first, double* __restrict__ partials,
               unsigned* __restrict__ tickets, const int* __restrict__ skip) {
    constexpr int W = Cfg::kW, S = Cfg::kS, U = 8;
    if (skip != nullptr && *skip) return;
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* wbase = smem + size_t(warp) * S * Cfg::kStageBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(W) * S * Cfg::kStageBytes) + warp * S;
    CsrItem* items = reinterpret_cast<CsrItem*>(smem + size_t(W) * S * Cfg::kStageBytes + size_t(W) * S * 8) + warp * S;
    auto sval = [&](int st) { return reinterpret_cast<double*>(wbase + size_t(st) * Cfg::kStageBytes); };
    auto scol = [&](int st) {
        return reinterpret_cast<int*>(wbase + size_t(st) * Cfg::kStageBytes + size_t(Cfg::kValSlots) * 8);
    };
    if (lane == 0) {
        for (int st = 0; st < S; ++st) mbar_init(bars + st, 1);
        fence_mbar_init();
    }
    __syncwarp();
    const int64_t gwarp = int64_t(blockIdx.x) * W + warp;
    const int64_t nwarps = int64_t(gridDim.x) * W;
    const uint64_t pol = policy_evict_first();

    // Producer: walk this warp's items; items (or parts) that need no staging
    // — long-row parts and runs of empty rows — are finished on the spot, the
    // short rows of the next item are streamed into stage `st` and its
    // geometry is queued for the consumer. Returns false when exhausted.
    const int4* __restrict__ descs = reinterpret_cast<const int4*>(first + csr_first_slots(nchunks));
    // descriptors of the warp's next 32 items, one per lane (one coalesced-
    // per-lane load hides the metadata latency of 32 items)
    int64_t pc = gwarp;
    int4 win = make_int4(0, 0, 0, 0);
    int wi = 32;
    auto next_desc = [&](int64_t& c, int4& d) -> bool {
        if (pc >= nchunks) return false;
        if (wi == 32) {
            const int64_t cl = pc + int64_t(lane) * nwarps;
            win = cl < nchunks ? __ldg(descs + cl) : make_int4(0, 0, 0, 0);
            wi = 0;
        }
        d.x = __shfl_sync(0xffffffffu, win.x, wi);
        d.y = __shfl_sync(0xffffffffu, win.y, wi);
        d.z = __shfl_sync(0xffffffffu, win.z, wi);
        d.w = __shfl_sync(0xffffffffu, win.w, wi);
        ++wi;
        c = pc;
        pc += nwarps;
        return true;
    };
    auto produce = [&](int st) -> bool {
        int64_t c;
        int4 d;
        while (next_desc(c, d)) {
            CsrItem it;
            it.rb = d.x;
            it.rs_end = d.y;
            it.base = d.z;
            it.cnt = d.w & kCntMask;
            const int64_t chunk_lo = c * kCsrChunk, chunk_hi = chunk_lo + kCsrChunk;
            if (d.w & kTailBit) {
                const int64_t L = it.rb - 1;
                const int64_t Ls = __ldg(ptrs + L), Le = __ldg(ptrs + it.rb);
                csr_long_part(L, chunk_lo, Le < chunk_hi ? Le : chunk_hi, 2 * c, Ls / kCsrChunk, (Le - 1) / kCsrChunk,
                              col, val, x, partials, tickets, y, lane);
            }
            if (d.w & kHeadBit) {
                const int64_t L = it.rs_end;
                const int64_t Ls = __ldg(ptrs + L), Le = __ldg(ptrs + L + 1);
                csr_long_part(L, Ls, chunk_hi, 2 * c + 1, c, (Le - 1) / kCsrChunk, col, val, x, partials, tickets, y,
                              lane);
            }
            if (it.rb >= it.rs_end) continue;
            if (it.cnt == 0) {  // only empty rows
                for (int64_t r = it.rb + lane; r < it.rs_end; r += 32) y[r] = 0.0;
                continue;
            }
            if (lane == 0) {
                const int64_t va = it.base & ~int64_t(1), ve = (it.base + it.cnt) & ~int64_t(1);
                const int64_t ca = it.base & ~int64_t(3), ce = (it.base + it.cnt) & ~int64_t(3);
                const uint32_t bv = uint32_t((ve - va) * 8), bc = uint32_t((ce - ca) * 4);
                items[st] = it;
                mbar_arrive_expect_tx(bars + st, bv + bc);
                if (bv) bulk_g2s_evict_first(sval(st), val + va, bv, bars + st, pol);
                if (bc) bulk_g2s_evict_first(scol(st), col + ca, bc, bars + st, pol);
            }
            {
                // the <= 1 value and <= 3 indices past the last 16-byte unit:
                // plain loads into the same stage (ordered by __syncwarp)
                const int64_t end = it.base + it.cnt;
                const int64_t va = it.base & ~int64_t(1), ve = end & ~int64_t(1);
                const int64_t ca = it.base & ~int64_t(3), ce = end & ~int64_t(3);
                if (lane < end - ve) sval(st)[ve - va + lane] = ld_stream(val + ve + lane);
                if (lane < end - ce) scol(st)[ce - ca + lane] = ld_stream(col + ce + lane);
            }
            __syncwarp();
            return true;
        }
        return false;
    };
    int live = 0;
    for (int st = 0; st < S; ++st)
        if (produce(st)) ++live;

    for (uint32_t i = 0; live > 0; ++i) {
        const int st = int(i % S);
        const CsrItem it = items[st];
        // row bounds of this lane's first row, loaded early to overlap latency
        const int64_t r0 = it.rb + lane;
        int lo0 = 0, hi0 = 0;
        if (r0 < it.rs_end) {
            lo0 = int(__ldg(ptrs + r0) - it.base);
            hi0 = int(__ldg(ptrs + r0 + 1) - it.base);
        }
        mbar_wait(bars + st, (i / S) & 1);
        double* sv = sval(st);
        const int* sc = scol(st);
        const int ov = int(it.base & 1), oc = int(it.base & 3);
        const int cnt = int(it.cnt);
        // products v * x[col] in place, U gathers in flight per lane
        for (int e0 = 0; e0 < cnt; e0 += 32 * U) {
            double v[U], xv[U];
            int cc[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int e = e0 + u * 32 + lane;
                cc[u] = 0;
                v[u] = 0.0;
                if (e < cnt) {
                    v[u] = sv[ov + e];
                    cc[u] = sc[oc + e];
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) xv[u] = (e0 + u * 32 + lane < cnt) ? ld_x(x, cc[u]) : 0.0;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int e = e0 + u * 32 + lane;
                if (e < cnt) sv[ov + e] = __dmul_rn(v[u], xv[u]);
            }
        }
        __syncwarp();
        // fold whole rows sequentially (the reference fold)
        for (int64_t r = r0; r < it.rs_end; r += 32) {
            int lo = lo0, hi = hi0;
            if (r != r0) {
                lo = int(__ldg(ptrs + r) - it.base);
                hi = int(__ldg(ptrs + r + 1) - it.base);
            }
            double acc = 0.0;
            const double* pr = sv + ov;
            int e = lo;
            for (; e + 4 <= hi; e += 4) {
                const double p0 = pr[e], p1 = pr[e + 1], p2 = pr[e + 2], p3 = pr[e + 3];
                acc = __dadd_rn(acc, p0);
                acc = __dadd_rn(acc, p1);
                acc = __dadd_rn(acc, p2);
                acc = __dadd_rn(acc, p3);
            }
            for (; e < hi; ++e) acc = __dadd_rn(acc, pr[e]);
            y[r] = acc;
        }
        __syncwarp();
        if (lane == 0) fence_proxy_async_smem();
        if (!produce(st)) --live;
    }
}

template <class Cfg>
int launch_csr_tma(int64_t nrows, int64_t nnz, int64_t nchunks, const int* ptrs, const int* col, const double* val,
                   const double* x, double* y, const int* first, double* partials, unsigned* tickets,
                   const int* skip, cudaStream_t st) {
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev & 63]) {
        WK_CUDA(cudaFuncSetAttribute(csr_tma_kernel<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(Cfg::kSmem)));
        attr_set[dev & 63] = true;
    }
    int per_sm = 0;  // persistent grid: every CTA the SM can hold
    WK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, csr_tma_kernel<Cfg>, Cfg::kW * 32, Cfg::kSmem));
    int64_t grid = int64_t(sm_count()) * (per_sm > 0 ? per_sm : 1);
    const int64_t need = ceil_div(nchunks, Cfg::kW);
    if (grid > need) grid = need;
    csr_tma_kernel<Cfg><<<(unsigned)grid, Cfg::kW * 32, Cfg::kSmem, st>>>(nrows, nnz, nchunks, ptrs, col, val, x, y,
                                                                        first, partials, tickets, skip);
    WK_LAUNCH_CHECK();
    return 0;
}

// ---------------------------------------------------------------------------
// CSR row-block kernel: items are fixed blocks of 32 consecutive rows, so the
// thread-per-row fold keeps every lane busy. A "light" block (<= kRbCap
// entries) is streamed into a per-warp shared-memory ring with cp.async.bulk
// and each lane folds its row sequentially from shared memory with x gathered
// through L1/L2 (the reference fold, bitwise). A "heavy" block (some long
// rows) is processed row by row with a warp-wide reduction over the row's
// entries (direct loads; reassociated, 1e-12 tolerance). No plan needed: the
// block extents are read from row_ptrs, 32 blocks ahead per lane.
// ---------------------------------------------------------------------------
template <int W, int S, int CAP = 1024>
struct CsrRbCfg {
    static constexpr int kW = W, kS = S, kCap = CAP;
    static constexpr int kValSlots = CAP + 2, kColSlots = CAP + 4;
    static constexpr size_t kStageBytes = size_t(kValSlots) * 8 + size_t(kColSlots) * 4;
    static constexpr size_t kSmem = size_t(W) * S * kStageBytes + W * S * 8 + W * S * 16 + 256;
};

template <class Cfg>
__global__ void __launch_bounds__(Cfg::kW * 32, 1)
csr_rowblock_kernel(int64_t nrows, int rows_per_lane, const int* __restrict__ ptrs, const int* __restrict__ col,
                    const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y,
                    const int* __restrict__ skip) {
    constexpr int W = Cfg::kW, S = Cfg::kS, U = 8;
    if (skip != nullptr && *skip) return;
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* wbase = smem + size_t(warp) * S * Cfg::kStageBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(W) * S * Cfg::kStageBytes) + warp * S;
    int2* qblk = reinterpret_cast<int2*>(smem + size_t(W) * S * Cfg::kStageBytes + size_t(W) * S * 8) + warp * S;
    auto sval = [&](int st) { return reinterpret_cast<double*>(wbase + size_t(st) * Cfg::kStageBytes); };
    auto scol = [&](int st) {
        return reinterpret_cast<int*>(wbase + size_t(st) * Cfg::kStageBytes + size_t(Cfg::kValSlots) * 8);
    };
    if (lane == 0) {
        for (int st = 0; st < S; ++st) mbar_init(bars + st, 1);
        fence_mbar_init();
    }
    __syncwarp();
    const int64_t brows = int64_t(rows_per_lane) * 32;  // rows per block
    const int64_t nblocks = (nrows + brows - 1) / brows;
    const int64_t gwarp = int64_t(blockIdx.x) * W + warp;
    const int64_t nwarps = int64_t(gridDim.x) * W;
    const uint64_t pol = policy_evict_first();

    int64_t pb = gwarp;
    int wlo = 0, whi = 0, wi = 32;
    auto next_block = [&](int64_t& b, int& lo, int& hi) -> bool {
        if (pb >= nblocks) return false;
        if (wi == 32) {
            const int64_t bl = pb + int64_t(lane) * nwarps;
            if (bl < nblocks) {
                wlo = __ldg(ptrs + bl * brows);
                const int64_t rend = (bl * brows + brows < nrows) ? bl * brows + brows : nrows;
                whi = __ldg(ptrs + rend);
            }
            wi = 0;
        }
        lo = __shfl_sync(0xffffffffu, wlo, wi);
        hi = __shfl_sync(0xffffffffu, whi, wi);
        ++wi;
        b = pb;
        pb += nwarps;
        return true;
    };
    // heavy block (> Cfg::kCap entries): rows of <= 64 entries are folded by
    // their lane with direct loads (still the reference fold), longer rows
    // with a warp-wide reduction (reassociated)
    auto heavy = [&](int64_t r0, int64_t rend) {
        for (int64_t r = r0 + lane; r < rend; r += 32) {
            const int64_t a = __ldg(ptrs + r), e = __ldg(ptrs + r + 1);
            if (e - a <= 64) {
                double acc = 0.0;
                for (int64_t k = a; k < e; ++k) acc = mul_add_rn(acc, ld_stream(val + k), ld_x(x, ld_stream(col + k)));
                y[r] = acc;
            }
        }
        for (int64_t r = r0; r < rend; ++r) {
            const int64_t a = __ldg(ptrs + r), e = __ldg(ptrs + r + 1);
            if (e - a <= 64) continue;
            double acc = 0.0;
            for (int64_t k = a + lane; k < e; k += 32) acc += __dmul_rn(ld_stream(val + k), ld_x(x, ld_stream(col + k)));
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
            if (lane == 0) y[r] = acc;
        }
    };
    // producer: heavy blocks are finished on the spot; the next light block is
    // streamed into stage st and queued
    auto produce = [&](int st) -> bool {
        int64_t b;
        int lo, hi;
        while (next_block(b, lo, hi)) {
            const int64_t r0 = b * brows;
            const int64_t cnt = int64_t(hi) - lo;
            if (cnt > Cfg::kCap) {
                heavy(r0, (r0 + brows < nrows) ? r0 + brows : nrows);
                continue;
            }
            const int64_t base = lo, end = hi;
            const int64_t va = base & ~int64_t(1), ve = end & ~int64_t(1);
            const int64_t ca = base & ~int64_t(3), ce = end & ~int64_t(3);
            if (lane == 0) {
                const uint32_t bv = uint32_t((ve - va) * 8), bc = uint32_t((ce - ca) * 4);
                qblk[st] = make_int2(int(b), int(base));
                mbar_arrive_expect_tx(bars + st, bv + bc);
                if (bv) bulk_g2s_evict_first(sval(st), val + va, bv, bars + st, pol);
                if (bc) bulk_g2s_evict_first(scol(st), col + ca, bc, bars + st, pol);
            }
            if (lane < end - ve) sval(st)[ve - va + lane] = ld_stream(val + ve + lane);
            if (lane < end - ce) scol(st)[ce - ca + lane] = ld_stream(col + ce + lane);
            __syncwarp();
            return true;
        }
        return false;
    };
    int live = 0;
    for (int st = 0; st < S; ++st)
        if (produce(st)) ++live;

    for (uint32_t i = 0; live > 0; ++i) {
        const int st = int(i % S);
        const int2 q = qblk[st];
        const int64_t rb = int64_t(q.x) * brows;
        const int64_t base = q.y;
        int64_t r = rb + lane;
        int lo = 0, hi = 0;
        if (r < nrows) {
            lo = int(__ldg(ptrs + r) - base);
            hi = int(__ldg(ptrs + r + 1) - base);
        }
        mbar_wait(bars + st, (i / S) & 1);
        const double* sv = sval(st) + (base & 1);
        const int* sc = scol(st) + (base & 3);
        for (int t = 0; t < rows_per_lane; ++t) {
            // prefetch the next round's row bounds
            const int64_t rn = r + 32;
            int nlo = 0, nhi = 0;
            if (t + 1 < rows_per_lane && rn < nrows) {
                nlo = int(__ldg(ptrs + rn) - base);
                nhi = int(__ldg(ptrs + rn + 1) - base);
            }
            double acc = 0.0;
            int e = lo;
            for (; e + U <= hi; e += U) {
                double v[U], xv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    v[u] = sv[e + u];
                    xv[u] = ld_x(x, sc[e + u]);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) acc = mul_add_rn(acc, v[u], xv[u]);
            }
            {
                double v[U], xv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (e + u < hi) {
                        v[u] = sv[e + u];
                        xv[u] = ld_x(x, sc[e + u]);
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (e + u < hi) acc = mul_add_rn(acc, v[u], xv[u]);
            }
            if (r < nrows) y[r] = acc;
            r = rn;
            lo = nlo;
            hi = nhi;
        }
        __syncwarp();
        if (lane == 0) fence_proxy_async_smem();
        if (!produce(st)) --live;
    }
}

// rows per lane so that a block of 32*k rows holds ~80% of `cap` entries on average
inline int csr_rows_per_lane(int64_t nrows, int64_t nnz, int cap) {
    if (nrows == 0) return 1;
    const double avg = double(nnz) / double(nrows);
    int k = int(double(cap) * 0.8 / (32.0 * (avg > 1.0 ? avg : 1.0)));
    return k < 1 ? 1 : (k > 16 ? 16 : k);
}

template <class Cfg>
int launch_csr_rowblock(int64_t nrows, int64_t nnz, const int* ptrs, const int* col, const double* val,
                        const double* x, double* y, const int* skip, cudaStream_t st) {
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev & 63]) {
        WK_CUDA(cudaFuncSetAttribute(csr_rowblock_kernel<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(Cfg::kSmem)));
        attr_set[dev & 63] = true;
    }
    const int k = csr_rows_per_lane(nrows, nnz, Cfg::kCap);
    int64_t grid = sm_count();
    const int64_t need = ceil_div(ceil_div(nrows, 32 * k), Cfg::kW);
    if (grid > need) grid = need;
    if (grid < 1) grid = 1;
    csr_rowblock_kernel<Cfg><<<(unsigned)grid, Cfg::kW * 32, Cfg::kSmem, st>>>(nrows, k, ptrs, col, val, x, y, skip);
    WK_LAUNCH_CHECK();
    return 0;
}

}  // namespace wk
