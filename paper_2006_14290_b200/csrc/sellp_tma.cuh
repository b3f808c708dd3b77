// SELL-P(64) SpMV with TMA bulk-copy staging — the B200 path for slice_size 64.
//
// Persistent grid, one CTA per SM, WARPS independent warp pipelines. Warp w
// owns slices w, w + W, w + 2W, ... (W = warps in the grid); each slice is cut
// into chunks of J columns (J * 64 entries: 512*J bytes of values + 256*J
// bytes of column indices, both contiguous in the SELL-P layout). Lane 0
// streams the chunks with cp.async.bulk (TMA engine, L2 evict-first) into an
// S-deep per-warp ring in shared memory, completion tracked by one mbarrier
// per stage; all 32 lanes consume a landed chunk (2 rows per lane, 128-bit
// shared loads), gather x[col] through L1/L2 and fold sequentially with
// separately rounded multiply/add (bitwise == reference fold). DRAM streaming
// is thereby decoupled from the gather latency: S-1 chunks per warp stay in
// flight while the current chunk's gathers resolve.
#pragma once

#include "cg_state.cuh"
#include "reduce.cuh"

namespace wk {

template <int J, int S, int WARPS, int CTAS = 1>
struct SellpTmaCfg {
    static constexpr int kJ = J, kS = S, kWarps = WARPS, kCtas = CTAS;
    static constexpr int kChunk = J * 64;
    static constexpr size_t kSmem = size_t(WARPS) * S * kChunk * (sizeof(double) + sizeof(int)) + WARPS * S * 8;
};

// Consume one landed chunk: nj <= J columns for this lane's two rows.
// kGuard (ELL's last, partial 64-row block): rows past nrows hold stale
// shared memory and must not gather.
// kColStride: distance between the staged columns (64 = one SELL-P slice).
// kCoh: gather x with ld.global.cg (coherent at L2, no L1 line) — the peer
// CG variant, whose x halo is written by the neighbours DURING the kernel:
// the non-coherent __ldg path is outside the memory model for such data.
template <int J, bool kLen, bool kGuard = false, int kColStride = 64, bool kCoh = false>
__device__ __forceinline__ void sellp_chunk(const double* __restrict__ v, const int* __restrict__ c, int nj,
                                            int j0, int len0, int len1, const double* __restrict__ x, double& a0,
                                            double& a1, bool ok0 = true, bool ok1 = true) {
    double2 vv[J];
    double x0[J], x1[J];
#pragma unroll
    for (int jj = 0; jj < J; ++jj) {
        if (jj < nj) {
            vv[jj] = *reinterpret_cast<const double2*>(v + jj * kColStride);
            const int2 cc = *reinterpret_cast<const int2*>(c + jj * kColStride);
            x0[jj] = (!kGuard || ok0) ? (kCoh ? __ldcg(x + cc.x) : ld_x(x, cc.x)) : 0.0;
            x1[jj] = (!kGuard || ok1) ? (kCoh ? __ldcg(x + cc.y) : ld_x(x, cc.y)) : 0.0;
        }
    }
#pragma unroll
    for (int jj = 0; jj < J; ++jj) {
        if (jj < nj) {
            if (!kLen || j0 + jj < len0) a0 = mul_add_rn(a0, vv[jj].x, x0[jj]);
            if (!kLen || j0 + jj < len1) a1 = mul_add_rn(a1, vv[jj].y, x1[jj]);
        }
    }
}

// One staged chunk of a slice in registers: the lane's two rows' values of up
// to J columns and the gathered x. Loading a chunk (shared-memory reads + the
// x gathers) and folding it are separate steps so a warp can issue the next
// chunk's gathers before it folds the current one: a 7-point slice is two
// chunks, and without the lookahead every chunk paid one full gather round
// trip in sequence (0.285 ms on the 256^3 operator).
template <int J>
struct SellpChunkRegs {
    double2 v[J];
    double x0[J], x1[J];
    int nj, j0;
};

template <int J, bool kCoh>
__device__ __forceinline__ void sellp_chunk_load(SellpChunkRegs<J>& c, const double* __restrict__ v,
                                                 const int* __restrict__ ci, int nj, int j0,
                                                 const double* __restrict__ x) {
    c.nj = nj;
    c.j0 = j0;
#pragma unroll
    for (int jj = 0; jj < J; ++jj) {
        if (jj < nj) {
            c.v[jj] = *reinterpret_cast<const double2*>(v + jj * 64);
            const int2 cc = *reinterpret_cast<const int2*>(ci + jj * 64);
            c.x0[jj] = kCoh ? __ldcg(x + cc.x) : ld_x(x, cc.x);
            c.x1[jj] = kCoh ? __ldcg(x + cc.y) : ld_x(x, cc.y);
        }
    }
}

template <int J, bool kLen>
__device__ __forceinline__ void sellp_chunk_fold(const SellpChunkRegs<J>& c, int len0, int len1, double& a0,
                                                 double& a1) {
#pragma unroll
    for (int jj = 0; jj < J; ++jj) {
        if (jj < c.nj) {
            if (!kLen || c.j0 + jj < len0) a0 = mul_add_rn(a0, c.v[jj].x, c.x0[jj]);
            if (!kLen || c.j0 + jj < len1) a1 = mul_add_rn(a1, c.v[jj].y, c.x1[jj]);
        }
    }
}

// kDot: also accumulate sum_r x[r] * y[r] over the owned rows (CG's p.Ap with
// x = p, y = q) and publish it through DotEpilogue (last-arriving CTA).
// kCoh: coherent x gathers (peer CG: the halo of x lands during the kernel).
// kBicg (BiCGSTAB, BicgEpilogue): 1 = r-hat.y, 2 = (y.y, y.x) over the rows.
template <class Cfg, bool kDot = false, bool kCoh = false, int kBicg = 0>
__global__ void __launch_bounds__(Cfg::kWarps * 32, Cfg::kCtas)
sellp64_tma_kernel(int64_t nrows, int64_t ncols, int64_t nslices, const int64_t* __restrict__ sets,
                   const int* __restrict__ col, const double* __restrict__ val, const int* __restrict__ row_lengths,
                   const double* __restrict__ x, double* __restrict__ y, const int* __restrict__ skip,
                   DotEpilogue dot, int rev = 0, BicgEpilogue bep = BicgEpilogue{nullptr, nullptr, nullptr, nullptr, 0}) {
    constexpr int J = Cfg::kJ, S = Cfg::kS, WARPS = Cfg::kWarps, CH = Cfg::kChunk;
    if (skip != nullptr && *skip) return;
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* sval = reinterpret_cast<double*>(smem) + size_t(warp) * S * CH;
    int* scol = reinterpret_cast<int*>(smem + size_t(WARPS) * S * CH * sizeof(double)) + size_t(warp) * S * CH;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(WARPS) * S * CH * 12) + warp * S;
    if (lane == 0) {
        for (int st = 0; st < S; ++st) mbar_init(bars + st, 1);
        fence_mbar_init();
    }
    __syncwarp();
    const bool finite0 = ncols == 0 || isfinite(__ldg(x));
    const int64_t gwarp = int64_t(blockIdx.x) * WARPS + warp;
    const int64_t nwarps = int64_t(gridDim.x) * WARPS;
    const uint64_t pol = policy_evict_first();
    // rev: walk the slices from the last one down (a CG iteration alternates
    // directions so each kernel starts on the rows the previous one touched
    // last, which are still in L2); per-row results do not depend on it
    auto SP = [&](int64_t k) -> int64_t { return rev ? nslices - 1 - k : k; };

    // ---- producer (lane 0 issues; cursor warp-uniform) ----
    int64_t ps = gwarp, pbase = 0;
    int pj = 0, pw = 0;
    bool pvalid = false;
    // slice offsets are read one slice ahead (registers), so the next
    // slice's sets[] loads are in flight while this slice streams
    // (slice offsets in 64-slot units: int32 is enough below 2^37 stored slots)
    int q0 = 0, q1 = 0, n0 = 0, n1 = 0;
    if (ps < nslices) {
        q0 = int(__ldg(sets + SP(ps)));
        q1 = int(__ldg(sets + SP(ps) + 1));
    }
    if (ps + nwarps < nslices) {
        n0 = int(__ldg(sets + SP(ps + nwarps)));
        n1 = int(__ldg(sets + SP(ps + nwarps) + 1));
    }
    auto seek = [&]() {
        pvalid = false;
        while (ps < nslices) {
            pw = int(q1 - q0);
            if (pj < pw) {
                pbase = int64_t(q0) * 64;
                pvalid = true;
                return;
            }
            ps += nwarps;
            pj = 0;
            q0 = n0;
            q1 = n1;
            if (ps + nwarps < nslices) {
                n0 = int(__ldg(sets + SP(ps + nwarps)));
                n1 = int(__ldg(sets + SP(ps + nwarps) + 1));
            }
        }
    };
    auto issue = [&](int st) {
        if (lane == 0) {
            const int nj = (pw - pj < J) ? pw - pj : J;
            const uint32_t bv = uint32_t(nj) * 64 * sizeof(double), bc = uint32_t(nj) * 64 * sizeof(int);
            mbar_arrive_expect_tx(bars + st, bv + bc);
            const int64_t off = pbase + int64_t(pj) * 64;
            bulk_g2s_evict_first(sval + st * CH, val + off, bv, bars + st, pol);
            bulk_g2s_evict_first(scol + st * CH, col + off, bc, bars + st, pol);
        }
        pj += J;
        seek();
    };
    seek();
    for (int st = 0; st < S && pvalid; ++st) issue(st);

    // peer-memory distributed CG: the neighbours push the halo of x while this
    // kernel runs. Slices in [int_lo, int_hi) gather no halo column, so a warp
    // waits for the halo flags only before gathering its first slice outside
    // that range: interior rows overlap the exchange, boundary rows run after
    // arrival. The slice order (and so every sum) is the same as without a halo.
    // (the halo exists only in the peer variant, which gathers coherently)
    constexpr bool kHalo = kDot && kCoh;
    bool halo_pending = kHalo && dot.halo != nullptr;
    int64_t int_lo = 0, int_hi = 0;
    if (kHalo && halo_pending) {
        int_lo = dot.halo->int_lo;
        int_hi = dot.halo->int_hi;
    }

    // ---- consumer: chunks in stream order, the next one's gathers issued
    // before the current one is folded ----
    int cst = 0;          // ring stage of the next chunk to load
    uint32_t cphase = 0;  // its mbarrier phase parity
    // load the next chunk of slice ls (width lw) at column lj0 into c, then
    // hand its stage back to the producer (the chunk now lives in registers)
    auto load = [&](SellpChunkRegs<J>& c, int64_t ls, int lw, int lj0) {
        if (kHalo && halo_pending && (SP(ls) < int_lo || SP(ls) >= int_hi)) {
            if (lane == 0) halo_wait(dot.peer, dot.halo);
            __syncwarp();
            halo_pending = false;
        }
        const int st = cst;
        mbar_wait(bars + st, cphase);
        const int nj = (lw - lj0 < J) ? lw - lj0 : J;
        sellp_chunk_load<J, kCoh>(c, sval + st * CH + 2 * lane, scol + st * CH + 2 * lane, nj, lj0, x);
        __syncwarp();
        if (pvalid) {
            if (lane == 0) fence_proxy_async_smem();
            issue(st);
        }
        if (++cst == S) {
            cst = 0;
            cphase ^= 1u;
        }
    };
    double dacc = 0.0, bacc0 = 0.0, bacc1 = 0.0;
    // kDot: x at the slice's own rows (CG: p[r]), read after the fold (L1/L2
    // hits: the same lines were just gathered)
    auto xown = [&](int64_t r0) -> double2 {
        if (!kDot) return make_double2(0.0, 0.0);
        if (r0 + 1 < nrows) return *reinterpret_cast<const double2*>(x + r0);
        return make_double2(r0 < nrows ? x[r0] : 0.0, 0.0);
    };
    // kDot (CG): q is read by the next kernel, which starts on the rows this
    // one wrote last (ping-pong): plain stores keep q's tail in L2 instead of
    // the evict-first streaming stores of the SpMV
    auto emit = [&](int64_t r0, double a0, double a1, double2 p) {
        if (kBicg == 1) {  // r-hat at the own rows
            if (r0 + 1 < nrows) {
                const double2 w = *reinterpret_cast<const double2*>(bep.w + r0);
                bacc0 += __dmul_rn(w.x, a0);
                bacc0 += __dmul_rn(w.y, a1);
            } else if (r0 < nrows) {
                bacc0 += __dmul_rn(bep.w[r0], a0);
            }
        } else if (kBicg == 2) {  // t.t and t.s (s = x at the own rows)
            if (r0 + 1 < nrows) {
                const double2 s2 = *reinterpret_cast<const double2*>(x + r0);
                bacc0 += __dmul_rn(a0, a0);
                bacc0 += __dmul_rn(a1, a1);
                bacc1 += __dmul_rn(a0, s2.x);
                bacc1 += __dmul_rn(a1, s2.y);
            } else if (r0 < nrows) {
                bacc0 += __dmul_rn(a0, a0);
                bacc1 += __dmul_rn(a0, x[r0]);
            }
        }
        if (r0 + 1 < nrows) {
            if (kDot)
                *reinterpret_cast<double2*>(y + r0) = make_double2(a0, a1);
            else
                __stcs(reinterpret_cast<double2*>(y + r0), make_double2(a0, a1));
            if (kDot) {
                dacc += __dmul_rn(p.x, a0);
                dacc += __dmul_rn(p.y, a1);
            }
        } else if (r0 < nrows) {
            if (kDot)
                y[r0] = a0;
            else
                st_stream(y + r0, a0);
            if (kDot) dacc += __dmul_rn(p.x, a0);
        }
    };
    auto width = [&](int64_t k) -> int {
        return k < nslices ? int(__ldg(sets + SP(k) + 1) - __ldg(sets + SP(k))) : 0;
    };
    // slice cursor: the current slice s (width w) and the next non-empty one
    // sn (width wn; wnn = width of sn + nwarps, read ahead). Empty slices in
    // between are stored (zeros) as they are skipped.
    int64_t s = gwarp, sn = 0;
    int w = width(s), wn = 0, wnn = width(s + nwarps);
    auto next_nonempty = [&](int64_t from, int wfrom) {
        sn = from;
        wn = wfrom;
        wnn = width(sn + nwarps);
        while (sn < nslices && wn == 0) {
            emit(SP(sn) * 64 + 2 * lane, 0.0, 0.0, xown(SP(sn) * 64 + 2 * lane));
            sn += nwarps;
            wn = wnn;
            wnn = width(sn + nwarps);
        }
    };
    next_nonempty(s, w);  // first non-empty slice
    s = sn;
    w = wn;
    if (s >= nslices) goto done;
    {
        next_nonempty(s + nwarps, wnn);
        int j0 = 0;
        int64_t r0 = SP(s) * 64 + 2 * lane;
        int len0 = w, len1 = w;
        auto lens = [&]() {
            len0 = w;
            len1 = w;
            if (!finite0) {
                len0 = r0 < nrows ? row_lengths[r0] : 0;
                len1 = r0 + 1 < nrows ? row_lengths[r0 + 1] : 0;
            }
        };
        lens();
        double a0 = 0.0, a1 = 0.0;
        SellpChunkRegs<J> ca, cb;
        load(ca, s, w, 0);
        // one step: issue the gathers of the chunk after `cur` into `nxt`, then
        // fold `cur`; false when `cur` was the warp's last chunk. Called with
        // (ca, cb) and (cb, ca) alternately so both stay in registers.
        auto step = [&](SellpChunkRegs<J>& cur, SellpChunkRegs<J>& nxt) -> bool {
            const bool last = j0 + J >= w;
            if (!last)
                load(nxt, s, w, j0 + J);
            else if (sn < nslices)
                load(nxt, sn, wn, 0);
            if (finite0)
                sellp_chunk_fold<J, false>(cur, len0, len1, a0, a1);
            else
                sellp_chunk_fold<J, true>(cur, len0, len1, a0, a1);
            if (!last) {
                j0 += J;
                return true;
            }
            emit(r0, a0, a1, xown(r0));
            if (sn >= nslices) return false;
            s = sn;
            w = wn;
            j0 = 0;
            r0 = SP(s) * 64 + 2 * lane;
            lens();
            a0 = 0.0;
            a1 = 0.0;
            next_nonempty(s + nwarps, wnn);
            return true;
        };
        while (step(ca, cb) && step(cb, ca)) {
        }
    }
done:
    if (kBicg != 0) {
        RedWorkspace ws{bep.partials, bep.ticket};
        double t0, t1;
        if (grid_reduce_last2<WARPS * 32>(bacc0, bacc1, ws, t0, t1) && threadIdx.x == 0) {
            if (kBicg == 1) {
                bep.state->rv = t0;
            } else {
                bep.state->tt = t0;
                bep.state->ts = t1;
            }
        }
    }
    if (kDot) {
        RedWorkspace ws{dot.partials, dot.ticket};
        double total;
        if (grid_reduce_last<WARPS * 32>(dacc, ws, total) && threadIdx.x == 0) {
            if (dot.peer != nullptr) {
                peer_push_scalar(dot.peer, total);  // consumed by the next kernel's prologue
            } else {
                dot.state->pq = total;
                if (dot.finalize) cg_alpha_step(dot.state);
            }
        }
    }
}

// Launch one configuration (persistent grid: one CTA per SM).
template <class Cfg, bool kDot = false, bool kCoh = false, int kBicg = 0>
int launch_sellp64_tma(int64_t nrows, int64_t ncols, const int64_t* sets, const int* col, const double* val,
                       const int* row_lengths, const double* x, double* y, const int* skip, cudaStream_t st,
                       DotEpilogue dot = DotEpilogue{nullptr, nullptr, nullptr, 0, nullptr, nullptr}, int rev = 0,
                       BicgEpilogue bep = BicgEpilogue{nullptr, nullptr, nullptr, nullptr, 0}) {
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev & 63]) {
        WK_CUDA(cudaFuncSetAttribute(sellp64_tma_kernel<Cfg, kDot, kCoh, kBicg>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(Cfg::kSmem)));
        attr_set[dev & 63] = true;
    }
    const int64_t nslices = ceil_div(nrows, 64);
    int64_t grid = int64_t(sm_count()) * Cfg::kCtas;
    const int64_t need = ceil_div(nslices, Cfg::kWarps);
    if (grid > need) grid = need;
    sellp64_tma_kernel<Cfg, kDot, kCoh, kBicg><<<(unsigned)grid, Cfg::kWarps * 32, Cfg::kSmem, st>>>(
        nrows, ncols, nslices, sets, col, val, row_lengths, x, y, skip, dot, rev, bep);
    WK_LAUNCH_CHECK();
    return 0;
}

}  // namespace wk
