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

// kDot: also accumulate sum_r x[r] * y[r] over the owned rows (CG's p.Ap with
// x = p, y = q) and publish it through DotEpilogue (last-arriving CTA).
// kEll: ELL(width, stride) — one "slice" per 64-row block, column j of block
// b at j*stride + 64b (stride % 4 == 0): J bulk copies per chunk instead of 2.
template <class Cfg, bool kDot = false, bool kEll = false, bool kCoh = false>
__global__ void __launch_bounds__(Cfg::kWarps * 32, Cfg::kCtas)
sellp64_tma_kernel(int64_t nrows, int64_t ncols, int64_t nslices, const int64_t* __restrict__ sets,
                   const int* __restrict__ col, const double* __restrict__ val, const int* __restrict__ row_lengths,
                   const double* __restrict__ x, double* __restrict__ y, const int* __restrict__ skip,
                   DotEpilogue dot, int64_t ell_width = 0, int64_t ell_stride = 0, int rev = 0) {
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

    // producer cursor (warp-uniform; lane 0 issues)
    int64_t ps = gwarp, pbase = 0;
    int pj = 0, pw = 0;
    bool pvalid = false;
    // slice offsets are read one slice ahead (registers): the loads of the
    // next slice's sets[] entries are in flight while this slice streams,
    // instead of stalling the warp at every slice change (7-point slices are
    // only 2 chunks long)
    int64_t q0 = 0, q1 = 0, n0 = 0, n1 = 0;
    if (!kEll) {
        if (ps < nslices) {
            q0 = __ldg(sets + SP(ps));
            q1 = __ldg(sets + SP(ps) + 1);
        }
        if (ps + nwarps < nslices) {
            n0 = __ldg(sets + SP(ps + nwarps));
            n1 = __ldg(sets + SP(ps + nwarps) + 1);
        }
    }
    auto seek = [&]() {
        pvalid = false;
        while (ps < nslices) {
            if (kEll) {
                pw = int(ell_width);
                if (pj < pw) {
                    pbase = SP(ps) * 64;
                    pvalid = true;
                    return;
                }
                ps += nwarps;
                pj = 0;
                continue;
            }
            pw = int(q1 - q0);
            if (pj < pw) {
                pbase = q0 * 64;
                pvalid = true;
                return;
            }
            ps += nwarps;
            pj = 0;
            q0 = n0;
            q1 = n1;
            if (ps + nwarps < nslices) {
                n0 = __ldg(sets + SP(ps + nwarps));
                n1 = __ldg(sets + SP(ps + nwarps) + 1);
            }
        }
    };
    auto issue = [&](int st) {
        if (lane == 0) {
            const int nj = (pw - pj < J) ? pw - pj : J;
            if (kEll) {
                const int64_t cnt = (ell_stride - pbase < 64) ? ell_stride - pbase : 64;
                const uint32_t bv = uint32_t(cnt) * sizeof(double), bc = uint32_t(cnt) * sizeof(int);
                mbar_arrive_expect_tx(bars + st, uint32_t(nj) * (bv + bc));
                for (int jj = 0; jj < nj; ++jj) {
                    const int64_t off = int64_t(pj + jj) * ell_stride + pbase;
                    bulk_g2s_evict_first(sval + st * CH + jj * 64, val + off, bv, bars + st, pol);
                    bulk_g2s_evict_first(scol + st * CH + jj * 64, col + off, bc, bars + st, pol);
                }
            } else {
                const uint32_t bv = uint32_t(nj) * 64 * sizeof(double), bc = uint32_t(nj) * 64 * sizeof(int);
                mbar_arrive_expect_tx(bars + st, bv + bc);
                const int64_t off = pbase + int64_t(pj) * 64;
                bulk_g2s_evict_first(sval + st * CH, val + off, bv, bars + st, pol);
                bulk_g2s_evict_first(scol + st * CH, col + off, bc, bars + st, pol);
            }
        }
        pj += J;
        seek();
    };
    seek();
    for (int st = 0; st < S && pvalid; ++st) issue(st);
    // peer-memory distributed CG: the neighbours push the halo of x while this
    // kernel runs. Slices in [int_lo, int_hi) gather no halo column, so a warp
    // waits for the halo flags only before its first slice outside that range:
    // interior rows overlap the exchange, boundary rows run after arrival.
    // The slice order (and so every sum) is the same as without a halo.
    bool halo_pending = kDot && dot.halo != nullptr;
    int64_t int_lo = 0, int_hi = 0;
    if (halo_pending) {
        int_lo = dot.halo->int_lo;
        int_hi = dot.halo->int_hi;
    }

    int cst = 0;            // ring stage of the next chunk
    uint32_t cphase = 0;    // its mbarrier phase parity
    double dacc = 0.0;
    int cw = 0, cwn = 0;  // consumer: this slice's width and the next one's (read ahead)
    if (!kEll) {
        if (gwarp < nslices) cw = int(__ldg(sets + SP(gwarp) + 1) - __ldg(sets + SP(gwarp)));
        if (gwarp + nwarps < nslices)
            cwn = int(__ldg(sets + SP(gwarp + nwarps) + 1) - __ldg(sets + SP(gwarp + nwarps)));
    }
    for (int64_t s = gwarp; s < nslices; s += nwarps) {
        const int w = kEll ? int(ell_width) : cw;
        if (!kEll) {
            cw = cwn;
            if (s + 2 * nwarps < nslices)
                cwn = int(__ldg(sets + SP(s + 2 * nwarps) + 1) - __ldg(sets + SP(s + 2 * nwarps)));
        }
        const int64_t r0 = SP(s) * 64 + 2 * lane;
        const bool partial = kEll && (SP(s) + 1) * 64 > nrows;
        if (kDot && halo_pending && (SP(s) < int_lo || SP(s) >= int_hi)) {
            if (lane == 0) halo_wait(dot.peer, dot.halo);
            __syncwarp();
            halo_pending = false;
        }
        int len0 = w, len1 = w;
        if (!finite0) {
            len0 = r0 < nrows ? row_lengths[r0] : 0;
            len1 = r0 + 1 < nrows ? row_lengths[r0 + 1] : 0;
        }
        double a0 = 0.0, a1 = 0.0;
        for (int j0 = 0; j0 < w; j0 += J) {
            const int st = cst;
            mbar_wait(bars + st, cphase);
            const int nj = (w - j0 < J) ? w - j0 : J;
            const double* v = sval + st * CH + 2 * lane;
            const int* c = scol + st * CH + 2 * lane;
            if (kEll && partial)
                sellp_chunk<J, true, true, 64, kCoh>(v, c, nj, j0, len0, len1, x, a0, a1, r0 < nrows, r0 + 1 < nrows);
            else if (finite0)
                sellp_chunk<J, false, false, 64, kCoh>(v, c, nj, j0, len0, len1, x, a0, a1);
            else
                sellp_chunk<J, true, false, 64, kCoh>(v, c, nj, j0, len0, len1, x, a0, a1);
            __syncwarp();
            if (pvalid) {
                if (lane == 0) fence_proxy_async_smem();
                issue(st);
            }
            if (++cst == S) {
                cst = 0;
                cphase ^= 1u;
            }
        }
        if (r0 + 1 < nrows) {
            __stcs(reinterpret_cast<double2*>(y + r0), make_double2(a0, a1));
            if (kDot) {
                const double2 p = *reinterpret_cast<const double2*>(x + r0);
                dacc += __dmul_rn(p.x, a0);
                dacc += __dmul_rn(p.y, a1);
            }
        } else if (r0 < nrows) {
            st_stream(y + r0, a0);
            if (kDot) dacc += __dmul_rn(x[r0], a0);
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

// Launch one configuration (persistent grid: one CTA per SM). kEll: sets is
// unused, the operand is ELL(ell_width, ell_stride).
template <class Cfg, bool kDot = false, bool kEll = false, bool kCoh = false>
int launch_sellp64_tma(int64_t nrows, int64_t ncols, const int64_t* sets, const int* col, const double* val,
                       const int* row_lengths, const double* x, double* y, const int* skip, cudaStream_t st,
                       DotEpilogue dot = DotEpilogue{nullptr, nullptr, nullptr, 0, nullptr, nullptr}, int64_t ell_width = 0,
                       int64_t ell_stride = 0, int rev = 0) {
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev & 63]) {
        WK_CUDA(cudaFuncSetAttribute(sellp64_tma_kernel<Cfg, kDot, kEll, kCoh>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(Cfg::kSmem)));
        attr_set[dev & 63] = true;
    }
    const int64_t nslices = ceil_div(nrows, 64);
    int64_t grid = int64_t(sm_count()) * Cfg::kCtas;
    const int64_t need = ceil_div(nslices, Cfg::kWarps);
    if (grid > need) grid = need;
    sellp64_tma_kernel<Cfg, kDot, kEll, kCoh><<<(unsigned)grid, Cfg::kWarps * 32, Cfg::kSmem, st>>>(
        nrows, ncols, nslices, sets, col, val, row_lengths, x, y, skip, dot, ell_width, ell_stride, rev);
    WK_LAUNCH_CHECK();
    return 0;
}

}  // namespace wk
