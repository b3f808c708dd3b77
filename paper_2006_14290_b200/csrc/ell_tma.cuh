// ELL SpMV with TMA bulk-copy staging and a producer warp (ell_kernel 2, the
// default for aligned ELL operands).
//
// ELL stores column j of every row contiguously (`col/val[j * stride + r]`,
// SELL-P with one slice of stride `stride`, sparse.py:233-241 addressing), so
// a block of R consecutive rows is R*8 bytes of values + R*4 bytes of column
// indices per column, `width` such pairs 8*stride / 4*stride bytes apart.
// The SELL-P(64) warp pipeline (sellp_tma.cuh, kEll) moves these as 512 B +
// 256 B copies — millions of tiny TMA transactions, 3.5x slower than plain
// loads. Here a CTA owns R = 2*T rows: one producer warp streams J columns
// per stage (two copies per column: 4 KB + 2 KB at R = 512) into an S-deep ring,
// T consumer threads fold two rows each from shared memory (128-bit loads),
// gather x through L1/L2 and fold with separately rounded multiply/add in
// column order (bitwise == the reference fold, sparse.py:405-416). Stage reuse
// is tracked by a `full` mbarrier (producer arrive + tx bytes) and an `empty`
// mbarrier (one arrive per consumer warp).
#pragma once

#include "sellp_tma.cuh"

namespace wk {

template <int J, int S, int T, int CTAS>
struct EllTmaCfg {
    static constexpr int kJ = J, kS = S, kT = T, kCtas = CTAS;
    static constexpr int kRows = 2 * T;
    static constexpr size_t kSmem = size_t(S) * J * kRows * (sizeof(double) + sizeof(int)) + 2 * S * 8;
};

// kDot (CG): also p.q over the owned rows into the DotEpilogue (x = p);
// rev: tiles walked from the last one (CG's L2 ping-pong, krylov.cu).
template <class Cfg, bool kDot = false>
__global__ void __launch_bounds__(Cfg::kT + 32, Cfg::kCtas)
ell_tma_kernel(int64_t nrows, int64_t ncols, int64_t width, int64_t stride, const int* __restrict__ col,
               const double* __restrict__ val, const int* __restrict__ row_lengths, const double* __restrict__ x,
               double* __restrict__ y, const int* __restrict__ skip,
               DotEpilogue dot = DotEpilogue{nullptr, nullptr, nullptr, 0, nullptr, nullptr}, int rev = 0) {
    constexpr int J = Cfg::kJ, S = Cfg::kS, T = Cfg::kT, R = Cfg::kRows;
    if (skip != nullptr && *skip) return;
    extern __shared__ __align__(128) unsigned char smem[];
    double* sval = reinterpret_cast<double*>(smem);                                  // [S][J][R]
    int* scol = reinterpret_cast<int*>(smem + size_t(S) * J * R * sizeof(double));    // [S][J][R]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(S) * J * R * 12);
    uint64_t* empty = full + S;
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int st = 0; st < S; ++st) {
            mbar_init(full + st, 1);
            mbar_init(empty + st, T / 32);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int64_t ntiles = (nrows + R - 1) / R;
    const int nchunks = int((width + J - 1) / J);
    auto TL = [&](int64_t k) -> int64_t { return (kDot && rev) ? ntiles - 1 - k : k; };
    double dacc = 0.0;

    if (tid >= T) {  // producer warp: lane 0 streams the (tile, chunk) sequence
        if (tid == T) {
        const uint64_t pol = policy_evict_first();
        uint32_t i = 0;
        for (int64_t tk = blockIdx.x; tk < ntiles; tk += gridDim.x) {
            const int64_t tile = TL(tk);
            const int64_t base = tile * R;
            const int64_t cnt = (stride - base < R) ? stride - base : R;  // multiple of 4 (stride % 4 == 0)
            for (int c = 0; c < nchunks; ++c, ++i) {
                const int st = int(i % S);
                if (i >= uint32_t(S)) mbar_wait(empty + st, ((i / S) - 1) & 1);
                const int nj = (width - int64_t(c) * J < J) ? int(width - int64_t(c) * J) : J;
                fence_proxy_async_smem();  // the consumers' reads of this stage before the new bulk writes
                mbar_arrive_expect_tx(full + st, uint32_t(nj) * uint32_t(cnt) * 12u);
                for (int jj = 0; jj < nj; ++jj) {
                    const int64_t off = (int64_t(c) * J + jj) * stride + base;
                    bulk_g2s_evict_first(sval + (size_t(st) * J + jj) * R, val + off, uint32_t(cnt) * 8u, full + st,
                                         pol);
                    bulk_g2s_evict_first(scol + (size_t(st) * J + jj) * R, col + off, uint32_t(cnt) * 4u, full + st,
                                         pol);
                }
            }
        }
        }
        if (!kDot) return;
    } else {

    const int lane = tid & 31;
    const bool finite0 = ncols == 0 || isfinite(__ldg(x));
    uint32_t i = 0;
    for (int64_t tk = blockIdx.x; tk < ntiles; tk += gridDim.x) {
        const int64_t tile = TL(tk);
        const int64_t r0 = tile * R + 2 * tid;
        const bool ok0 = r0 < nrows, ok1 = r0 + 1 < nrows;
        const bool partial = (tile + 1) * R > nrows;
        int len0 = int(width), len1 = int(width);
        if (!finite0) {
            len0 = ok0 ? row_lengths[r0] : 0;
            len1 = ok1 ? row_lengths[r0 + 1] : 0;
        }
        double a0 = 0.0, a1 = 0.0;
        for (int c = 0; c < nchunks; ++c, ++i) {
            const int st = int(i % S);
            mbar_wait(full + st, (i / S) & 1);
            const int j0 = c * J;
            const int nj = (width - j0 < J) ? int(width - j0) : J;
            const double* v = sval + size_t(st) * J * R + 2 * tid;
            const int* cc = scol + size_t(st) * J * R + 2 * tid;
            if (partial)
                sellp_chunk<J, true, true, R>(v, cc, nj, j0, len0, len1, x, a0, a1, ok0, ok1);
            else if (finite0)
                sellp_chunk<J, false, false, R>(v, cc, nj, j0, len0, len1, x, a0, a1);
            else
                sellp_chunk<J, true, false, R>(v, cc, nj, j0, len0, len1, x, a0, a1);
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + st);
        }
        if (ok1) {
            __stcs(reinterpret_cast<double2*>(y + r0), make_double2(a0, a1));
            if (kDot) {
                const double2 p = *reinterpret_cast<const double2*>(x + r0);
                dacc += __dmul_rn(p.x, a0);
                dacc += __dmul_rn(p.y, a1);
            }
        } else if (ok0) {
            st_stream(y + r0, a0);
            if (kDot) dacc += __dmul_rn(x[r0], a0);
        }
    }
    }
    if (kDot) {
        RedWorkspace ws{dot.partials, dot.ticket};
        double total;
        if (grid_reduce_last<T + 32>(dacc, ws, total) && threadIdx.x == 0) {
            if (dot.peer != nullptr) {
                peer_push_scalar(dot.peer, total);
            } else {
                dot.state->pq = total;
                if (dot.finalize) cg_alpha_step(dot.state);
            }
        }
    }
}

template <class Cfg, bool kDot = false>
int launch_ell_tma(int64_t nrows, int64_t ncols, int64_t width, int64_t stride, const int* col, const double* val,
                   const int* row_lengths, const double* x, double* y, const int* skip, cudaStream_t st,
                   DotEpilogue dot = DotEpilogue{nullptr, nullptr, nullptr, 0, nullptr, nullptr}, int rev = 0) {
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev & 63]) {
        WK_CUDA(cudaFuncSetAttribute(ell_tma_kernel<Cfg, kDot>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(Cfg::kSmem)));
        attr_set[dev & 63] = true;
    }
    int64_t grid = int64_t(sm_count()) * Cfg::kCtas;
    const int64_t ntiles = ceil_div(nrows, int64_t(Cfg::kRows));
    if (grid > ntiles) grid = ntiles;
    ell_tma_kernel<Cfg, kDot><<<(unsigned)grid, Cfg::kT + 32, Cfg::kSmem, st>>>(nrows, ncols, width, stride, col,
                                                                               val, row_lengths, x, y, skip, dot, rev);
    WK_LAUNCH_CHECK();
    return 0;
}

}  // namespace wk
