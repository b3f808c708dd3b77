// SpMV kernels for B200 (sm_100a), fp64 values, int32 indices.
//
// Formats and their reference anchors:
//   SELL-P  warpkit/sparse.py:147-209 (layout), kernels.py:116-157 (thread per
//           row over the full slice width), sparse.py:397-417 (oracle fold)
//   ELL     SELL-P with one slice of stride `stride` (no reference)
//   CSR     kernels.py:163-203 (subwarp per row), sparse.py:384-396 (fold)
//   COO     kernels.py:209-264 (segmented reduction + atomics), sparse.py:374-383
//   Hybrid  ELL part + COO remainder (no reference; Ginkgo's hybrid format)
//
// Bit-exactness: the column-major kernels (SELL-P, ELL) and the CSR "stream"
// kernel fold every row sequentially in stored order with separately rounded
// multiply and add — the reference fold — so they are bitwise equal to the
// oracle. The library is compiled with -fmad=false and the folds use
// __dmul_rn/__dadd_rn explicitly. Padding slots hold (col 0, 0.0): adding
// 0.0*x[0] never changes a fold (acc starts at +0.0 and x + (+-0) == x for
// x != 0, +0 + -0 == +0) as long as x[0] is finite; if it is not, the
// kernels switch to the `row_lengths`-bounded loop of the oracle.
#include "common.cuh"
#include "csr_merge.cuh"
#include "segwarp.cuh"
#include "csr_tma.cuh"
#include "sellp_tma.cuh"
#include "ell_tma.cuh"

namespace wk {

constexpr int kSpmvThreads = 256;

// ---------------------------------------------------------------------------
// Column-major sliced storage (SELL-P, ELL). Thread handles R adjacent rows of
// one slice; R == 2 uses 128-bit value loads and 64-bit index loads.
// ---------------------------------------------------------------------------
template <int R, bool kEll>
__global__ void __launch_bounds__(kSpmvThreads)
sliced_spmv_kernel(int64_t nrows, int64_t ncols, int log2ss, int64_t ell_width, int64_t ell_stride,
                   const int64_t* __restrict__ sets, const int* __restrict__ col,
                   const double* __restrict__ val, const int* __restrict__ row_lengths,
                   const double* __restrict__ x, double* __restrict__ y, const int* __restrict__ skip) {
    if (skip != nullptr && *skip) return;
    const int64_t r0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * R;
    if (r0 >= nrows) return;
    const bool finite0 = ncols == 0 || isfinite(__ldg(x));
    int64_t k, stride, width;
    if (kEll) {
        k = r0;
        stride = ell_stride;
        width = ell_width;
    } else {
        const int64_t s = r0 >> log2ss;
        const int64_t s0 = __ldg(sets + s);
        k = (s0 << log2ss) + (r0 & ((int64_t(1) << log2ss) - 1));
        stride = int64_t(1) << log2ss;
        width = __ldg(sets + s + 1) - s0;
    }
    if (R == 1) {
        const int64_t len = finite0 ? width : row_lengths[r0];
        double acc = 0.0;
        int64_t j = 0;
        for (; j + 4 <= len; j += 4) {
            double v[4];
            int c[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                v[u] = ld_stream(val + k + u * stride);
                c[u] = ld_stream(col + k + u * stride);
            }
            double xv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) xv[u] = ld_x(x, c[u]);
#pragma unroll
            for (int u = 0; u < 4; ++u) acc = mul_add_rn(acc, v[u], xv[u]);
            k += 4 * stride;
        }
        for (; j < len; ++j, k += stride) acc = mul_add_rn(acc, ld_stream(val + k), ld_x(x, ld_stream(col + k)));
        st_stream(y + r0, acc);
    } else {
        const bool has1 = r0 + 1 < nrows;
        int64_t len0 = width, len1 = width;
        if (!finite0) {
            len0 = row_lengths[r0];
            len1 = has1 ? row_lengths[r0 + 1] : 0;
        }
        const int64_t len = len0 > len1 ? len0 : len1;
        double a0 = 0.0, a1 = 0.0;
        int64_t j = 0;
        if (finite0) {
            for (; j + 4 <= len; j += 4) {
                double2 v[4];
                int2 c[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    v[u] = ld_stream(reinterpret_cast<const double2*>(val + k + u * stride));
                    c[u] = ld_stream(reinterpret_cast<const int2*>(col + k + u * stride));
                }
                double x0[4], x1[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    x0[u] = ld_x(x, c[u].x);
                    x1[u] = ld_x(x, c[u].y);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    a0 = mul_add_rn(a0, v[u].x, x0[u]);
                    a1 = mul_add_rn(a1, v[u].y, x1[u]);
                }
                k += 4 * stride;
            }
        }
        for (; j < len; ++j, k += stride) {
            const double2 v = ld_stream(reinterpret_cast<const double2*>(val + k));
            const int2 c = ld_stream(reinterpret_cast<const int2*>(col + k));
            if (j < len0) a0 = mul_add_rn(a0, v.x, ld_x(x, c.x));
            if (j < len1) a1 = mul_add_rn(a1, v.y, ld_x(x, c.y));
        }
        if (has1) {
            // y + r0 is 16-byte aligned when y is (r0 even).
            __stcs(reinterpret_cast<double2*>(y + r0), make_double2(a0, a1));
        } else {
            st_stream(y + r0, a0);
        }
    }
}

static bool aligned(const void* p, int a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

static int log2i(int64_t v) {
    int l = 0;
    while ((int64_t(1) << l) < v) ++l;
    return l;
}

// SELL-P(64) TMA pipeline configuration by mean slice width (`stored` =
// stored slots; 0 = unknown): narrow slices (the 7-point operators of CG,
// BiCGSTAB, GMRES: width 7) stream 2-column chunks through 5-stage rings of
// 24 warps — more independent warp pipelines, each with shorter gather
// rounds; wide slices (27-point: width 27) 4-column chunks, 3 stages, 16
// warps. Sweeps: profiles/r01/sellp_sweep*.jsonl, profiles/r02/sellp_sweep.log
// (7-pt 256^3: 0.267 vs 0.275 ms; 27-pt 200^3: 0.389 vs 0.405 ms).
using SellpNarrow = SellpTmaCfg<2, 5, 24, 1>;
using SellpWide = SellpTmaCfg<4, 3, 16, 1>;
constexpr int64_t kSellpNarrowWidth = 12;

static bool sellp_narrow(int64_t nrows, int64_t stored) {
    return stored > 0 && stored <= kSellpNarrowWidth * 64 * ceil_div(nrows, 64);
}

int launch_sellp(int64_t nrows, int64_t ncols, int64_t ss, const int64_t* sets, const int* col,
                 const double* val, const int* row_lengths, const double* x, double* y,
                 const int* skip, cudaStream_t st, int64_t stored = 0) {
    if (nrows == 0) return 0;
    const int l2 = log2i(ss);
    // SELL-P(64), 16-byte aligned: the TMA pipeline; otherwise the register kernel.
    if (ss == 64 && aligned(val, 16) && aligned(col, 16) && aligned(y, 16)) {
        if (sellp_narrow(nrows, stored))
            return launch_sellp64_tma<SellpNarrow>(nrows, ncols, sets, col, val, row_lengths, x, y, skip, st);
        return launch_sellp64_tma<SellpWide>(nrows, ncols, sets, col, val, row_lengths, x, y, skip, st);
    }
    const bool vec = ss >= 2 && aligned(val, 16) && aligned(col, 8) && aligned(y, 16);
    if (vec) {
        const int64_t threads = ceil_div(nrows, 2);
        sliced_spmv_kernel<2, false><<<(unsigned)ceil_div(threads, kSpmvThreads), kSpmvThreads, 0, st>>>(
            nrows, ncols, l2, 0, 0, sets, col, val, row_lengths, x, y, skip);
    } else {
        sliced_spmv_kernel<1, false><<<(unsigned)ceil_div(nrows, kSpmvThreads), kSpmvThreads, 0, st>>>(
            nrows, ncols, l2, 0, 0, sets, col, val, row_lengths, x, y, skip);
    }
    WK_LAUNCH_CHECK();
    return 0;
}

// CG's q = A p with p.q fused into the SpMV (SELL-P(64) TMA kernel only).
// Returns 1 when the operand cannot take the fused path (caller falls back to
// SpMV + separate dot), 0 on success, an error code otherwise.
int spmv_dot_fused(const wk_matrix* A, const double* p, double* q, wk_cg_state* s, void* red_ws, int finalize,
                   cudaStream_t st, void* peer, const void* halo, int rev) {
    if (A->format == WK_FMT_ELL && halo == nullptr && A->stride % 4 == 0 &&
        A->width > 0 && aligned(A->values, 16) && aligned(A->col_idx, 16) && aligned(q, 16) && aligned(p, 16) &&
        A->nrows > 0) {
        char* w = reinterpret_cast<char*>(red_ws);
        DotEpilogue dot{reinterpret_cast<double*>(w),
                        reinterpret_cast<unsigned*>(w + sizeof(double) * kRedMaxVec * kRedMaxBlocks), s, finalize,
                        reinterpret_cast<PeerCtx*>(peer), nullptr};
        return launch_ell_tma<EllTmaCfg<4, 4, 448, 1>, true>(A->nrows, A->ncols, A->width, A->stride, A->col_idx,
                                                            A->values, A->row_lengths, p, q, &s->done, st, dot, rev);
    }
    if (A->format != WK_FMT_SELLP || A->slice_size != 64 || !aligned(A->values, 16) ||
        !aligned(A->col_idx, 16) || !aligned(q, 16) || !aligned(p, 16) || A->nrows == 0)
        return 1;
    char* w = reinterpret_cast<char*>(red_ws);
    DotEpilogue dot{reinterpret_cast<double*>(w),
                    reinterpret_cast<unsigned*>(w + sizeof(double) * kRedMaxVec * kRedMaxBlocks), s, finalize,
                    reinterpret_cast<PeerCtx*>(peer), reinterpret_cast<const PeerHalo*>(halo)};
    // narrow slices (CG's 7-point operator): the narrow configuration (the
    // register-lean cursor state keeps its fused-dot variant at 80 registers,
    // no spills: 279 vs 287 us for the wide one); the peer variant, with its
    // halo logic, keeps the wide configuration
    if (halo == nullptr && sellp_narrow(A->nrows, A->nnz))
        return launch_sellp64_tma<SellpNarrow, true>(A->nrows, A->ncols, A->slice_sets, A->col_idx, A->values,
                                                     A->row_lengths, p, q, &s->done, st, dot, rev);
    if (halo != nullptr)  // peer CG: the halo of p lands during the kernel (coherent gathers)
        return launch_sellp64_tma<SellpWide, true, true>(A->nrows, A->ncols, A->slice_sets, A->col_idx, A->values,
                                                         A->row_lengths, p, q, &s->done, st, dot, rev);
    return launch_sellp64_tma<SellpWide, true>(A->nrows, A->ncols, A->slice_sets, A->col_idx, A->values,
                                               A->row_lengths, p, q, &s->done, st, dot, rev);
}

// BiCGSTAB's SpMVs with their dots fused (wk_bicgstab_solve): mode 1
// (v = A p): state->rv = r-hat.v; mode 2 (t = A s): state->tt = t.t,
// state->ts = t.s. SELL-P(64), 16-byte aligned only; returns 1 otherwise (the
// caller runs the SpMV and the dot pass separately).
int spmv_bicg_fused(const wk_matrix* A, const double* xin, double* y, wk_bicg_state* s, const double* w, int mode,
                    void* red_ws, cudaStream_t st) {
    if (A->format != WK_FMT_SELLP || A->slice_size != 64 || A->nrows == 0 || !aligned(A->values, 16) ||
        !aligned(A->col_idx, 16) || !aligned(y, 16) || !aligned(xin, 16) || (mode == 1 && !aligned(w, 16)))
        return 1;
    char* wb = reinterpret_cast<char*>(red_ws);
    BicgEpilogue bep{reinterpret_cast<double*>(wb),
                     reinterpret_cast<unsigned*>(wb + sizeof(double) * kRedMaxVec * kRedMaxBlocks), s, w, mode};
    const DotEpilogue none{nullptr, nullptr, nullptr, 0, nullptr, nullptr};
    const bool narrow = sellp_narrow(A->nrows, A->nnz);
    if (mode == 1) {
        if (narrow)
            return launch_sellp64_tma<SellpNarrow, false, false, 1>(A->nrows, A->ncols, A->slice_sets, A->col_idx,
                                                                   A->values, A->row_lengths, xin, y, &s->done, st,
                                                                   none, 0, bep);
        return launch_sellp64_tma<SellpWide, false, false, 1>(A->nrows, A->ncols, A->slice_sets, A->col_idx, A->values,
                                                             A->row_lengths, xin, y, &s->done, st, none, 0, bep);
    }
    if (narrow)
        return launch_sellp64_tma<SellpNarrow, false, false, 2>(A->nrows, A->ncols, A->slice_sets, A->col_idx,
                                                               A->values, A->row_lengths, xin, y, &s->done, st, none,
                                                               0, bep);
    return launch_sellp64_tma<SellpWide, false, false, 2>(A->nrows, A->ncols, A->slice_sets, A->col_idx, A->values,
                                                         A->row_lengths, xin, y, &s->done, st, none, 0, bep);
}

int launch_ell(int64_t nrows, int64_t ncols, int64_t width, int64_t stride, const int* col,
               const double* val, const int* row_lengths, const double* x, double* y, const int* skip,
               cudaStream_t st) {
    if (nrows == 0) return 0;
    // aligned, stride % 4 == 0: the producer-warp TMA kernel (896-row tiles,
    // 4 columns per stage, 4 stages); otherwise the register kernel. (The
    // SELL-P(64) warp pipeline with ELL addressing moves 512 B + 256 B copies
    // per column and 64-row block and was 3.5x slower: removed.)
    if (stride % 4 == 0 && aligned(val, 16) && aligned(col, 16) && aligned(y, 16) && width > 0)
        return launch_ell_tma<EllTmaCfg<4, 4, 448, 1>>(nrows, ncols, width, stride, col, val, row_lengths, x, y, skip,
                                                       st);
    const bool vec = (stride % 2 == 0) && aligned(val, 16) && aligned(col, 8) && aligned(y, 16);
    if (vec) {
        const int64_t threads = ceil_div(nrows, 2);
        sliced_spmv_kernel<2, true><<<(unsigned)ceil_div(threads, kSpmvThreads), kSpmvThreads, 0, st>>>(
            nrows, ncols, 0, width, stride, nullptr, col, val, row_lengths, x, y, skip);
    } else {
        sliced_spmv_kernel<1, true><<<(unsigned)ceil_div(nrows, kSpmvThreads), kSpmvThreads, 0, st>>>(
            nrows, ncols, 0, width, stride, nullptr, col, val, row_lengths, x, y, skip);
    }
    WK_LAUNCH_CHECK();
    return 0;
}

// ---------------------------------------------------------------------------
// CSR "stream" (load-balanced, bitwise for rows of <= kCsrChunk entries).
//
// The nonzeros are cut into chunks of kCsrChunk entries; work item c owns the
// rows whose first entry lies in chunk c (first[c] .. first[c+1]), so every
// item covers < 2*kCsrChunk entries of short rows. The products v*x[c] of an
// item are staged in shared memory with coalesced 128-bit loads, then each
// thread folds whole rows sequentially from shared memory (the reference
// fold, bit for bit). A "long" row (> kCsrChunk entries) is split across the
// items its entries fall into; each item writes a partial and the last one to
// arrive (atomic ticket) adds the partials in chunk order — deterministic,
// but reassociated, so long rows are checked with the 1e-12 tolerance.
// ---------------------------------------------------------------------------
// kCsrChunk / kCsrCap: csr_tma.cuh (shared plan geometry)

__global__ void csr_plan_kernel(int64_t nrows, int64_t nnz, int64_t nchunks, const int* __restrict__ ptrs,
                                int* __restrict__ first) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r > nrows) return;
    // first[c] = min{ r : ptrs[r] >= c*S }, rows r in [0, nrows]; ptrs[nrows] = nnz.
    // Only the virtual row r == nrows writes first[nchunks] (= nrows), so the
    // last item also covers trailing empty rows.
    int64_t hi = (r == nrows) ? nchunks : int64_t(ptrs[r]) / kCsrChunk;
    if (r < nrows && hi > nchunks - 1) hi = nchunks - 1;
    const int64_t lo = (r == 0) ? 0 : int64_t(ptrs[r - 1]) / kCsrChunk + 1;
    for (int64_t c = lo; c <= hi; ++c) first[c] = int(r);
}

int64_t csr_stream_chunks(int64_t nnz) {
    const int64_t n = ceil_div(nnz, kCsrChunk);
    return n < 1 ? 1 : n;
}

// ---------------------------------------------------------------------------
// CSR subwarp-per-row (Ginkgo "classical"; kernels.py:163-196): a tile of T
// lanes strides the row, butterfly reduction, rank 0 writes. T == 1 is the
// sequential thread-per-row fold (bitwise).
// ---------------------------------------------------------------------------
// Two rows per tile in flight, software-pipelined: the next group's row
// bounds load while this group's first entries and x gathers are in flight,
// so a group costs two dependent round trips instead of three. Measured on
// the 27-point 200^3 operator (tools/subwarp_probe.py, same box): 4 rows
// unpipelined 1.06 ms (T = 32) / 0.84 ms (T = 4); this kernel 0.69 ms at
// T = 16; 4 or 8 rows with deeper prefetch 0.94-1.33 ms (registers: fewer
// resident warps). Per row the arithmetic is unchanged: lane l folds entries
// lo + l, lo + l + T, ... in order, then the butterfly.
template <unsigned T>
__global__ void __launch_bounds__(kSpmvThreads)
csr_subwarp_kernel(int64_t nrows, const int* __restrict__ ptrs, const int* __restrict__ col,
                   const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y,
                   const int* __restrict__ skip) {
    constexpr int kRows = 2;
    if (skip != nullptr && *skip) return;
    auto tile = cg::tiled_partition<T>(cg::this_thread_block());
    const int64_t tiles_per_grid = int64_t(gridDim.x) * (kSpmvThreads / T);
    const int64_t step = kRows * tiles_per_grid;
    const int tr = int(tile.thread_rank());
    int lo[kRows], hi[kRows];
    auto bounds = [&](int64_t r0, int* l, int* h) {
#pragma unroll
        for (int u = 0; u < kRows; ++u) {
            const int64_t row = r0 + u * tiles_per_grid;
            l[u] = row < nrows ? __ldg(ptrs + row) : 0;
            h[u] = row < nrows ? __ldg(ptrs + row + 1) : 0;
        }
    };
    int64_t row0 = int64_t(blockIdx.x) * (kSpmvThreads / T) + tile.meta_group_rank();
    bounds(row0, lo, hi);
    for (; row0 < nrows; row0 += step) {
        int c0[kRows];
        double v0[kRows], x0[kRows];
#pragma unroll
        for (int u = 0; u < kRows; ++u) {
            const int k = lo[u] + tr;
            c0[u] = k < hi[u] ? ld_stream(col + k) : 0;
            v0[u] = k < hi[u] ? ld_stream(val + k) : 0.0;
        }
        int nlo[kRows], nhi[kRows];
        bounds(row0 + step, nlo, nhi);
#pragma unroll
        for (int u = 0; u < kRows; ++u) x0[u] = lo[u] + tr < hi[u] ? ld_x(x, c0[u]) : 0.0;
        double acc[kRows];
#pragma unroll
        for (int u = 0; u < kRows; ++u) {
            acc[u] = 0.0;
            if (lo[u] + tr < hi[u]) acc[u] = mul_add_rn(0.0, v0[u], x0[u]);
            for (int k = lo[u] + tr + int(T); k < hi[u]; k += T)
                acc[u] = mul_add_rn(acc[u], ld_stream(val + k), ld_x(x, ld_stream(col + k)));
        }
#pragma unroll
        for (int u = 0; u < kRows; ++u) {
            const double r = reduce_subwarp(tile, acc[u]);
            const int64_t row = row0 + u * tiles_per_grid;
            if (tr == 0 && row < nrows) y[row] = r;
            lo[u] = nlo[u];
            hi[u] = nhi[u];
        }
    }
}

// CSR rows of at most a few entries (rowblock strategy, mean row length <=
// kShortRow). A small cold operand (config 1: 80 MB, under the L2 size) is
// bound by the dependent round trips row_ptrs -> col/val -> x, not by
// bandwidth: one thread per row over a full grid (every row in flight as soon
// as a slot frees), the row's kShortRow column/value loads issued together,
// then its kShortRow gathers together, then the sequential fold (the
// reference fold, bitwise). Longer rows repeat the batch. The persistent TMA
// row-block kernel spends one more round trip per block on its staging ring
// (24.5 us vs this kernel's ... us on config 1; profiles/r02).
constexpr int kShortRow = 8;

__global__ void __launch_bounds__(kSpmvThreads)
csr_short_kernel(int64_t nrows, const int* __restrict__ ptrs, const int* __restrict__ col,
                 const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y,
                 const int* __restrict__ skip) {
    if (skip != nullptr && *skip) return;
    const int64_t r = int64_t(blockIdx.x) * kSpmvThreads + threadIdx.x;
    if (r >= nrows) return;
    const int lo = ld_stream(ptrs + r), hi = ld_stream(ptrs + r + 1);
    double acc = 0.0;
    for (int k0 = lo; k0 < hi; k0 += kShortRow) {
        int c[kShortRow];
        double v[kShortRow], xv[kShortRow];
#pragma unroll
        for (int u = 0; u < kShortRow; ++u) {
            c[u] = k0 + u < hi ? ld_stream(col + k0 + u) : 0;
            v[u] = k0 + u < hi ? ld_stream(val + k0 + u) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kShortRow; ++u) xv[u] = k0 + u < hi ? ld_x(x, c[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < kShortRow; ++u)
            if (k0 + u < hi) acc = mul_add_rn(acc, v[u], xv[u]);
    }
    st_stream(y + r, acc);
}

__global__ void zero_masked_kernel(double* __restrict__ y, int64_t n, const int* __restrict__ skip) {
    if (*skip) return;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) y[i] = 0.0;
}

static int launch_zero_masked(double* y, int64_t n, const int* skip, cudaStream_t st) {
    if (n == 0) return 0;
    int64_t blocks = ceil_div(n, 256);
    if (blocks > int64_t(sm_count()) * 8) blocks = int64_t(sm_count()) * 8;
    zero_masked_kernel<<<(unsigned)blocks, 256, 0, st>>>(y, n, skip);
    WK_LAUNCH_CHECK();
    return 0;
}

int launch_csr(int64_t nrows, int64_t ncols, int64_t nnz, const int* ptrs, const int* col, const double* val,
               const double* x, double* y, int strategy, int subwarp, const int* first, double* partials,
               unsigned* tickets, const int* skip, cudaStream_t st, void* merge_plan = nullptr) {
    (void)ncols;
    if (nrows == 0) return 0;
    if (strategy == WK_CSR_MERGE) {
        WK_REQUIRE(merge_plan != nullptr, WK_ERR_INVALID, "csr merge strategy needs a plan (wk_csr_merge_plan_build)");
        return launch_csr_merge(nrows, nnz, ptrs, col, val, x, y, merge_plan, skip, st);
    }
    if (strategy == WK_CSR_LOAD_BALANCE) {
        WK_REQUIRE(merge_plan != nullptr, WK_ERR_INVALID,
                   "csr load_balance strategy needs a plan (wk_csr_load_balance_plan_build)");
        // skip-aware zero fill: rows without entries are never stored by the
        // kernel (every other row is stored once, by the range closing it)
        if (skip == nullptr) {
            WK_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * size_t(nrows), st));
        } else {
            WK_TRY(launch_zero_masked(y, nrows, skip, st));
        }
        if (nnz == 0) return 0;
        WK_REQUIRE(aligned(col, 16) && aligned(val, 16), WK_ERR_INVALID,
                   "csr load_balance needs 16-byte aligned col_idx / values");
        const HeadPlanMut h = head_plan_views(merge_plan, nrows, nnz);
        return launch_seg8(true, nnz, 0, nullptr, col, val, x, y, skip, st,
                           HeadPlan{h.hoff, h.mask, h.hrow, h.crow, h.cval, h.rrow});
    }
    if (strategy == WK_CSR_ROWBLOCK) {
        // mean row length <= 8 (2-D stencils, BASELINE config 1): one thread
        // per row, every load of a row issued at once (csr_short_kernel)
        if (nnz <= int64_t(kShortRow) * nrows) {
            csr_short_kernel<<<(unsigned)ceil_div(nrows, kSpmvThreads), kSpmvThreads, 0, st>>>(nrows, ptrs, col, val,
                                                                                            x, y, skip);
            WK_LAUNCH_CHECK();
            return 0;
        }
        // 32*k-row blocks; the stage capacity is the smallest that keeps a
        // 32-row block of mean-length rows "light" (more warps per SM when
        // rows are short). Measured sweep: profiles/r01/csr_sweep.jsonl.
        const double need = 32.0 * double(nnz) / double(nrows) * 1.25;
        if (need <= 640.0) return launch_csr_rowblock<CsrRbCfg<24, 1, 640>>(nrows, nnz, ptrs, col, val, x, y, skip, st);
        if (need <= 768.0) return launch_csr_rowblock<CsrRbCfg<20, 1, 768>>(nrows, nnz, ptrs, col, val, x, y, skip, st);
        // rows of up to ~26.9 entries on average, 4% slack (27-point stencils:
        // 855-entry mean blocks): 896-entry stages fit 20 warps per SM, not 16
        // (27-point 200^3: 0.441 -> 0.411 ms, tools/merge_probe.py rowblock)
        if (32.0 * double(nnz) / double(nrows) * 1.04 <= 896.0)
            return launch_csr_rowblock<CsrRbCfg<20, 1, 896>>(nrows, nnz, ptrs, col, val, x, y, skip, st);
        return launch_csr_rowblock<CsrRbCfg<16, 1, 1024>>(nrows, nnz, ptrs, col, val, x, y, skip, st);
    }
    if (strategy == WK_CSR_STREAM) {
        WK_REQUIRE(first != nullptr && partials != nullptr && tickets != nullptr, WK_ERR_INVALID,
                   "csr stream strategy needs a plan (wk_csr_plan_build)");
        const int64_t nchunks = csr_stream_chunks(nnz);
        // 8 warps, one stage each, <= 80 registers: three CTAs per SM (24
        // warps); 16 warps x 2 stages left one CTA per SM (94 registers,
        // 200 KB): R-MAT 24 4.82 -> 2.29 ms, 27-point 0.995 -> 0.784 ms
        // (tools/merge_probe.py stream; 64-register caps spill)
        return launch_csr_tma<CsrTmaCfg<8, 1, 3>>(nrows, nnz, nchunks, ptrs, col, val, x, y, first, partials, tickets,
                                                skip, st);
    }
    WK_REQUIRE(strategy == WK_CSR_SUBWARP, WK_ERR_INVALID, "unknown CSR strategy %d", strategy);
    int T = subwarp;
    if (T <= 0) {
        // auto: the largest power of two <= the mean row length, clamped to
        // [1, 32] (rounding up left most lanes of a short row idle: 27-point
        // rows at T = 32 take 0.86 ms vs 0.69 at T = 16; 5-point rows 32 vs
        // 25 us at T = 8 vs 4)
        const int64_t avg = nnz / (nrows > 0 ? nrows : 1);
        T = 1;
        while (2 * T <= avg && T < 32) T <<= 1;
    }
    const int64_t tiles_per_block = kSpmvThreads / T;
    int64_t blocks = ceil_div(nrows, tiles_per_block);
    const int64_t cap = int64_t(sm_count()) * 16;
    if (blocks > cap) blocks = cap;
    switch (T) {
#define WK_SW(N) \
    case N: csr_subwarp_kernel<N><<<(unsigned)blocks, kSpmvThreads, 0, st>>>(nrows, ptrs, col, val, x, y, skip); break;
        WK_SW(1) WK_SW(2) WK_SW(4) WK_SW(8) WK_SW(16) WK_SW(32)
#undef WK_SW
        default:
            WK_REQUIRE(false, WK_ERR_INVALID, "csr subwarp size must be a power of two <= 32, got %d", T);
    }
    WK_LAUNCH_CHECK();
    return 0;
}

// COO (kernels.py:209-264 semantics): seg8 warp ranges of 2048 sorted
// entries, warp segmented scans, atomics for the two rows a range can share
// with its neighbours (segwarp.cuh).
int launch_coo(int64_t nrows, int64_t nnz, const int* row, const int* col, const double* val, const double* x,
               double* y, int accumulate, const int* skip, cudaStream_t st) {
    if (nrows == 0) return 0;
    if (!accumulate) {
        // skip-aware zero fill is not needed: a skipped SpMV leaves y untouched
        // only in the solver loops, which never use COO with accumulate == 0
        // behind a skip flag (they call wk_spmv with the full operator).
        WK_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * size_t(nrows), st));
    }
    if (nnz == 0) return 0;
    return launch_seg8(false, nnz, accumulate, row, col, val, x, y, skip, st);
}

}  // namespace wk

// ============================ C ABI ==========================================
using namespace wk;

extern "C" {

int wk_spmv_sellp_f64(int64_t nrows, int64_t ncols, int64_t slice_size, const int64_t* slice_sets,
                      const int32_t* col_idx, const double* values, const int32_t* row_lengths, const double* x,
                      double* y, wk_stream_t stream) {
    clear_error();
    WK_REQUIRE(slice_size > 0 && (slice_size & (slice_size - 1)) == 0, WK_ERR_SLICE,
               "slice_size must be a positive power of two, got %lld", (long long)slice_size);
    return launch_sellp(nrows, ncols, slice_size, slice_sets, col_idx, values, row_lengths, x, y, nullptr,
                        as_stream(stream));
}

int wk_spmv_ell_f64(int64_t nrows, int64_t ncols, int64_t width, int64_t stride, const int32_t* col_idx,
                    const double* values, const int32_t* row_lengths, const double* x, double* y,
                    wk_stream_t stream) {
    clear_error();
    WK_REQUIRE(stride >= nrows, WK_ERR_INVALID, "ELL stride %lld < nrows %lld", (long long)stride,
               (long long)nrows);
    return launch_ell(nrows, ncols, width, stride, col_idx, values, row_lengths, x, y, nullptr, as_stream(stream));
}

int64_t wk_csr_plan_chunks(int64_t nnz) { return csr_stream_chunks(nnz); }

int64_t wk_csr_plan_bytes(int64_t nnz) {
    const int64_t c = csr_stream_chunks(nnz);
    // first[c+1] int32 (padded to 16 B) | item descriptors[c] int4 | partials[2c] f64 | tickets[c] u32
    return csr_first_slots(c) * 4 + c * 16 + 2 * c * 8 + ceil_div(c * 4, 16) * 16;
}

int wk_csr_plan_build(int64_t nrows, int64_t nnz, const int32_t* row_ptrs, void* plan, wk_stream_t stream) {
    clear_error();
    const int64_t c = csr_stream_chunks(nnz);
    cudaStream_t st = as_stream(stream);
    WK_CUDA(cudaMemsetAsync(plan, 0, size_t(wk_csr_plan_bytes(nnz)), st));
    int* first = reinterpret_cast<int*>(plan);
    csr_plan_kernel<<<(unsigned)ceil_div(nrows + 1, 256), 256, 0, st>>>(nrows, nnz, c, row_ptrs, first);
    WK_LAUNCH_CHECK();
    csr_items_kernel<<<(unsigned)ceil_div(c, 256), 256, 0, st>>>(c, row_ptrs, first,
                                                                reinterpret_cast<int4*>(first + csr_first_slots(c)));
    WK_LAUNCH_CHECK();
    return 0;
}

int64_t wk_csr_merge_plan_bytes(int64_t nrows, int64_t nnz) { return csr_merge_plan_bytes(nrows, nnz); }

int64_t wk_csr_load_balance_plan_bytes(int64_t nrows, int64_t nnz) { return head_plan_bytes(nrows, nnz); }

int wk_csr_load_balance_plan_build(int64_t nrows, int64_t nnz, const int32_t* row_ptrs, void* plan,
                                   wk_stream_t stream) {
    clear_error();
    return build_head_plan(nrows, nnz, row_ptrs, plan, as_stream(stream));
}

int wk_csr_merge_plan_build(int64_t nrows, int64_t nnz, const int32_t* row_ptrs, void* plan, wk_stream_t stream) {
    clear_error();
    cudaStream_t st = as_stream(stream);
    WK_CUDA(cudaMemsetAsync(plan, 0, size_t(csr_merge_plan_bytes(nrows, nnz)), st));
    return build_csr_merge_plan(nrows, nnz, row_ptrs, plan, st);
}

static void csr_plan_views(void* plan, int64_t nnz, int** first, double** partials, unsigned** tickets) {
    const int64_t c = csr_stream_chunks(nnz);
    char* p = reinterpret_cast<char*>(plan);
    *first = reinterpret_cast<int*>(p);
    p += csr_first_slots(c) * 4 + c * 16;
    *partials = reinterpret_cast<double*>(p);
    p += 2 * c * 8;
    *tickets = reinterpret_cast<unsigned*>(p);
}

int wk_spmv_csr_f64(int64_t nrows, int64_t ncols, int64_t nnz, const int32_t* row_ptrs, const int32_t* col_idx,
                    const double* values, const double* x, double* y, int32_t strategy, int32_t subwarp_size,
                    void* plan, wk_stream_t stream) {
    clear_error();
    int* first = nullptr;
    double* partials = nullptr;
    unsigned* tickets = nullptr;
    if (plan != nullptr && strategy == WK_CSR_STREAM) csr_plan_views(plan, nnz, &first, &partials, &tickets);
    return launch_csr(nrows, ncols, nnz, row_ptrs, col_idx, values, x, y, strategy, subwarp_size, first, partials,
                      tickets, nullptr, as_stream(stream), (strategy == WK_CSR_MERGE || strategy == WK_CSR_LOAD_BALANCE) ? plan : nullptr);
}

int wk_spmv_coo_f64(int64_t nrows, int64_t ncols, int64_t nnz, const int32_t* row_idx, const int32_t* col_idx,
                    const double* values, const double* x, double* y, int32_t accumulate, wk_stream_t stream) {
    clear_error();
    (void)ncols;
    return launch_coo(nrows, nnz, row_idx, col_idx, values, x, y, accumulate, nullptr, as_stream(stream));
}

int wk_spmv_hybrid_f64(int64_t nrows, int64_t ncols, int64_t ell_width, int64_t ell_stride,
                       const int32_t* ell_col, const double* ell_val, const int32_t* ell_row_lengths,
                       int64_t coo_nnz, const int32_t* coo_row, const int32_t* coo_col, const double* coo_val,
                       const double* x, double* y, wk_stream_t stream) {
    clear_error();
    cudaStream_t st = as_stream(stream);
    int rc = launch_ell(nrows, ncols, ell_width, ell_stride, ell_col, ell_val, ell_row_lengths, x, y, nullptr, st);
    if (rc) return rc;
    return launch_coo(nrows, coo_nnz, coo_row, coo_col, coo_val, x, y, /*accumulate=*/1, nullptr, st);
}

int wk_spmv(const wk_matrix* A, const double* x, double* y, wk_stream_t stream) {
    clear_error();
    return wk_spmv_masked(A, x, y, nullptr, stream);
}

int wk_spmv_masked(const wk_matrix* A, const double* x, double* y, const int32_t* skip, wk_stream_t stream) {
    cudaStream_t st = as_stream(stream);
    switch (A->format) {
        case WK_FMT_CSR: {
            int* first = nullptr;
            double* partials = nullptr;
            unsigned* tickets = nullptr;
            if (A->plan != nullptr && A->csr_strategy == WK_CSR_STREAM)
                csr_plan_views(A->plan, A->nnz, &first, &partials, &tickets);
            return launch_csr(A->nrows, A->ncols, A->nnz, A->row_ptrs, A->col_idx, A->values, x, y,
                              A->csr_strategy, A->subwarp_size, first, partials, tickets, skip, st,
                              (A->csr_strategy == WK_CSR_MERGE || A->csr_strategy == WK_CSR_LOAD_BALANCE) ? A->plan : nullptr);
        }
        case WK_FMT_COO:
            WK_REQUIRE(skip == nullptr, WK_ERR_INVALID, "masked COO SpMV is not supported");
            return launch_coo(A->nrows, A->nnz, A->row_idx, A->col_idx, A->values, x, y, 0, nullptr, st);
        case WK_FMT_ELL:
            return launch_ell(A->nrows, A->ncols, A->width, A->stride, A->col_idx, A->values, A->row_lengths, x,
                              y, skip, st);
        case WK_FMT_SELLP:
            return launch_sellp(A->nrows, A->ncols, A->slice_size, A->slice_sets, A->col_idx, A->values,
                                A->row_lengths, x, y, skip, st, A->nnz);
        case WK_FMT_HYBRID: {
            int rc = launch_ell(A->nrows, A->ncols, A->width, A->stride, A->col_idx, A->values, A->row_lengths, x,
                                y, skip, st);
            if (rc) return rc;
            if (A->coo_nnz == 0) return 0;
            return launch_coo(A->nrows, A->coo_nnz, A->coo_row, A->coo_col, A->coo_val, x, y, /*accumulate=*/1,
                              skip, st);
        }
        default:
            WK_REQUIRE(false, WK_ERR_INVALID, "unknown matrix format %d", A->format);
    }
}

}  // extern "C"
