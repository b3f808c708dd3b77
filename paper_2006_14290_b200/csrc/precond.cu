// Jacobi-preconditioned CG and the subwarp-reduction microbenchmark
// (the adjacent solver step and the paper's Fig. 2
// experiment).
//
// * Diagonal extraction for every format (the operand of the reference
//   fixture's `apply_jacobi`, tests/golden/src/cuda/solver/preconditioner.cu:9-17:
//   z = r / diag). A missing diagonal entry gives 0.0 and z = +-inf, exactly as
//   the fixture's division.
// * PCG = the reference CG loop (kernels.py:283-331) with z = M^-1 r inserted:
//   rho = r.z drives alpha / beta, the history and the stopping test use
//   ||r|| (the reference's criterion), the true residual replaces r every 50th
//   iteration, breakdown on p.Ap <= 0. The z update, r.z and r.r are fused
//   into the x/r update pass (two reductions in one sweep); the 50-iteration
//   period is a CUDA graph replayed until the device `done` flag is set.
//   There is no reference PCG: the order is fixed by oracle/krylov_ref.py
//   (pcg_jacobi_solve), parity unpinned by the reference.
// * wk_reduce_microbench: the paper's coop-group subwarp reduction
//   (reduce_subwarp<size> on cg::thread_block_tile, kernels.py:341-364 /
//   reduce_driver.cu:5-23) against the legacy shared-memory tree
//   (residual_check.cu:17-32), clock64-timed on the device.
#include "cg_state.cuh"
#include "krylov_common.cuh"
#include "reduce.cuh"

namespace wk {

// ---- diagonal ------------------------------------------------------------------

__global__ void diag_csr_kernel(int64_t n, const int* __restrict__ ptrs, const int* __restrict__ col,
                                const double* __restrict__ val, double* __restrict__ d) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= n) return;
    double v = 0.0;
    for (int64_t k = ptrs[r]; k < ptrs[r + 1]; ++k)
        if (col[k] == r) {
            v = val[k];
            break;
        }
    d[r] = v;
}

// SELL-P / ELL: entry j of row r at base(r) + j * stride
__global__ void diag_sliced_kernel(int64_t n, int64_t ss, const int64_t* __restrict__ sets, int64_t stride,
                                   const int* __restrict__ lengths, const int* __restrict__ col,
                                   const double* __restrict__ val, double* __restrict__ d) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= n) return;
    int64_t base, step;
    if (sets != nullptr) {
        const int64_t s = r / ss;
        base = sets[s] * ss + (r - s * ss);
        step = ss;
    } else {
        base = r;
        step = stride;
    }
    double v = 0.0;
    for (int j = 0; j < lengths[r]; ++j)
        if (col[base + j * step] == r) {
            v = val[base + j * step];
            break;
        }
    d[r] = v;
}

__global__ void diag_coo_kernel(int64_t nnz, const int* __restrict__ row, const int* __restrict__ col,
                                const double* __restrict__ val, double* __restrict__ d) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k < nnz && row[k] == col[k]) d[row[k]] = val[k];
}

static int extract_diagonal(const wk_matrix* A, double* d, cudaStream_t st) {
    const int64_t n = A->nrows < A->ncols ? A->nrows : A->ncols;
    if (n == 0) return 0;
    const unsigned gb = (unsigned)ceil_div(n, 256);
    switch (A->format) {
        case WK_FMT_CSR:
            diag_csr_kernel<<<gb, 256, 0, st>>>(n, A->row_ptrs, A->col_idx, A->values, d);
            break;
        case WK_FMT_SELLP:
            diag_sliced_kernel<<<gb, 256, 0, st>>>(n, A->slice_size, A->slice_sets, 0, A->row_lengths, A->col_idx,
                                                  A->values, d);
            break;
        case WK_FMT_ELL:
        case WK_FMT_HYBRID:
            diag_sliced_kernel<<<gb, 256, 0, st>>>(n, 0, nullptr, A->stride, A->row_lengths, A->col_idx, A->values,
                                                  d);
            if (A->format == WK_FMT_HYBRID && A->coo_nnz > 0) {
                WK_LAUNCH_CHECK();
                diag_coo_kernel<<<(unsigned)ceil_div(A->coo_nnz, 256), 256, 0, st>>>(A->coo_nnz, A->coo_row,
                                                                                     A->coo_col, A->coo_val, d);
            }
            break;
        case WK_FMT_COO:
            WK_CUDA(cudaMemsetAsync(d, 0, sizeof(double) * size_t(n), st));
            if (A->nnz > 0)
                diag_coo_kernel<<<(unsigned)ceil_div(A->nnz, 256), 256, 0, st>>>(A->nnz, A->row_idx, A->col_idx,
                                                                                  A->values, d);
            break;
        default:
            WK_REQUIRE(false, WK_ERR_INVALID, "unknown matrix format %d", A->format);
    }
    WK_LAUNCH_CHECK();
    return 0;
}

// ---- Jacobi PCG ------------------------------------------------------------------

// hist / beta / rho / convergence from the fused (r.z, r.r) totals
__device__ __forceinline__ void pcg_beta_step(wk_cg_state* s, double* hist, double rz, double rr) {
    if (s->done) return;
    const double rn = sqrt(rr);
    hist[s->iteration] = rn;
    s->rr = rr;
    s->beta = rz / s->rho;
    s->rho = rz;
    s->done = !(s->iteration < s->max_iters && rn > s->threshold);
}

static int pcg_init(int64_t n, const double* b, const double* d, double* x, double* r, double* z, double* p,
                    wk_cg_state* s, double* hist, double tol, int64_t max_iters, void* ws, cudaStream_t st) {
    auto finish = [=] __device__(double rz, double bb) {
        const double bn = sqrt(bb);
        hist[0] = bn;
        s->rho = rz;
        s->rr = bb;
        s->threshold = tol * bn;
        s->max_iters = max_iters;
        s->alpha = 0.0;
        s->beta = 0.0;
        s->iteration = 0;
        s->breakdown = 0;
        s->done = !(bn != 0.0 && 0 < max_iters && bn > s->threshold);
    };
    if (n == 0) return launch_scalar([=] __device__() { finish(0.0, 0.0); }, st);
    return launch_map_reduce_n<2>(
        n,
        [=] __device__(int64_t i, double(&acc)[2]) {
            const double bi = b[i];
            const double zi = bi / d[i];
            x[i] = 0.0;
            r[i] = bi;
            z[i] = zi;
            p[i] = zi;
            acc[0] += __dmul_rn(bi, zi);
            acc[1] += __dmul_rn(bi, bi);
        },
        [=] __device__(double(&t)[2]) { finish(t[0], t[1]); }, ws, nullptr, st);
}

// x += alpha p; r -= alpha q (or, in a replacement iteration, x only);
// z = r / d; (r.z, r.r) -> beta step
static int pcg_update(int64_t n, const double* p, const double* q, const double* d, double* x, double* r, double* z,
                      wk_cg_state* s, double* hist, void* ws, cudaStream_t st) {
    return launch_map_reduce_n<2>(
        n,
        [=] __device__(int64_t i, double(&acc)[2]) {
            const double alpha = s->alpha;
            x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
            if (cg_replacing(s)) return;
            const double ri = __dadd_rn(r[i], -__dmul_rn(alpha, q[i]));
            const double zi = ri / d[i];
            r[i] = ri;
            z[i] = zi;
            acc[0] += __dmul_rn(ri, zi);
            acc[1] += __dmul_rn(ri, ri);
        },
        [=] __device__(double(&t)[2]) {
            if (!cg_replacing(s)) pcg_beta_step(s, hist, t[0], t[1]);
        },
        ws, &s->done, st);
}

// replacement iteration: r = b - A x (q holds A x), z = r / d
static int pcg_replace(int64_t n, const double* b, const double* q, const double* d, double* r, double* z,
                       wk_cg_state* s, double* hist, void* ws, cudaStream_t st) {
    return launch_map_reduce_n<2>(
        n,
        [=] __device__(int64_t i, double(&acc)[2]) {
            if (!cg_replacing(s)) return;
            const double ri = __dadd_rn(b[i], -q[i]);
            const double zi = ri / d[i];
            r[i] = ri;
            z[i] = zi;
            acc[0] += __dmul_rn(ri, zi);
            acc[1] += __dmul_rn(ri, ri);
        },
        [=] __device__(double(&t)[2]) {
            if (cg_replacing(s)) pcg_beta_step(s, hist, t[0], t[1]);
        },
        ws, &s->done, st);
}

// ---- reduction microbenchmark ------------------------------------------------------

// every lane of a 32-lane warp reduces (rank + 1) over its tile of `Size`
// lanes `loops` times with the butterfly (coop groups), or with the legacy
// shared-memory tree of the same width (__syncwarp between levels)
template <unsigned Size, bool kShared>
__global__ void reduce_microbench_kernel(int loops, double* __restrict__ out, long long* __restrict__ cycles) {
    auto tile = cg::tiled_partition<Size>(cg::this_thread_block());
    __shared__ double work[32];
    const double v = double(tile.thread_rank() + 1);
    double total = 0.0;
    const long long t0 = clock64();
    for (int l = 0; l < loops; ++l) {
        double x = v + 0.0 * double(l);  // loop-carried to keep every iteration
        if (kShared) {
            const unsigned base = threadIdx.x - tile.thread_rank();
            work[threadIdx.x] = x;
            __syncwarp();
            for (unsigned span = Size / 2; span > 0; span >>= 1) {
                if (tile.thread_rank() < span) work[threadIdx.x] += work[threadIdx.x + span];
                __syncwarp();
            }
            x = work[base];
            __syncwarp();
        } else {
            x = reduce_subwarp(tile, x);
        }
        total = x;
    }
    const long long t1 = clock64();
    out[threadIdx.x] = total;
    if (threadIdx.x == 0) *cycles = t1 - t0;
}

}  // namespace wk

using namespace wk;

extern "C" {

int wk_extract_diagonal(const wk_matrix* A, double* diag, wk_stream_t stream) {
    clear_error();
    return extract_diagonal(A, diag, as_stream(stream));
}

int64_t wk_pcg_workspace_bytes(int64_t n) {
    return 256 + red_ws_bytes() + 256 + 4 * (ceil_div(n * 8, 256) * 256) + 256;
}

int wk_pcg_jacobi_solve(const wk_matrix* A, const double* diag, const double* b, double tol, int64_t max_iters,
                        double* x, double* hist, int64_t* iterations, void* workspace, wk_stream_t stream) {
    clear_error();
    WK_TRY(check_square(A));
    WK_REQUIRE(tol > 0, WK_ERR_INVALID, "tol must be positive");
    const int64_t n = A->nrows;
    Carver cv{reinterpret_cast<char*>(workspace)};
    wk_cg_state* s = cv.take<wk_cg_state>(1);
    void* red = cv.take<char>(red_ws_bytes());
    double* r = cv.take<double>(n);
    double* p = cv.take<double>(n);
    double* q = cv.take<double>(n);
    double* z = cv.take<double>(n);
    cudaStream_t user = as_stream(stream);
    GraphRunner g;
    WK_CUDA(cudaStreamCreateWithFlags(&g.cs, cudaStreamNonBlocking));
    cudaEvent_t ev;
    WK_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    WK_CUDA(cudaEventRecord(ev, user));
    WK_CUDA(cudaStreamWaitEvent(g.cs, ev, 0));
    cudaStream_t st = g.cs;
    WK_CUDA(cudaMemsetAsync(red, 0, size_t(red_ws_bytes()), st));
    WK_TRY(pcg_init(n, b, diag, x, r, z, p, s, hist, tol, max_iters, red, st));
    int rc = capture(g, [&](cudaStream_t cs) -> int {
        for (int i = 0; i < kReplaceEvery; ++i) {
            // q = A p, p.q and the alpha step (shared with CG: alpha = rho / p.q)
            WK_TRY(wk_spmv_masked(A, p, q, &s->done, cs));
            WK_TRY(launch_map_reduce(
                n, [=] __device__(int64_t k) { return __dmul_rn(p[k], q[k]); },
                [=] __device__(double t) {
                    s->pq = t;
                    cg_alpha_step(s);
                },
                red, &s->done, cs));
            WK_TRY(pcg_update(n, p, q, diag, x, r, z, s, hist, red, cs));
            if (i == kReplaceEvery - 1) {
                WK_TRY(wk_spmv_masked(A, x, q, &s->done, cs));
                WK_TRY(pcg_replace(n, b, q, diag, r, z, s, hist, red, cs));
            }
            // p = z + beta p
            WK_TRY(launch_masked_map(
                n, [=] __device__(int64_t k) { p[k] = __dadd_rn(z[k], __dmul_rn(s->beta, p[k])); }, &s->done, cs));
        }
        return 0;
    });
    if (rc) {
        cudaEventDestroy(ev);
        return rc;
    }
    wk_cg_state h{};
    for (;;) {
        WK_CUDA(cudaMemcpyAsync(&h, s, sizeof(h), cudaMemcpyDeviceToHost, st));
        WK_CUDA(cudaStreamSynchronize(st));
        if (h.done) break;
        WK_CUDA(cudaGraphLaunch(g.exec, st));
    }
    WK_CUDA(cudaEventRecord(ev, st));
    WK_CUDA(cudaStreamWaitEvent(user, ev, 0));
    cudaEventDestroy(ev);
    *iterations = h.iteration;
    if (h.breakdown) {
        set_error("p.Ap <= 0 at iteration %lld; system is not SPD", (long long)h.iteration);
        return WK_ERR_BREAKDOWN;
    }
    return 0;
}

int wk_reduce_microbench(int32_t size, int32_t inner_loops, int32_t shared_memory, double* out,
                         long long* cycles, wk_stream_t stream) {
    clear_error();
    cudaStream_t st = as_stream(stream);
#define WK_RB(N)                                                                                   \
    case N:                                                                                        \
        if (shared_memory)                                                                         \
            reduce_microbench_kernel<N, true><<<1, 32, 0, st>>>(inner_loops, out, cycles);        \
        else                                                                                       \
            reduce_microbench_kernel<N, false><<<1, 32, 0, st>>>(inner_loops, out, cycles);       \
        break;
    switch (size) {
        WK_RB(1) WK_RB(2) WK_RB(4) WK_RB(8) WK_RB(16) WK_RB(32)
        default:
            WK_REQUIRE(false, WK_ERR_INVALID, "subwarp size must be a power of two <= 32, got %d", size);
    }
#undef WK_RB
    WK_LAUNCH_CHECK();
    return 0;
}

}  // extern "C"
