// Krylov solvers with all scalar control on the device.
//
// CG follows the reference statement for statement (warpkit/kernels.py:283-331):
//   q = A p ; pq = p.q ; breakdown if pq <= 0 ; alpha = rho/pq ; x = x + alpha p ;
//   iteration += 1 ; every 50th iteration r = b - A x else r = r - alpha q ;
//   rho' = r.r ; hist += sqrt(rho') ; beta = rho'/rho ; p = r + beta p ; rho = rho'
//   loop while iteration < max_iters and hist[-1] > tol*||b||.
// Vector updates are separately rounded (-fmad=false, __dmul_rn/__dadd_rn), so
// the only difference from the reference is the dot-product summation order.
//
// Every vector kernel is "masked": it returns immediately while the device
// flag `done` is set, so a fixed CUDA graph of 50 iterations (one residual
// replacement period) can be replayed until convergence without per-iteration
// host synchronisation. Scalar steps run in the epilogue of the reduction
// that produces their input (last-arriving block, single GPU) or as 1-thread
// kernels after the caller's all-reduce (row-block distributed path).
//
// BiCGSTAB and GMRES(m) have no reference; they follow the update order of
// oracle/krylov_ref.py (van der Vorst BiCGSTAB; restarted GMRES with classical
// Gram-Schmidt via batched dots and Givens rotations on one device thread).
#include <vector>

#include "cg_state.cuh"
#include "reduce.cuh"

namespace wk {


template <typename F>
__global__ void __launch_bounds__(256) masked_map_kernel(int64_t n, F f, const int* __restrict__ skip) {
    if (skip != nullptr && *skip) return;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) f(i);
}

template <typename F>
static int launch_masked_map(int64_t n, F f, const int* skip, cudaStream_t st) {
    if (n == 0) return 0;
    int64_t blocks = ceil_div(n, 256);
    const int64_t cap = int64_t(sm_count()) * 16;
    if (blocks > cap) blocks = cap;
    masked_map_kernel<<<(unsigned)blocks, 256, 0, st>>>(n, f, skip);
    WK_LAUNCH_CHECK();
    return 0;
}

template <typename F>
__global__ void scalar_kernel(F f) {
    f();
}

template <typename F>
static int launch_scalar(F f, cudaStream_t st) {
    scalar_kernel<<<1, 1, 0, st>>>(f);
    WK_LAUNCH_CHECK();
    return 0;
}

// ---- CG building blocks -------------------------------------------------------

static int cg_init_local(int64_t n, const double* b, double* x, double* r, double* p, wk_cg_state* s, void* ws,
                         cudaStream_t st) {
    if (n == 0) {
        return launch_scalar([=] __device__() {
            s->rho = 0.0;
            s->iteration = 0;
            s->done = 0;
            s->breakdown = 0;
        }, st);
    }
    return launch_map_reduce(
        n,
        [=] __device__(int64_t i) {
            const double bi = b[i];
            x[i] = 0.0;
            r[i] = bi;
            p[i] = bi;
            return __dmul_rn(bi, bi);
        },
        [=] __device__(double t) {
            s->rho = t;
            s->iteration = 0;
            s->done = 0;
            s->breakdown = 0;
        },
        ws, nullptr, st);
}

static int cg_init_finish(wk_cg_state* s, double tol, int64_t max_iters, double* hist, cudaStream_t st) {
    return launch_scalar([=] __device__() {
        const double bn = sqrt(s->rho);  // np.linalg.norm(b) == sqrt(b.b)
        hist[0] = bn;
        s->threshold = tol * bn;
        s->max_iters = max_iters;
        s->alpha = 0.0;
        s->beta = 0.0;
        s->done = !(bn != 0.0 && 0 < max_iters && bn > s->threshold);
    }, st);
}

static int cg_dot_pq(int64_t n, const double* p, const double* q, wk_cg_state* s, void* ws, bool finalize,
                     cudaStream_t st) {
    return launch_map_reduce(
        n, [=] __device__(int64_t i) { return __dmul_rn(__ldcs(p + i), __ldcs(q + i)); },
        [=] __device__(double t) {
            s->pq = t;
            if (finalize) cg_alpha_step(s);
        },
        ws, &s->done, st);
}

// q = A p and state->pq = p.q: fused into the SELL-P(64) kernel when
// possible, else SpMV then a separate reduction.
static int cg_spmv_dot(const wk_matrix* A, int64_t n, const double* p, double* q, wk_cg_state* s, void* ws,
                       bool finalize, cudaStream_t st) {
    const int rc = spmv_dot_fused(A, p, q, s, ws, finalize ? 1 : 0, st);
    if (rc != 1) return rc;
    WK_TRY(wk_spmv_masked(A, p, q, &s->done, st));
    if (n == 0)
        return launch_scalar([=] __device__() {
            if (!s->done) {
                s->pq = 0.0;
                if (finalize) cg_alpha_step(s);
            }
        }, st);
    return cg_dot_pq(n, p, q, s, ws, finalize, st);
}

// Vectorised CG vector updates (double2, two independent pairs in flight per
// thread, restrict-qualified so loads are issued ahead of the stores). Same
// arithmetic as the scalar lambdas below (and as kernels.py:320-329).
static bool vec_ok(const void* a, const void* b, const void* c, const void* d) {
    auto al = [](const void* v) { return (reinterpret_cast<uintptr_t>(v) & 15) == 0; };
    return al(a) && al(b) && al(c) && al(d);
}

static int vec_grid(int64_t n) {
    int64_t g = ceil_div(ceil_div(n, 2), 256 * 2);
    const int64_t cap = int64_t(sm_count()) * 8;
    if (g > cap) g = cap;
    if (g > kRedMaxBlocks) g = kRedMaxBlocks;
    return int(g < 1 ? 1 : g);
}

// kAlphaIn: the alpha step (kernels.py:316-321) is evaluated here from the
// all-reduced p.Ap (distributed path) instead of by a separate 1-thread kernel.
template <bool kAlphaIn>
__global__ void __launch_bounds__(256)
cg_update_xr_vec(int64_t n, const double* __restrict__ p, const double* __restrict__ q, double* __restrict__ x,
                 double* __restrict__ r, wk_cg_state* s, double* hist, RedWorkspace ws, int finalize) {
    if (s->done) return;
    double alpha;
    bool repl, brk = false;
    int64_t it_new = 0;
    if (kAlphaIn) {
        const double pq = s->pq;
        it_new = s->iteration + 1;
        brk = pq <= 0.0;  // kernels.py:317 (NaN falls through)
        alpha = s->rho / pq;
        repl = it_new % kReplaceEvery == 0;
    } else {
        alpha = s->alpha;
        repl = cg_replacing(s);
    }
    const int64_t n_eff = brk ? 0 : n;
    const int64_t np = n >> 1, T = int64_t(gridDim.x) * 256;
    const double2* p2 = reinterpret_cast<const double2*>(p);
    const double2* q2 = reinterpret_cast<const double2*>(q);
    double2* x2 = reinterpret_cast<double2*>(x);
    double2* r2 = reinterpret_cast<double2*>(r);
    double acc = 0.0;
    const int64_t np_eff = n_eff >> 1;
    for (int64_t k = int64_t(blockIdx.x) * 256 + threadIdx.x; k < np_eff; k += 2 * T) {
        const int64_t k1 = k + T;
        const bool h1 = k1 < np;
        double2 pa = __ldcs(p2 + k), xa = __ldcs(x2 + k), pb{0, 0}, xb{0, 0}, qa{0, 0}, ra{0, 0}, qb{0, 0}, rb{0, 0};
        if (h1) {
            pb = __ldcs(p2 + k1);
            xb = __ldcs(x2 + k1);
        }
        if (!repl) {
            qa = __ldcs(q2 + k);
            ra = __ldcs(r2 + k);
            if (h1) {
                qb = __ldcs(q2 + k1);
                rb = __ldcs(r2 + k1);
            }
        }
        xa.x = __dadd_rn(xa.x, __dmul_rn(alpha, pa.x));
        xa.y = __dadd_rn(xa.y, __dmul_rn(alpha, pa.y));
        __stcs(x2 + k, xa);
        if (h1) {
            xb.x = __dadd_rn(xb.x, __dmul_rn(alpha, pb.x));
            xb.y = __dadd_rn(xb.y, __dmul_rn(alpha, pb.y));
            __stcs(x2 + k1, xb);
        }
        if (!repl) {
            ra.x = __dadd_rn(ra.x, -__dmul_rn(alpha, qa.x));
            ra.y = __dadd_rn(ra.y, -__dmul_rn(alpha, qa.y));
            r2[k] = ra;
            acc += __dmul_rn(ra.x, ra.x);
            acc += __dmul_rn(ra.y, ra.y);
            if (h1) {
                rb.x = __dadd_rn(rb.x, -__dmul_rn(alpha, qb.x));
                rb.y = __dadd_rn(rb.y, -__dmul_rn(alpha, qb.y));
                r2[k1] = rb;
                acc += __dmul_rn(rb.x, rb.x);
                acc += __dmul_rn(rb.y, rb.y);
            }
        }
    }
    if ((n_eff & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const int64_t i = n - 1;
        x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
        if (!repl) {
            r[i] = __dadd_rn(r[i], -__dmul_rn(alpha, q[i]));
            acc += __dmul_rn(r[i], r[i]);
        }
    }
    double total;
    if (grid_reduce_last(acc, ws, total) && threadIdx.x == 0) {
        if (kAlphaIn) {
            s->iteration = it_new;
            if (brk) {
                s->breakdown = 1;
                s->done = 1;
                return;
            }
            s->alpha = alpha;
        }
        if (!repl) {
            s->rr = total;
            if (finalize) cg_beta_step(s, hist);
        }
    }
}

// kBetaIn: beta = r.r / rho is evaluated here from the all-reduced r.r and the
// last block performs the beta step (history, rho, convergence flag).
template <bool kBetaIn>
__global__ void __launch_bounds__(256)
cg_update_p_vec(int64_t n, const double* __restrict__ r, double* __restrict__ p, wk_cg_state* s, double* hist,
                RedWorkspace ws) {
    if (s->done) return;
    const double beta = kBetaIn ? s->rr / s->rho : s->beta;
    const int64_t np = n >> 1, T = int64_t(gridDim.x) * 256;
    const double2* r2 = reinterpret_cast<const double2*>(r);
    double2* p2 = reinterpret_cast<double2*>(p);
    for (int64_t k = int64_t(blockIdx.x) * 256 + threadIdx.x; k < np; k += 2 * T) {
        const int64_t k1 = k + T;
        const bool h1 = k1 < np;
        double2 ra = __ldcs(r2 + k), pa = p2[k], rb{0, 0}, pb{0, 0};
        if (h1) {
            rb = __ldcs(r2 + k1);
            pb = p2[k1];
        }
        pa.x = __dadd_rn(ra.x, __dmul_rn(beta, pa.x));
        pa.y = __dadd_rn(ra.y, __dmul_rn(beta, pa.y));
        p2[k] = pa;
        if (h1) {
            pb.x = __dadd_rn(rb.x, __dmul_rn(beta, pb.x));
            pb.y = __dadd_rn(rb.y, __dmul_rn(beta, pb.y));
            p2[k1] = pb;
        }
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) p[n - 1] = __dadd_rn(r[n - 1], __dmul_rn(beta, p[n - 1]));
    if (kBetaIn) {
        double total;
        if (grid_reduce_last(0.0, ws, total) && threadIdx.x == 0) cg_beta_step(s, hist);
    }
}

static int cg_update_xr(int64_t n, const double* p, const double* q, double* x, double* r, wk_cg_state* s,
                        double* hist, void* ws, bool finalize, cudaStream_t st) {
    if (n > 0 && vec_ok(p, q, x, r)) {
        cg_update_xr_vec<false><<<vec_grid(n), 256, 0, st>>>(n, p, q, x, r, s, hist, red_ws(ws), finalize ? 1 : 0);
        WK_LAUNCH_CHECK();
        return 0;
    }
    return launch_map_reduce(
        n,
        [=] __device__(int64_t i) {
            const double alpha = s->alpha;
            x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
            if (cg_replacing(s)) return 0.0;
            const double ri = __dadd_rn(r[i], -__dmul_rn(alpha, q[i]));
            r[i] = ri;
            return __dmul_rn(ri, ri);
        },
        [=] __device__(double t) {
            if (cg_replacing(s)) return;
            s->rr = t;
            if (finalize) cg_beta_step(s, hist);
        },
        ws, &s->done, st);
}

static int cg_replace_r(int64_t n, const double* b, const double* q, double* r, wk_cg_state* s, double* hist,
                        void* ws, bool finalize, cudaStream_t st) {
    return launch_map_reduce(
        n,
        [=] __device__(int64_t i) {
            if (!cg_replacing(s)) return 0.0;
            const double ri = __dadd_rn(b[i], -q[i]);
            r[i] = ri;
            return __dmul_rn(ri, ri);
        },
        [=] __device__(double t) {
            if (!cg_replacing(s)) return;
            s->rr = t;
            if (finalize) cg_beta_step(s, hist);
        },
        ws, &s->done, st);
}

static int cg_update_p(int64_t n, const double* r, double* p, const wk_cg_state* s, cudaStream_t st) {
    if (n > 0 && vec_ok(r, p, r, p)) {
        cg_update_p_vec<false><<<vec_grid(n), 256, 0, st>>>(n, r, p, const_cast<wk_cg_state*>(s), nullptr,
                                                          RedWorkspace{nullptr, nullptr});
        WK_LAUNCH_CHECK();
        return 0;
    }
    return launch_masked_map(
        n, [=] __device__(int64_t i) { p[i] = __dadd_rn(r[i], __dmul_rn(s->beta, p[i])); }, &s->done, st);
}

// ---- workspace carving --------------------------------------------------------

struct Carver {
    char* p;
    template <typename T>
    T* take(int64_t count) {
        T* r = reinterpret_cast<T*>(p);
        p += ceil_div(int64_t(sizeof(T)) * count, 256) * 256;
        return r;
    }
};

// Captures `body` (which enqueues work on `cs`) into a graph once, then the
// caller replays it. Work is done on an internal capture stream ordered after
// and before the caller's stream with events.
struct GraphRunner {
    cudaStream_t cs = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraph_t graph = nullptr;
    ~GraphRunner() {
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        if (cs) cudaStreamDestroy(cs);
    }
};

template <typename Body>
static int capture(GraphRunner& g, Body body) {
    WK_CUDA(cudaStreamBeginCapture(g.cs, cudaStreamCaptureModeThreadLocal));
    int rc = body(g.cs);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(g.cs, &graph);
    if (rc) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
    }
    WK_CUDA(e);
    g.graph = graph;
    WK_CUDA(cudaGraphInstantiate(&g.exec, graph, 0));
    return 0;
}

}  // namespace wk

using namespace wk;

extern "C" {

// ---------------- CG building blocks (distributed path) -------------------------

int wk_cg_init_local(int64_t n, const double* b, double* x, double* r, double* p, wk_cg_state* state,
                     void* workspace, wk_stream_t stream) {
    clear_error();
    return cg_init_local(n, b, x, r, p, state, workspace, as_stream(stream));
}

int wk_cg_init_finish(wk_cg_state* state, double tol, int64_t max_iters, double* hist, wk_stream_t stream) {
    clear_error();
    return cg_init_finish(state, tol, max_iters, hist, as_stream(stream));
}

int wk_cg_dot_pq(int64_t n, const double* p, const double* q, wk_cg_state* state, void* workspace,
                 wk_stream_t stream) {
    clear_error();
    if (n == 0)
        return launch_scalar([=] __device__() { if (!state->done) state->pq = 0.0; }, as_stream(stream));
    return cg_dot_pq(n, p, q, state, workspace, false, as_stream(stream));
}

int wk_cg_spmv_dot(const wk_matrix* A, const double* p, double* q, wk_cg_state* state, void* workspace,
                   wk_stream_t stream) {
    clear_error();
    return cg_spmv_dot(A, A->nrows, p, q, state, workspace, false, as_stream(stream));
}

int wk_cg_step_alpha(wk_cg_state* state, wk_stream_t stream) {
    clear_error();
    return launch_scalar([=] __device__() { cg_alpha_step(state); }, as_stream(stream));
}

int wk_cg_update_xr(int64_t n, const double* p, const double* q, double* x, double* r, wk_cg_state* state,
                    void* workspace, wk_stream_t stream) {
    clear_error();
    if (n == 0)
        return launch_scalar([=] __device__() { if (!state->done && !cg_replacing(state)) state->rr = 0.0; },
                             as_stream(stream));
    return cg_update_xr(n, p, q, x, r, state, nullptr, workspace, false, as_stream(stream));
}

int wk_cg_replace_r(int64_t n, const double* b, const double* q, double* r, wk_cg_state* state, void* workspace,
                    wk_stream_t stream) {
    clear_error();
    if (n == 0)
        return launch_scalar([=] __device__() { if (!state->done && cg_replacing(state)) state->rr = 0.0; },
                             as_stream(stream));
    return cg_replace_r(n, b, q, r, state, nullptr, workspace, false, as_stream(stream));
}

int wk_cg_update_xr_alpha(int64_t n, const double* p, const double* q, double* x, double* r, wk_cg_state* state,
                          void* workspace, wk_stream_t stream) {
    clear_error();
    WK_REQUIRE(vec_ok(p, q, x, r), WK_ERR_INVALID, "wk_cg_update_xr_alpha needs 16-byte aligned vectors");
    cg_update_xr_vec<true><<<vec_grid(n > 0 ? n : 1), 256, 0, as_stream(stream)>>>(n, p, q, x, r, state, nullptr,
                                                                                  red_ws(workspace), 0);
    WK_LAUNCH_CHECK();
    return 0;
}

int wk_cg_update_p_beta(int64_t n, const double* r, double* p, wk_cg_state* state, double* hist, void* workspace,
                        wk_stream_t stream) {
    clear_error();
    WK_REQUIRE(vec_ok(r, p, r, p), WK_ERR_INVALID, "wk_cg_update_p_beta needs 16-byte aligned vectors");
    cg_update_p_vec<true><<<vec_grid(n > 0 ? n : 1), 256, 0, as_stream(stream)>>>(n, r, p, state, hist,
                                                                                 red_ws(workspace));
    WK_LAUNCH_CHECK();
    return 0;
}

int wk_cg_step_beta(wk_cg_state* state, double* hist, wk_stream_t stream) {
    clear_error();
    return launch_scalar([=] __device__() { cg_beta_step(state, hist); }, as_stream(stream));
}

int wk_cg_update_p(int64_t n, const double* r, double* p, const wk_cg_state* state, wk_stream_t stream) {
    clear_error();
    return cg_update_p(n, r, p, state, as_stream(stream));
}

// ---------------- single-GPU CG ---------------------------------------------------

int64_t wk_cg_workspace_bytes(int64_t n) {
    return 256 + red_ws_bytes() + 256 + 3 * (ceil_div(n * 8, 256) * 256) + 256;
}

static int check_square(const wk_matrix* A) {
    WK_REQUIRE(A->nrows == A->ncols, WK_ERR_DIMENSION, "solver needs a square matrix, got %lldx%lld",
               (long long)A->nrows, (long long)A->ncols);
    return 0;
}

int wk_cg_solve(const wk_matrix* A, const double* b, double tol, int64_t max_iters, double* x, double* hist,
                int64_t* iterations, void* workspace, wk_stream_t stream) {
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
    cudaStream_t user = as_stream(stream);
    GraphRunner g;
    WK_CUDA(cudaStreamCreateWithFlags(&g.cs, cudaStreamNonBlocking));
    cudaEvent_t ev;
    WK_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    WK_CUDA(cudaEventRecord(ev, user));
    WK_CUDA(cudaStreamWaitEvent(g.cs, ev, 0));
    cudaStream_t st = g.cs;
    WK_CUDA(cudaMemsetAsync(red, 0, size_t(red_ws_bytes()), st));
    WK_TRY(cg_init_local(n, b, x, r, p, s, red, st));
    WK_TRY(cg_init_finish(s, tol, max_iters, hist, st));
    int rc = capture(g, [&](cudaStream_t cs) -> int {
        for (int i = 0; i < kReplaceEvery; ++i) {
            WK_TRY(cg_spmv_dot(A, n, p, q, s, red, true, cs));
            WK_TRY(cg_update_xr(n, p, q, x, r, s, hist, red, true, cs));
            if (i == kReplaceEvery - 1) {
                WK_TRY(wk_spmv_masked(A, x, q, &s->done, cs));
                WK_TRY(cg_replace_r(n, b, q, r, s, hist, red, true, cs));
            }
            WK_TRY(cg_update_p(n, r, p, s, cs));
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

}  // extern "C"

// ============================== BiCGSTAB ===========================================

namespace wk {

struct BicgState {
    double rho, rho_new, alpha, omega, beta, threshold;
    int64_t iteration, max_iters;
    int32_t done, breakdown, apply_half, pad;
};

}  // namespace wk

extern "C" {

int64_t wk_bicgstab_workspace_bytes(int64_t n) {
    return 256 + red_ws_bytes() + 256 + 6 * (ceil_div(n * 8, 256) * 256) + 256;
}

int wk_bicgstab_solve(const wk_matrix* A, const double* b, double tol, int64_t max_iters, double* x, double* hist,
                      int64_t* iterations, void* workspace, wk_stream_t stream) {
    clear_error();
    WK_TRY(check_square(A));
    WK_REQUIRE(tol > 0, WK_ERR_INVALID, "tol must be positive");
    const int64_t n = A->nrows;
    Carver cv{reinterpret_cast<char*>(workspace)};
    BicgState* s = cv.take<BicgState>(1);
    void* red = cv.take<char>(red_ws_bytes());
    double* r = cv.take<double>(n);
    double* rh = cv.take<double>(n);
    double* p = cv.take<double>(n);
    double* v = cv.take<double>(n);
    double* sv = cv.take<double>(n);
    double* t = cv.take<double>(n);
    cudaStream_t user = as_stream(stream);
    GraphRunner g;
    WK_CUDA(cudaStreamCreateWithFlags(&g.cs, cudaStreamNonBlocking));
    cudaEvent_t ev;
    WK_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    WK_CUDA(cudaEventRecord(ev, user));
    WK_CUDA(cudaStreamWaitEvent(g.cs, ev, 0));
    cudaStream_t st = g.cs;
    WK_CUDA(cudaMemsetAsync(red, 0, size_t(red_ws_bytes()), st));
    // x = 0, r = rh = b, p = v = 0, ||b||
    WK_TRY(launch_map_reduce(
        n,
        [=] __device__(int64_t i) {
            const double bi = b[i];
            x[i] = 0.0;
            r[i] = bi;
            rh[i] = bi;
            p[i] = 0.0;
            v[i] = 0.0;
            return __dmul_rn(bi, bi);
        },
        [=] __device__(double tt) {
            const double bn = sqrt(tt);
            hist[0] = bn;
            s->rho = s->alpha = s->omega = 1.0;
            s->threshold = tol * bn;
            s->iteration = 0;
            s->max_iters = max_iters;
            s->breakdown = 0;
            s->apply_half = 0;
            s->done = !(bn != 0.0 && 0 < max_iters && bn > s->threshold);
        },
        red, nullptr, st));
    if (n == 0) WK_TRY(launch_scalar([=] __device__() { hist[0] = 0.0; s->done = 1; s->iteration = 0; s->breakdown = 0; }, st));
    const int* done = &s->done;
    const int kChunk = 10;
    int rc = capture(g, [&](cudaStream_t cs) -> int {
        for (int i = 0; i < kChunk; ++i) {
            // rho_new = rh.r ; beta
            WK_TRY(launch_map_reduce(
                n, [=] __device__(int64_t k) { return __dmul_rn(rh[k], r[k]); },
                [=] __device__(double tt) {
                    s->rho_new = tt;
                    if (tt == 0.0) {
                        s->breakdown = 1;
                        s->done = 1;
                        s->iteration += 1;
                        return;
                    }
                    s->beta = __dmul_rn(s->rho_new / s->rho, s->alpha / s->omega);
                },
                red, done, cs));
            // p = r + beta (p - omega v)
            WK_TRY(launch_masked_map(
                n,
                [=] __device__(int64_t k) {
                    p[k] = __dadd_rn(r[k], __dmul_rn(s->beta, __dadd_rn(p[k], -__dmul_rn(s->omega, v[k]))));
                },
                done, cs));
            WK_TRY(wk_spmv_masked(A, p, v, done, cs));
            // alpha = rho_new / (rh.v)
            WK_TRY(launch_map_reduce(
                n, [=] __device__(int64_t k) { return __dmul_rn(rh[k], v[k]); },
                [=] __device__(double tt) {
                    if (tt == 0.0) {
                        s->breakdown = 1;
                        s->done = 1;
                        s->iteration += 1;
                        return;
                    }
                    s->alpha = s->rho_new / tt;
                },
                red, done, cs));
            // s = r - alpha v ; ||s||
            WK_TRY(launch_map_reduce(
                n,
                [=] __device__(int64_t k) {
                    const double sk = __dadd_rn(r[k], -__dmul_rn(s->alpha, v[k]));
                    sv[k] = sk;
                    return __dmul_rn(sk, sk);
                },
                [=] __device__(double tt) {
                    s->iteration += 1;
                    const double sn = sqrt(tt);
                    if (sn <= s->threshold) {
                        hist[s->iteration] = sn;
                        s->apply_half = 1;
                        s->done = 1;
                    }
                },
                red, done, cs));
            // half-step convergence: x = x + alpha p
            WK_TRY(launch_map_reduce(
                n,
                [=] __device__(int64_t k) {
                    if (!s->apply_half) return 0.0;
                    x[k] = __dadd_rn(x[k], __dmul_rn(s->alpha, p[k]));
                    return 0.0;
                },
                [=] __device__(double) { s->apply_half = 0; }, red, nullptr, cs));
            WK_TRY(wk_spmv_masked(A, sv, t, done, cs));
            // omega = (t.s)/(t.t)
            WK_TRY(launch_map_reduce_n<2>(
                n,
                [=] __device__(int64_t k, double(&acc)[2]) {
                    const double tk = t[k];
                    acc[0] += __dmul_rn(tk, tk);
                    acc[1] += __dmul_rn(tk, sv[k]);
                },
                [=] __device__(double(&tot)[2]) {
                    if (tot[0] == 0.0) {
                        s->breakdown = 1;
                        s->done = 1;
                        return;
                    }
                    s->omega = tot[1] / tot[0];
                },
                red, done, cs));
            // x = x + alpha p + omega s ; r = s - omega t ; ||r||
            WK_TRY(launch_map_reduce(
                n,
                [=] __device__(int64_t k) {
                    x[k] = __dadd_rn(__dadd_rn(x[k], __dmul_rn(s->alpha, p[k])), __dmul_rn(s->omega, sv[k]));
                    const double rk = __dadd_rn(sv[k], -__dmul_rn(s->omega, t[k]));
                    r[k] = rk;
                    return __dmul_rn(rk, rk);
                },
                [=] __device__(double tt) {
                    const double rn = sqrt(tt);
                    hist[s->iteration] = rn;
                    s->rho = s->rho_new;
                    s->done = !(s->iteration < s->max_iters && rn > s->threshold);
                },
                red, done, cs));
        }
        return 0;
    });
    if (rc) {
        cudaEventDestroy(ev);
        return rc;
    }
    BicgState h{};
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
        set_error("BiCGSTAB breakdown at iteration %lld", (long long)h.iteration);
        return WK_ERR_BREAKDOWN;
    }
    return 0;
}

}  // extern "C"

// =============================== GMRES(m) ==========================================

namespace wk {

struct GmresState {
    double beta, threshold, hn;
    int64_t iteration, max_iters;
    int32_t done, cycle_done, j_done, pad;
};

}  // namespace wk

extern "C" {

int64_t wk_gmres_workspace_bytes(int64_t n, int32_t restart) {
    const int64_t m = restart;
    const int64_t vec = ceil_div(n * 8, 256) * 256;
    return 256 + red_ws_bytes() + 256 + (m + 1) * vec + 2 * vec + ceil_div((m + 1) * m * 8 + 4 * (m + 1) * 8, 256) * 256 +
           256;
}

int wk_gmres_solve(const wk_matrix* A, const double* b, double tol, int64_t max_iters, int32_t restart, double* x,
                   double* hist, int64_t* iterations, void* workspace, wk_stream_t stream) {
    clear_error();
    WK_TRY(check_square(A));
    WK_REQUIRE(tol > 0, WK_ERR_INVALID, "tol must be positive");
    WK_REQUIRE(restart >= 1 && restart <= kRedMaxVec - 1, WK_ERR_INVALID, "restart must be in [1, %d]",
               kRedMaxVec - 1);
    const int64_t n = A->nrows;
    const int m = restart;
    Carver cv{reinterpret_cast<char*>(workspace)};
    GmresState* s = cv.take<GmresState>(1);
    void* red = cv.take<char>(red_ws_bytes());
    const int64_t ld = ceil_div(n * 8, 256) * 256 / 8;
    double* V = cv.take<double>(ld * (m + 1));
    double* w = cv.take<double>(n);
    double* rv = cv.take<double>(n);
    double* small = cv.take<double>((m + 1) * m + 4 * (m + 1));
    double* H = small;                 // (m+1) x m, column-major H[i + j*(m+1)]
    double* cs_ = H + (m + 1) * m;     // m
    double* sn_ = cs_ + (m + 1);       // m
    double* g = sn_ + (m + 1);         // m + 1
    double* y = g + (m + 1);           // m
    cudaStream_t user = as_stream(stream);
    GraphRunner gr;
    WK_CUDA(cudaStreamCreateWithFlags(&gr.cs, cudaStreamNonBlocking));
    cudaEvent_t ev;
    WK_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    WK_CUDA(cudaEventRecord(ev, user));
    WK_CUDA(cudaStreamWaitEvent(gr.cs, ev, 0));
    cudaStream_t st = gr.cs;
    WK_CUDA(cudaMemsetAsync(red, 0, size_t(red_ws_bytes()), st));
    // x = 0, r = b, beta = ||b||
    WK_TRY(launch_map_reduce(
        n,
        [=] __device__(int64_t i) {
            x[i] = 0.0;
            rv[i] = b[i];
            return __dmul_rn(b[i], b[i]);
        },
        [=] __device__(double tt) {
            const double bn = sqrt(tt);
            hist[0] = bn;
            s->beta = bn;
            s->threshold = tol * bn;
            s->iteration = 0;
            s->max_iters = max_iters;
            s->done = !(bn != 0.0 && 0 < max_iters && bn > s->threshold);
            s->cycle_done = s->done;
        },
        red, nullptr, st));
    if (n == 0) WK_TRY(launch_scalar([=] __device__() { hist[0] = 0.0; s->done = 1; s->cycle_done = 1; s->iteration = 0; }, st));
    const int* done = &s->done;
    const int* cdone = &s->cycle_done;
    int rc = capture(gr, [&](cudaStream_t cs) -> int {
        // cycle start: V0 = r / beta ; g = beta e1
        WK_TRY(launch_masked_map(n, [=] __device__(int64_t i) { V[i] = rv[i] / s->beta; }, done, cs));
        WK_TRY(launch_scalar([=] __device__() {
            if (s->done) return;
            for (int i = 0; i <= m; ++i) g[i] = 0.0;
            g[0] = s->beta;
            s->j_done = 0;
            s->cycle_done = 0;
        }, cs));
        for (int j = 0; j < m; ++j) {
            double* Vj = V + int64_t(j) * ld;
            double* Hj = H + int64_t(j) * (m + 1);
            WK_TRY(wk_spmv_masked(A, Vj, w, cdone, cs));
            // h_i = V_i . w (batched classical Gram-Schmidt)
            {
                // multidot writes its results unconditionally; mask by running it
                // into H only while the cycle is live (the kernel reads cdone)
                const int k = j + 1;
                auto f = [=] __device__(int64_t i, double(&acc)[kRedMaxVec]) {
                    const double wi = w[i];
#pragma unroll
                    for (int q = 0; q < kRedMaxVec; ++q)
                        if (q < k) acc[q] += __dmul_rn(V[int64_t(q) * ld + i], wi);
                };
                auto epi = [=] __device__(double(&tot)[kRedMaxVec]) {
                    for (int q = 0; q < k; ++q) Hj[q] = tot[q];
                };
                if (k <= 8) {
                    WK_TRY(launch_map_reduce_n<8>(
                        n, [=] __device__(int64_t i, double(&acc)[8]) {
                            const double wi = w[i];
#pragma unroll
                            for (int q = 0; q < 8; ++q)
                                if (q < k) acc[q] += __dmul_rn(V[int64_t(q) * ld + i], wi);
                        },
                        [=] __device__(double(&tot)[8]) { for (int q = 0; q < k; ++q) Hj[q] = tot[q]; }, red, cdone, cs));
                } else if (k <= 16) {
                    WK_TRY(launch_map_reduce_n<16>(
                        n, [=] __device__(int64_t i, double(&acc)[16]) {
                            const double wi = w[i];
#pragma unroll
                            for (int q = 0; q < 16; ++q)
                                if (q < k) acc[q] += __dmul_rn(V[int64_t(q) * ld + i], wi);
                        },
                        [=] __device__(double(&tot)[16]) { for (int q = 0; q < k; ++q) Hj[q] = tot[q]; }, red, cdone, cs));
                } else {
                    WK_TRY(launch_map_reduce_n<kRedMaxVec>(n, f, epi, red, cdone, cs));
                }
            }
            // w = w - sum_i h_i V_i (in i order) ; hn^2 = w.w
            WK_TRY(launch_map_reduce(
                n,
                [=] __device__(int64_t i) {
                    double wi = w[i];
                    for (int q = 0; q <= j; ++q) wi = __dadd_rn(wi, -__dmul_rn(Hj[q], V[int64_t(q) * ld + i]));
                    w[i] = wi;
                    return __dmul_rn(wi, wi);
                },
                [=] __device__(double tt) { s->hn = sqrt(tt); }, red, cdone, cs));
            // Givens on one thread (oracle/krylov_ref.py gmres_solve)
            WK_TRY(launch_scalar([=] __device__() {
                if (s->cycle_done) return;
                const double hn = s->hn;
                Hj[j + 1] = hn;
                for (int i = 0; i < j; ++i) {
                    const double a = Hj[i], c = Hj[i + 1];
                    Hj[i] = __dadd_rn(__dmul_rn(cs_[i], a), __dmul_rn(sn_[i], c));
                    Hj[i + 1] = __dadd_rn(-__dmul_rn(sn_[i], a), __dmul_rn(cs_[i], c));
                }
                const double a = Hj[j], c = Hj[j + 1];
                double cj = 1.0, sj = 0.0;
                if (c != 0.0) {
                    const double h = hypot(a, c);
                    cj = a / h;
                    sj = c / h;
                }
                cs_[j] = cj;
                sn_[j] = sj;
                Hj[j] = __dadd_rn(__dmul_rn(cj, Hj[j]), __dmul_rn(sj, Hj[j + 1]));
                Hj[j + 1] = 0.0;
                g[j + 1] = -__dmul_rn(sj, g[j]);
                g[j] = __dmul_rn(cj, g[j]);
                s->iteration += 1;
                s->j_done = j + 1;
                const double res = fabs(g[j + 1]);
                hist[s->iteration] = res;
                if (res <= s->threshold || s->iteration >= s->max_iters || hn == 0.0 || j + 1 == m) s->cycle_done = 1;
            }, cs));
            // V_{j+1} = w / hn (only when the cycle continues)
            if (j + 1 < m) {
                double* Vn = V + int64_t(j + 1) * ld;
                WK_TRY(launch_masked_map(n, [=] __device__(int64_t i) { Vn[i] = w[i] / s->hn; }, cdone, cs));
            }
        }
        // cycle end: y = H^-1 g ; x = x + sum y_i V_i ; r = b - A x ; beta = ||r||
        WK_TRY(launch_scalar([=] __device__() {
            if (s->done) return;
            const int jd = s->j_done;
            for (int i = jd - 1; i >= 0; --i) {
                double acc = g[i];
                for (int k = i + 1; k < jd; ++k) acc = __dadd_rn(acc, -__dmul_rn(H[i + k * (m + 1)], y[k]));
                y[i] = acc / H[i + i * (m + 1)];
            }
        }, cs));
        WK_TRY(launch_masked_map(
            n,
            [=] __device__(int64_t i) {
                const int jd = s->j_done;
                double xi = x[i];
                for (int q = 0; q < jd; ++q) xi = __dadd_rn(xi, __dmul_rn(y[q], V[int64_t(q) * ld + i]));
                x[i] = xi;
            },
            done, cs));
        WK_TRY(wk_spmv_masked(A, x, w, done, cs));
        WK_TRY(launch_map_reduce(
            n,
            [=] __device__(int64_t i) {
                const double ri = __dadd_rn(b[i], -w[i]);
                rv[i] = ri;
                return __dmul_rn(ri, ri);
            },
            [=] __device__(double tt) {
                const double bt = sqrt(tt);
                s->beta = bt;
                hist[s->iteration] = bt;
                s->done = !(s->iteration < s->max_iters && bt > s->threshold);
                s->cycle_done = s->done;
            },
            red, done, cs));
        return 0;
    });
    if (rc) {
        cudaEventDestroy(ev);
        return rc;
    }
    GmresState h{};
    for (;;) {
        WK_CUDA(cudaMemcpyAsync(&h, s, sizeof(h), cudaMemcpyDeviceToHost, st));
        WK_CUDA(cudaStreamSynchronize(st));
        if (h.done) break;
        WK_CUDA(cudaGraphLaunch(gr.exec, st));
    }
    WK_CUDA(cudaEventRecord(ev, st));
    WK_CUDA(cudaStreamWaitEvent(user, ev, 0));
    cudaEventDestroy(ev);
    *iterations = h.iteration;
    return 0;
}

}  // extern "C"
