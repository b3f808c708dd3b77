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
#include "krylov_common.cuh"
#include "reduce.cuh"

namespace wk {


// ---- CG building blocks -------------------------------------------------------

static int cg_init_local(int64_t n, const double* b, double* x, double* r, double* p, wk_cg_state* s, void* ws,
                         cudaStream_t st) {
    if (n == 0) {
        return launch_scalar([=] __device__() {
            s->rho = 0.0;
            s->iteration = 0;
            s->done = 0;
            s->breakdown = 0;
            s->xpend = 0;
            s->xdefer = 0;
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
            s->xpend = 0;
            s->xdefer = 0;
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
                     cudaStream_t st, PeerCtx* peer = nullptr) {
    return launch_map_reduce(
        n, [=] __device__(int64_t i) { return __dmul_rn(__ldcs(p + i), __ldcs(q + i)); },
        [=] __device__(double t) {
            if (peer != nullptr) {
                peer_push_scalar(peer, t);
                return;
            }
            s->pq = t;
            if (finalize) cg_alpha_step(s);
        },
        ws, &s->done, st);
}

// q = A p and state->pq = p.q: fused into the SELL-P(64) kernel when
// possible, else SpMV then a separate reduction.
__global__ void halo_wait_kernel(const PeerCtx* c, const PeerHalo* h, const int* skip) {
    if (*skip) return;
    halo_wait(c, h);
}

static int cg_spmv_dot(const wk_matrix* A, int64_t n, const double* p, double* q, wk_cg_state* s, void* ws,
                       bool finalize, cudaStream_t st, PeerCtx* peer = nullptr, const PeerHalo* halo = nullptr,
                       int rev = 0) {
    const int rc = spmv_dot_fused(A, p, q, s, ws, finalize ? 1 : 0, st, peer, halo, rev);
    if (rc != 1) return rc;
    if (halo != nullptr) {  // other formats: a separate wait before the SpMV
        halo_wait_kernel<<<1, 32, 0, st>>>(peer, halo, &s->done);
        WK_LAUNCH_CHECK();
    }
    WK_TRY(wk_spmv_masked(A, p, q, &s->done, st));
    if (n == 0)
        return launch_scalar([=] __device__() {
            if (!s->done) {
                if (peer != nullptr) {
                    peer_push_scalar(peer, 0.0);
                    return;
                }
                s->pq = 0.0;
                if (finalize) cg_alpha_step(s);
            }
        }, st);
    return cg_dot_pq(n, p, q, s, ws, finalize, st, peer);
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
                 double* __restrict__ r, wk_cg_state* s, double* hist, RedWorkspace ws, int finalize,
                 PeerCtx* peer, int rev = 0, int defer_x = 0) {
    if (s->done) return;
    double alpha;
    bool repl, brk = false;
    int64_t it_new = 0;
    if (kAlphaIn) {
        // p.Ap: all-reduced by the caller (state->pq), or the peers' pushed partials
        const double pq = (peer != nullptr) ? peer_wait_sum_block(peer) : s->pq;
        it_new = s->iteration + 1;
        brk = pq <= 0.0;  // kernels.py:317 (NaN falls through)
        alpha = s->rho / pq;
        repl = it_new % kReplaceEvery == 0;
    } else {
        alpha = s->alpha;
        repl = cg_replacing(s);
    }
    const int64_t n_eff = brk ? 0 : n;
    // defer_x (distributed two-pass iteration): x += alpha p moves into the p
    // update, which reads p anyway; replacement iterations need x here
    const bool upd_x = !(defer_x && !repl);
    const int64_t np = n >> 1, T = int64_t(gridDim.x) * 256;
    const double2* p2 = reinterpret_cast<const double2*>(p);
    const double2* q2 = reinterpret_cast<const double2*>(q);
    double2* x2 = reinterpret_cast<double2*>(x);
    double2* r2 = reinterpret_cast<double2*>(r);
    double acc = 0.0;
    const int64_t np_eff = n_eff >> 1;
    // rev: pairs visited from the end (see cg_solve: kernels alternate directions)
    for (int64_t kl = int64_t(blockIdx.x) * 256 + threadIdx.x; kl < np_eff; kl += 2 * T) {
        const bool h1 = kl + T < np;
        const int64_t k = rev ? np - 1 - kl : kl, k1 = rev ? np - 1 - (kl + T) : kl + T;
        // p is read again by the p update, which starts on the rows read here
        // last: a plain load (not evict-first) lets it hit L2
        double2 pa{0, 0}, xa{0, 0}, pb{0, 0}, xb{0, 0}, qa{0, 0}, ra{0, 0}, qb{0, 0}, rb{0, 0};
        if (upd_x) {
            pa = p2[k];
            xa = __ldcs(x2 + k);
            if (h1) {
                pb = p2[k1];
                xb = __ldcs(x2 + k1);
            }
        }
        if (!repl) {
            qa = __ldcs(q2 + k);
            ra = __ldcs(r2 + k);
            if (h1) {
                qb = __ldcs(q2 + k1);
                rb = __ldcs(r2 + k1);
            }
        }
        if (upd_x) {
            xa.x = __dadd_rn(xa.x, __dmul_rn(alpha, pa.x));
            xa.y = __dadd_rn(xa.y, __dmul_rn(alpha, pa.y));
            __stcs(x2 + k, xa);
            if (h1) {
                xb.x = __dadd_rn(xb.x, __dmul_rn(alpha, pb.x));
                xb.y = __dadd_rn(xb.y, __dmul_rn(alpha, pb.y));
                __stcs(x2 + k1, xb);
            }
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
        if (upd_x) x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
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
            if (peer != nullptr) {
                peer_push_scalar(peer, total);
            } else {
                s->rr = total;
                if (finalize) cg_beta_step(s, hist);
            }
        }
    }
}

// kBetaIn: beta = r.r / rho is evaluated here from the all-reduced r.r and the
// last block performs the beta step (history, rho, convergence flag).
template <bool kBetaIn>
__global__ void __launch_bounds__(256)
cg_update_p_vec(int64_t n, const double* __restrict__ r, double* __restrict__ p, wk_cg_state* s, double* hist,
                RedWorkspace ws, PeerCtx* peer, const PeerHalo* halo, int rev = 0, double* __restrict__ x = nullptr) {
    if (s->done) return;
    double rr = 0.0;
    if (kBetaIn) rr = (peer != nullptr) ? peer_wait_sum_block(peer) : s->rr;
    const double beta = kBetaIn ? rr / s->rho : s->beta;
    // x != nullptr (distributed two-pass iteration): the x += alpha p_old the
    // x/r update deferred, on every iteration but the residual replacement
    const bool upd_x = x != nullptr && !cg_replacing(s);
    const double alpha = s->alpha;
    const int64_t np = n >> 1, T = int64_t(gridDim.x) * 256;
    const double2* r2 = reinterpret_cast<const double2*>(r);
    double2* p2 = reinterpret_cast<double2*>(p);
    double2* x2 = reinterpret_cast<double2*>(x);
    // four pairs of r and p in flight per thread (a copy-shaped step: two
    // pairs left it at 5.7 TB/s)
    constexpr int U = 4;
    for (int64_t kl = int64_t(blockIdx.x) * 256 + threadIdx.x; kl < np; kl += U * T) {
        double2 ra[U], pa[U], xa[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t ku = kl + u * T;
            const int64_t k = rev ? np - 1 - ku : ku;
            ra[u] = ku < np ? __ldcs(r2 + k) : make_double2(0.0, 0.0);
            pa[u] = ku < np ? p2[k] : make_double2(0.0, 0.0);
            xa[u] = ku < np && upd_x ? __ldcs(x2 + k) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t ku = kl + u * T;
            if (ku >= np) break;
            const int64_t k = rev ? np - 1 - ku : ku;
            if (upd_x) {
                xa[u].x = __dadd_rn(xa[u].x, __dmul_rn(alpha, pa[u].x));
                xa[u].y = __dadd_rn(xa[u].y, __dmul_rn(alpha, pa[u].y));
                __stcs(x2 + k, xa[u]);
            }
            double2 q;
            q.x = __dadd_rn(ra[u].x, __dmul_rn(beta, pa[u].x));
            q.y = __dadd_rn(ra[u].y, __dmul_rn(beta, pa[u].y));
            p2[k] = q;
            if (halo != nullptr) {  // the boundary rows go straight into the neighbours' halo copies
                halo_store(peer, halo, 2 * k, q.x);
                halo_store(peer, halo, 2 * k + 1, q.y);
            }
        }
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        if (upd_x) x[n - 1] = __dadd_rn(x[n - 1], __dmul_rn(alpha, p[n - 1]));
        p[n - 1] = __dadd_rn(r[n - 1], __dmul_rn(beta, p[n - 1]));
        if (halo != nullptr) halo_store(peer, halo, n - 1, p[n - 1]);
    }
    if (halo != nullptr) {
        __syncthreads();
        if (threadIdx.x == 0) __threadfence_system();  // this block's peer stores, before its ticket
    }
    if (kBetaIn) {
        double total;
        if (grid_reduce_last(0.0, ws, total) && threadIdx.x == 0) {
            s->rr = rr;
            cg_beta_step(s, hist);
            if (halo != nullptr) halo_release(peer, halo);
        }
    }
}

// Single-GPU CG iteration in two vector passes instead of three (the
// non-replacement iterations of wk_cg_solve's graph). The reference updates x
// then r (kernels.py:320-325) and then p (329); the three updates are
// element-wise and independent of each other's order, so x can wait for the
// p pass, which reads p_old anyway:
//   cg_update_r_vec   r -= alpha q, r.r (beta step in the last block); marks
//                     the x update of this iteration pending (xpend)
//   cg_update_xp_vec  x += alpha p_old and, unless the beta step ended the
//                     solve, p = r + beta p_old; the last block clears xpend
// 8 vector passes per iteration instead of 9 (p is read once less), every
// element bitwise as before (7.5 with the x updates of two iterations applied
// together, cg_update_xp_pair). Residual-replacement iterations need the new
// x before the next r, so they keep cg_update_xr_vec + cg_update_p_vec.
__global__ void __launch_bounds__(256)
cg_update_r_vec(int64_t n, const double* __restrict__ q, double* __restrict__ r, wk_cg_state* s, double* hist,
                RedWorkspace ws, int rev) {
    if (s->done) return;
    const double alpha = s->alpha;
    const int64_t np = n >> 1, T = int64_t(gridDim.x) * 256;
    const double2* q2 = reinterpret_cast<const double2*>(q);
    double2* r2 = reinterpret_cast<double2*>(r);
    double acc = 0.0;
    constexpr int U = 4;
    for (int64_t kl = int64_t(blockIdx.x) * 256 + threadIdx.x; kl < np; kl += U * T) {
        double2 qa[U], ra[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t ku = kl + u * T;
            const int64_t k = rev ? np - 1 - ku : ku;
            qa[u] = ku < np ? __ldcs(q2 + k) : make_double2(0.0, 0.0);
            ra[u] = ku < np ? __ldcs(r2 + k) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t ku = kl + u * T;
            if (ku >= np) break;
            const int64_t k = rev ? np - 1 - ku : ku;
            ra[u].x = __dadd_rn(ra[u].x, -__dmul_rn(alpha, qa[u].x));
            ra[u].y = __dadd_rn(ra[u].y, -__dmul_rn(alpha, qa[u].y));
            r2[k] = ra[u];  // read next by the x/p pass, which starts on these rows
            acc += __dmul_rn(ra[u].x, ra[u].x);
            acc += __dmul_rn(ra[u].y, ra[u].y);
        }
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const int64_t i = n - 1;
        r[i] = __dadd_rn(r[i], -__dmul_rn(alpha, q[i]));
        acc += __dmul_rn(r[i], r[i]);
    }
    double total;
    if (grid_reduce_last(acc, ws, total) && threadIdx.x == 0) {
        s->rr = total;
        cg_beta_step(s, hist);
        s->xpend = 1;
    }
}

__global__ void __launch_bounds__(256)
cg_update_xp_vec(int64_t n, const double* __restrict__ r, double* __restrict__ x, double* __restrict__ p,
                 wk_cg_state* s, RedWorkspace ws, int rev) {
    if (!s->xpend) return;
    const double alpha = s->alpha, beta = s->beta;
    const bool upd_p = !s->done;
    const int64_t np = n >> 1, T = int64_t(gridDim.x) * 256;
    const double2* r2 = reinterpret_cast<const double2*>(r);
    double2* x2 = reinterpret_cast<double2*>(x);
    double2* p2 = reinterpret_cast<double2*>(p);
    constexpr int U = 2;
    for (int64_t kl = int64_t(blockIdx.x) * 256 + threadIdx.x; kl < np; kl += U * T) {
        double2 pa[U], xa[U], ra[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t ku = kl + u * T;
            const int64_t k = rev ? np - 1 - ku : ku;
            const bool ok = ku < np;
            pa[u] = ok ? p2[k] : make_double2(0.0, 0.0);
            xa[u] = ok ? __ldcs(x2 + k) : make_double2(0.0, 0.0);
            ra[u] = ok && upd_p ? __ldcs(r2 + k) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t ku = kl + u * T;
            if (ku >= np) break;
            const int64_t k = rev ? np - 1 - ku : ku;
            xa[u].x = __dadd_rn(xa[u].x, __dmul_rn(alpha, pa[u].x));
            xa[u].y = __dadd_rn(xa[u].y, __dmul_rn(alpha, pa[u].y));
            __stcs(x2 + k, xa[u]);
            if (upd_p) {
                double2 q;
                q.x = __dadd_rn(ra[u].x, __dmul_rn(beta, pa[u].x));
                q.y = __dadd_rn(ra[u].y, __dmul_rn(beta, pa[u].y));
                p2[k] = q;
            }
        }
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const int64_t i = n - 1;
        const double pi = p[i];
        x[i] = __dadd_rn(x[i], __dmul_rn(alpha, pi));
        if (upd_p) p[i] = __dadd_rn(r[i], __dmul_rn(beta, pi));
    }
    double total;
    if (grid_reduce_last(0.0, ws, total) && threadIdx.x == 0) s->xpend = 0;  // every block has read it
}

// The x update of every other iteration deferred and applied together with
// the next one (pairs of two-pass iterations, wk_cg_solve):
//   kPair = 0  p_next = r + beta p into the other p buffer; x += alpha p is
//              deferred (alpha kept in alpha_prev, p stays in its buffer).
//              If the beta step ended the solve, x += alpha p is applied now.
//   kPair = 1  x += alpha_prev p_prev, then x += alpha p (two separately
//              rounded adds per element: the same roundings, in the same
//              order, as two passes); p_next = r + beta p into p_prev's buffer.
// x is read and written once per two iterations instead of every iteration:
// 3 + 6 vectors per pair instead of 5 + 5, every element bitwise as before.
template <int kPair>
__global__ void __launch_bounds__(256)
cg_update_xp_pair(int64_t n, const double* __restrict__ r, double* __restrict__ x, const double* __restrict__ p,
                  const double* __restrict__ pprev, double* __restrict__ pn, wk_cg_state* s, RedWorkspace ws,
                  int rev) {
    if (!s->xpend) return;
    const double alpha = s->alpha, beta = s->beta, alpha0 = kPair ? s->alpha_prev : 0.0;
    const bool upd_p = !s->done;
    const bool upd_x = kPair == 1 || !upd_p;
    const int64_t np = n >> 1, T = int64_t(gridDim.x) * 256;
    const double2* r2 = reinterpret_cast<const double2*>(r);
    const double2* p2 = reinterpret_cast<const double2*>(p);
    const double2* q2 = reinterpret_cast<const double2*>(pprev);
    double2* x2 = reinterpret_cast<double2*>(x);
    double2* n2 = reinterpret_cast<double2*>(pn);
    constexpr int U = 2;
    const double2 z = make_double2(0.0, 0.0);
    for (int64_t kl = int64_t(blockIdx.x) * 256 + threadIdx.x; kl < np; kl += U * T) {
        double2 pa[U], xa[U], ra[U], qa[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t ku = kl + u * T;
            const int64_t k = rev ? np - 1 - ku : ku;
            const bool ok = ku < np;
            pa[u] = ok ? p2[k] : z;
            xa[u] = ok && upd_x ? __ldcs(x2 + k) : z;
            ra[u] = ok && upd_p ? __ldcs(r2 + k) : z;
            qa[u] = ok && kPair == 1 ? __ldcs(q2 + k) : z;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t ku = kl + u * T;
            if (ku >= np) break;
            const int64_t k = rev ? np - 1 - ku : ku;
            if (upd_x) {
                if (kPair == 1) {
                    xa[u].x = __dadd_rn(xa[u].x, __dmul_rn(alpha0, qa[u].x));
                    xa[u].y = __dadd_rn(xa[u].y, __dmul_rn(alpha0, qa[u].y));
                }
                xa[u].x = __dadd_rn(xa[u].x, __dmul_rn(alpha, pa[u].x));
                xa[u].y = __dadd_rn(xa[u].y, __dmul_rn(alpha, pa[u].y));
                __stcs(x2 + k, xa[u]);
            }
            if (upd_p) {
                double2 v;
                v.x = __dadd_rn(ra[u].x, __dmul_rn(beta, pa[u].x));
                v.y = __dadd_rn(ra[u].y, __dmul_rn(beta, pa[u].y));
                n2[k] = v;
            }
        }
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const int64_t i = n - 1;
        const double pi = p[i];
        if (upd_x) {
            double xi = x[i];
            if (kPair == 1) xi = __dadd_rn(xi, __dmul_rn(alpha0, pprev[i]));
            x[i] = __dadd_rn(xi, __dmul_rn(alpha, pi));
        }
        if (upd_p) pn[i] = __dadd_rn(r[i], __dmul_rn(beta, pi));
    }
    double total;
    if (grid_reduce_last(0.0, ws, total) && threadIdx.x == 0) {  // every block has read the state
        s->xpend = 0;
        s->xdefer = upd_x ? 0 : 1;
        if (!upd_x) s->alpha_prev = alpha;
    }
}

static int cg_update_xr(int64_t n, const double* p, const double* q, double* x, double* r, wk_cg_state* s,
                        double* hist, void* ws, bool finalize, cudaStream_t st, int rev = 0) {
    if (n > 0 && vec_ok(p, q, x, r)) {
        cg_update_xr_vec<false><<<vec_grid(n), 256, 0, st>>>(n, p, q, x, r, s, hist, red_ws(ws), finalize ? 1 : 0,
                                                            nullptr, rev);
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
                        void* ws, bool finalize, cudaStream_t st, PeerCtx* peer = nullptr) {
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
            if (peer != nullptr) {
                peer_push_scalar(peer, t);
                return;
            }
            s->rr = t;
            if (finalize) cg_beta_step(s, hist);
        },
        ws, &s->done, st);
}

static int cg_update_p(int64_t n, const double* r, double* p, const wk_cg_state* s, cudaStream_t st, int rev = 0) {
    if (n > 0 && vec_ok(r, p, r, p)) {
        cg_update_p_vec<false><<<vec_grid(n), 256, 0, st>>>(n, r, p, const_cast<wk_cg_state*>(s), nullptr,
                                                          RedWorkspace{nullptr, nullptr}, nullptr, nullptr, rev);
        WK_LAUNCH_CHECK();
        return 0;
    }
    return launch_masked_map(
        n, [=] __device__(int64_t i) { p[i] = __dadd_rn(r[i], __dmul_rn(s->beta, p[i])); }, &s->done, st);
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
    cg_update_xr_vec<true><<<vec_grid(n > 0 ? n : 1), 256, 0, as_stream(stream)>>>(
        n, p, q, x, r, state, nullptr, red_ws(workspace), 0, nullptr, 0, 1);
    WK_LAUNCH_CHECK();
    return 0;
}

int wk_cg_update_p_beta(int64_t n, const double* r, double* p, double* x, wk_cg_state* state, double* hist,
                        void* workspace, wk_stream_t stream) {
    clear_error();
    WK_REQUIRE(vec_ok(r, p, x, p), WK_ERR_INVALID, "wk_cg_update_p_beta needs 16-byte aligned vectors");
    cg_update_p_vec<true><<<vec_grid(n > 0 ? n : 1), 256, 0, as_stream(stream)>>>(
        n, r, p, state, hist, red_ws(workspace), nullptr, nullptr, 0, x);
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

// ---------------- CG steps with the all-reduces fused (peer-memory path) ---------
// Each producer's reduction epilogue pushes its local partial to every rank
// (peer_dev.cuh); the next kernel's prologue waits for the P partials and sums
// them in rank order. One iteration: spmv_dot (push p.Ap) -> update_xr_alpha
// (wait p.Ap, alpha, x/r, push r.r) [-> replace_r on replacement iterations]
// -> update_p_beta (wait r.r, beta, p): no separate all-reduce kernels.

int wk_cg_spmv_dot_peer(const wk_matrix* A, const double* p, double* q, wk_cg_state* state, void* workspace,
                        void* peer, const void* halo, wk_stream_t stream) {
    clear_error();
    return cg_spmv_dot(A, A->nrows, p, q, state, workspace, false, as_stream(stream),
                       reinterpret_cast<PeerCtx*>(peer), reinterpret_cast<const PeerHalo*>(halo));
}

int wk_cg_update_xr_alpha_peer(int64_t n, const double* p, const double* q, double* x, double* r,
                               wk_cg_state* state, void* workspace, void* peer, wk_stream_t stream) {
    clear_error();
    WK_REQUIRE(vec_ok(p, q, x, r), WK_ERR_INVALID, "wk_cg_update_xr_alpha_peer needs 16-byte aligned vectors");
    cg_update_xr_vec<true><<<vec_grid(n > 0 ? n : 1), 256, 0, as_stream(stream)>>>(
        n, p, q, x, r, state, nullptr, red_ws(workspace), 0, reinterpret_cast<PeerCtx*>(peer), 0, 1);
    WK_LAUNCH_CHECK();
    return 0;
}

int wk_cg_replace_r_peer(int64_t n, const double* b, const double* q, double* r, wk_cg_state* state,
                         void* workspace, void* peer, wk_stream_t stream) {
    clear_error();
    PeerCtx* pc = reinterpret_cast<PeerCtx*>(peer);
    if (n == 0)
        return launch_scalar([=] __device__() {
            if (!state->done && cg_replacing(state)) peer_push_scalar(pc, 0.0);
        }, as_stream(stream));
    return cg_replace_r(n, b, q, r, state, nullptr, workspace, false, as_stream(stream), pc);
}

int wk_cg_update_p_beta_peer(int64_t n, const double* r, double* p, double* x, wk_cg_state* state, double* hist,
                             void* workspace, void* peer, const void* halo, wk_stream_t stream) {
    clear_error();
    WK_REQUIRE(vec_ok(r, p, x, p), WK_ERR_INVALID, "wk_cg_update_p_beta_peer needs 16-byte aligned vectors");
    cg_update_p_vec<true><<<vec_grid(n > 0 ? n : 1), 256, 0, as_stream(stream)>>>(
        n, r, p, state, hist, red_ws(workspace), reinterpret_cast<PeerCtx*>(peer),
        reinterpret_cast<const PeerHalo*>(halo), 0, x);
    WK_LAUNCH_CHECK();
    return 0;
}

// ---------------- single-GPU CG ---------------------------------------------------

int64_t wk_cg_workspace_bytes(int64_t n) {
    return 256 + red_ws_bytes() + 256 + 4 * (ceil_div(n * 8, 256) * 256) + 256;
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
    double* p1 = cv.take<double>(n);  // the second p buffer of paired iterations
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
    // L2 ping-pong: consecutive kernels walk the rows in opposite directions,
    // so each starts on the rows the previous one touched last (the most
    // recently written q / r / p are still in the 126 MB L2). Iteration i:
    // SpMV d, x/r update !d, p update d, with d flipping every iteration (the
    // 50-iteration period is even).
    // the two-pass iteration (cg_update_r_vec / cg_update_xp_vec) for every
    // iteration but the residual replacement, when the vectors are aligned
    // Iterations 0..47 run in pairs (cg_update_xp_pair): the even one leaves
    // its x update pending and writes the next p into p1, the odd one applies
    // both x updates and writes the next p back into p; iteration 48 is a
    // plain two-pass iteration and 49 the residual replacement (both in p).
    const bool two_pass = n > 0 && vec_ok(p, q, x, r) && vec_ok(p1, p1, p1, p1) && vec_grid(n) <= kRedMaxBlocks;
    int rc = capture(g, [&](cudaStream_t cs) -> int {
        for (int i = 0; i < kReplaceEvery; ++i) {
            const int d = i & 1;
            const bool paired = two_pass && i < kReplaceEvery - 2;
            const double* pcur = paired && (i & 1) ? p1 : p;
            WK_TRY(cg_spmv_dot(A, n, pcur, q, s, red, true, cs, nullptr, nullptr, d));
            if (two_pass && i < kReplaceEvery - 1) {
                cg_update_r_vec<<<vec_grid(n), 256, 0, cs>>>(n, q, r, s, hist, red_ws(red), 1 - d);
                WK_LAUNCH_CHECK();
                if (paired && !(i & 1))
                    cg_update_xp_pair<0><<<vec_grid(n), 256, 0, cs>>>(n, r, x, p, nullptr, p1, s, red_ws(red), d);
                else if (paired)
                    cg_update_xp_pair<1><<<vec_grid(n), 256, 0, cs>>>(n, r, x, p1, p, p, s, red_ws(red), d);
                else
                    cg_update_xp_vec<<<vec_grid(n), 256, 0, cs>>>(n, r, x, p, s, red_ws(red), d);
                WK_LAUNCH_CHECK();
                continue;
            }
            WK_TRY(cg_update_xr(n, p, q, x, r, s, hist, red, true, cs, 1 - d));
            if (i == kReplaceEvery - 1) {
                WK_TRY(wk_spmv_masked(A, x, q, &s->done, cs));
                WK_TRY(cg_replace_r(n, b, q, r, s, hist, red, true, cs));
            }
            WK_TRY(cg_update_p(n, r, p, s, cs, d));
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
    if (h.xdefer) {  // stopped by a breakdown right after an even iteration of a pair: x += alpha_prev p
        WK_TRY(launch_masked_map(
            n, [=] __device__(int64_t i) { x[i] = __dadd_rn(x[i], __dmul_rn(s->alpha_prev, p[i])); }, nullptr, st));
        WK_CUDA(cudaStreamSynchronize(st));
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

