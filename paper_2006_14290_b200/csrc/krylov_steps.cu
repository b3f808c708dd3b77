// BiCGSTAB and GMRES(m) as device step kernels (no reference implementation;
// update order of oracle/krylov_ref.py: van der Vorst BiCGSTAB, restarted
// GMRES with classical Gram-Schmidt via batched dots and Givens rotations on
// one device thread).
//
// Every vector step reduces into a LOCAL slot of the solver state; between a
// vector step and the scalar step that consumes it the row-block distributed
// driver (distributed.py) all-reduces that slot over NCCL, the single-GPU
// solvers below simply run the scalar step next. All steps are no-ops once
// the device `done` flag is set, so a fixed period can be captured as a CUDA
// graph and replayed until convergence.
#include "krylov_common.cuh"

namespace wk {

using BS = wk_bicg_state;
using GS = wk_gmres_state;

// ---------------------------------- BiCGSTAB ---------------------------------------

static int bicg_init(int64_t n, const double* b, double* x, double* r, double* rh, double* p, double* v, BS* s,
                     void* ws, cudaStream_t st) {
    if (n == 0) return launch_scalar([=] __device__() { s->rr = 0.0; }, st);
    return launch_map_reduce(
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
        [=] __device__(double t) { s->rr = t; }, ws, nullptr, st);
}

static int bicg_init_finish(BS* s, double tol, int64_t max_iters, double* hist, cudaStream_t st) {
    return launch_scalar([=] __device__() {
        const double bn = sqrt(s->rr);
        hist[0] = bn;
        s->rho = s->alpha = s->omega = 1.0;
        s->threshold = tol * bn;
        s->iteration = 0;
        s->max_iters = max_iters;
        s->breakdown = 0;
        s->apply_half = 0;
        s->done = !(bn != 0.0 && 0 < max_iters && bn > s->threshold);
    }, st);
}

template <typename F, typename E>
static int local_dot(int64_t n, F f, E epi, void* ws, const int* skip, cudaStream_t st) {
    if (n == 0) return launch_scalar([=] __device__() { if (!*skip) epi(0.0); }, st);
    return launch_map_reduce(n, f, epi, ws, skip, st);
}

// Vectorised paths (vmap_kernel, reduce.cuh) when every vector is 16-byte
// aligned; the scalar map_reduce lambdas below are the fallback. Same
// element arithmetic; the per-thread summation order of the dots differs.
struct NoScalars {
    __device__ int operator()() const { return 0; }
};
template <int N>
struct NoEpi {
    __device__ void operator()(double (&)[N]) const {}
};

static int bicg_rho(int64_t n, const double* rh, const double* r, BS* s, void* ws, cudaStream_t st) {
    if (n > 0 && vmap_ok({rh, r}))
        return launch_vmap<2, 0, 1>(
            n, VecArgs<2, 0>{{rh, r}, {nullptr}}, NoScalars{},
            [] __device__(int, const double(&in)[2], double(&)[1], double(&red)[1]) { red[0] = __dmul_rn(in[0], in[1]); },
            [=] __device__(double(&t)[1]) { s->rho_new = t[0]; }, ws, &s->done, st);
    return local_dot(
        n, [=] __device__(int64_t i) { return __dmul_rn(rh[i], r[i]); },
        [=] __device__(double t) { s->rho_new = t; }, ws, &s->done, st);
}

static int bicg_step_beta(BS* s, cudaStream_t st) {
    return launch_scalar([=] __device__() {
        if (s->done) return;
        if (s->rho_new == 0.0) {
            s->breakdown = 1;
            s->done = 1;
            s->iteration += 1;
            return;
        }
        s->beta = __dmul_rn(s->rho_new / s->rho, s->alpha / s->omega);
    }, st);
}

static int bicg_update_p(int64_t n, const double* r, const double* v, double* p, BS* s, cudaStream_t st) {
    if (n > 0 && vmap_ok({r, v, p}))
        return launch_vmap<3, 1, 0>(
            n, VecArgs<3, 1>{{r, v, p}, {p}}, [=] __device__() { return make_double2(s->beta, s->omega); },
            [] __device__(double2 c, const double(&in)[3], double(&out)[1], double(&)[1]) {
                out[0] = __dadd_rn(in[0], __dmul_rn(c.x, __dadd_rn(in[2], -__dmul_rn(c.y, in[1]))));
            },
            NoEpi<1>{}, nullptr, &s->done, st);
    return launch_masked_map(
        n,
        [=] __device__(int64_t i) {
            p[i] = __dadd_rn(r[i], __dmul_rn(s->beta, __dadd_rn(p[i], -__dmul_rn(s->omega, v[i]))));
        },
        &s->done, st);
}

static int bicg_rv(int64_t n, const double* rh, const double* v, BS* s, void* ws, cudaStream_t st) {
    if (n > 0 && vmap_ok({rh, v}))
        return launch_vmap<2, 0, 1>(
            n, VecArgs<2, 0>{{rh, v}, {nullptr}}, NoScalars{},
            [] __device__(int, const double(&in)[2], double(&)[1], double(&red)[1]) { red[0] = __dmul_rn(in[0], in[1]); },
            [=] __device__(double(&t)[1]) { s->rv = t[0]; }, ws, &s->done, st);
    return local_dot(
        n, [=] __device__(int64_t i) { return __dmul_rn(rh[i], v[i]); }, [=] __device__(double t) { s->rv = t; },
        ws, &s->done, st);
}

static int bicg_step_alpha(BS* s, cudaStream_t st) {
    return launch_scalar([=] __device__() {
        if (s->done) return;
        if (s->rv == 0.0) {
            s->breakdown = 1;
            s->done = 1;
            s->iteration += 1;
            return;
        }
        s->alpha = s->rho_new / s->rv;
    }, st);
}

static int bicg_update_s(int64_t n, const double* r, const double* v, double* sv, BS* s, void* ws, cudaStream_t st) {
    if (n > 0 && vmap_ok({r, v, sv}))
        return launch_vmap<2, 1, 1>(
            n, VecArgs<2, 1>{{r, v}, {sv}}, [=] __device__() { return s->alpha; },
            [] __device__(double alpha, const double(&in)[2], double(&out)[1], double(&red)[1]) {
                const double si = __dadd_rn(in[0], -__dmul_rn(alpha, in[1]));
                out[0] = si;
                red[0] = __dmul_rn(si, si);
            },
            [=] __device__(double(&t)[1]) { s->ss = t[0]; }, ws, &s->done, st);
    return local_dot(
        n,
        [=] __device__(int64_t i) {
            const double si = __dadd_rn(r[i], -__dmul_rn(s->alpha, v[i]));
            sv[i] = si;
            return __dmul_rn(si, si);
        },
        [=] __device__(double t) { s->ss = t; }, ws, &s->done, st);
}

static int bicg_step_s(BS* s, double* hist, cudaStream_t st) {
    return launch_scalar([=] __device__() {
        if (s->done) return;
        s->iteration += 1;
        const double sn = sqrt(s->ss);
        if (sn <= s->threshold) {
            hist[s->iteration] = sn;
            s->apply_half = 1;
            s->done = 1;
        }
    }, st);
}

static int bicg_half_x(int64_t n, const double* p, double* x, BS* s, void* ws, cudaStream_t st) {
    if (n == 0) return launch_scalar([=] __device__() { s->apply_half = 0; }, st);
    if (vmap_ok({p, x}))  // runs only when the flag is set (once, at an early exit)
        return launch_vmap<2, 1, 1, true>(
            n, VecArgs<2, 1>{{x, p}, {x}}, [=] __device__() { return s->alpha; },
            [] __device__(double alpha, const double(&in)[2], double(&out)[1], double(&red)[1]) {
                out[0] = __dadd_rn(in[0], __dmul_rn(alpha, in[1]));
                red[0] = 0.0;
            },
            [=] __device__(double(&)[1]) { s->apply_half = 0; }, ws, &s->apply_half, st);
    return launch_map_reduce(
        n,
        [=] __device__(int64_t i) {
            if (s->apply_half) x[i] = __dadd_rn(x[i], __dmul_rn(s->alpha, p[i]));
            return 0.0;
        },
        [=] __device__(double) { s->apply_half = 0; }, ws, nullptr, st);
}

static int bicg_tt_ts(int64_t n, const double* t, const double* sv, BS* s, void* ws, cudaStream_t st) {
    if (n == 0)
        return launch_scalar([=] __device__() {
            if (!s->done) s->tt = s->ts = 0.0;
        }, st);
    if (vmap_ok({t, sv}))
        return launch_vmap<2, 0, 2>(
            n, VecArgs<2, 0>{{t, sv}, {nullptr}}, NoScalars{},
            [] __device__(int, const double(&in)[2], double(&)[1], double(&red)[2]) {
                red[0] = __dmul_rn(in[0], in[0]);
                red[1] = __dmul_rn(in[0], in[1]);
            },
            [=] __device__(double(&tot)[2]) {
                s->tt = tot[0];
                s->ts = tot[1];
            },
            ws, &s->done, st);
    return launch_map_reduce_n<2>(
        n,
        [=] __device__(int64_t i, double(&acc)[2]) {
            const double ti = t[i];
            acc[0] += __dmul_rn(ti, ti);
            acc[1] += __dmul_rn(ti, sv[i]);
        },
        [=] __device__(double(&tot)[2]) {
            s->tt = tot[0];
            s->ts = tot[1];
        },
        ws, &s->done, st);
}

static int bicg_step_omega(BS* s, cudaStream_t st) {
    return launch_scalar([=] __device__() {
        if (s->done) return;
        if (s->tt == 0.0) {
            s->breakdown = 1;
            s->done = 1;
            return;
        }
        s->omega = s->ts / s->tt;
    }, st);
}

static int bicg_update_xr(int64_t n, const double* p, const double* sv, const double* t, double* x, double* r, BS* s,
                          void* ws, cudaStream_t st) {
    if (n > 0 && vmap_ok({p, sv, t, x, r}))
        return launch_vmap<4, 2, 1>(
            n, VecArgs<4, 2>{{x, p, sv, t}, {x, r}}, [=] __device__() { return make_double2(s->alpha, s->omega); },
            [] __device__(double2 c, const double(&in)[4], double(&out)[2], double(&red)[1]) {
                out[0] = __dadd_rn(__dadd_rn(in[0], __dmul_rn(c.x, in[1])), __dmul_rn(c.y, in[2]));
                const double ri = __dadd_rn(in[2], -__dmul_rn(c.y, in[3]));
                out[1] = ri;
                red[0] = __dmul_rn(ri, ri);
            },
            [=] __device__(double(&tot)[1]) { s->rr = tot[0]; }, ws, &s->done, st);
    return local_dot(
        n,
        [=] __device__(int64_t i) {
            x[i] = __dadd_rn(__dadd_rn(x[i], __dmul_rn(s->alpha, p[i])), __dmul_rn(s->omega, sv[i]));
            const double ri = __dadd_rn(sv[i], -__dmul_rn(s->omega, t[i]));
            r[i] = ri;
            return __dmul_rn(ri, ri);
        },
        [=] __device__(double tot) { s->rr = tot; }, ws, &s->done, st);
}

// wk_bicgstab_solve's fused variant of bicg_update_xr + the next iteration's
// bicg_rho: the new r is in registers, so rh.r (rho_new of the next
// iteration) is summed in the same pass (one read of rh instead of a pass
// over rh and r). Same vmap traversal and grid as bicg_rho: the sum is
// bitwise the one bicg_rho would return.
static int bicg_update_xr_rho(int64_t n, const double* p, const double* sv, const double* t, const double* rh,
                              double* x, double* r, BS* s, void* ws, cudaStream_t st) {
    return launch_vmap<5, 2, 2>(
        n, VecArgs<5, 2>{{x, p, sv, t, rh}, {x, r}}, [=] __device__() { return make_double2(s->alpha, s->omega); },
        [] __device__(double2 c, const double(&in)[5], double(&out)[2], double(&red)[2]) {
            out[0] = __dadd_rn(__dadd_rn(in[0], __dmul_rn(c.x, in[1])), __dmul_rn(c.y, in[2]));
            const double ri = __dadd_rn(in[2], -__dmul_rn(c.y, in[3]));
            out[1] = ri;
            red[0] = __dmul_rn(ri, ri);
            red[1] = __dmul_rn(in[4], ri);
        },
        [=] __device__(double(&tot)[2]) {
            s->rr = tot[0];
            s->rho_next = tot[1];
        },
        ws, &s->done, st);
}

// rho_new of the coming iteration from the previous fused x/r step (or from
// bicg_rho_first before the first iteration)
static int bicg_take_rho(BS* s, cudaStream_t st) {
    return launch_scalar([=] __device__() {
        if (!s->done) s->rho_new = s->rho_next;
    }, st);
}

static int bicg_rho_first(int64_t n, const double* rh, const double* r, BS* s, void* ws, cudaStream_t st) {
    return launch_vmap<2, 0, 1>(
        n, VecArgs<2, 0>{{rh, r}, {nullptr}}, NoScalars{},
        [] __device__(int, const double(&in)[2], double(&)[1], double(&red)[1]) { red[0] = __dmul_rn(in[0], in[1]); },
        [=] __device__(double(&t)[1]) { s->rho_next = t[0]; }, ws, &s->done, st);
}

static int bicg_step_r(BS* s, double* hist, cudaStream_t st) {
    return launch_scalar([=] __device__() {
        if (s->done) return;
        const double rn = sqrt(s->rr);
        hist[s->iteration] = rn;
        s->rho = s->rho_new;
        s->done = !(s->iteration < s->max_iters && rn > s->threshold);
    }, st);
}

// ----------------------------------- GMRES ---------------------------------------------

static int gmres_init(int64_t n, const double* b, double* x, double* r, GS* s, void* ws, cudaStream_t st) {
    if (n == 0) return launch_scalar([=] __device__() { s->sq = 0.0; }, st);
    return launch_map_reduce(
        n,
        [=] __device__(int64_t i) {
            x[i] = 0.0;
            r[i] = b[i];
            return __dmul_rn(b[i], b[i]);
        },
        [=] __device__(double t) { s->sq = t; }, ws, nullptr, st);
}

static int gmres_init_finish(GS* s, double tol, int64_t max_iters, int restart, double* hist, cudaStream_t st) {
    return launch_scalar([=] __device__() {
        const double bn = sqrt(s->sq);
        hist[0] = bn;
        s->beta = bn;
        s->threshold = tol * bn;
        s->iteration = 0;
        s->max_iters = max_iters;
        s->restart = restart;
        s->done = !(bn != 0.0 && 0 < max_iters && bn > s->threshold);
        s->cycle_done = s->done;
        s->j_done = 0;
    }, st);
}

static int gmres_cycle_start(int64_t n, const double* r, double* V0, double* g, GS* s, cudaStream_t st) {
    int rc;
    if (n > 0 && vmap_ok({r, V0}))
        rc = launch_vmap<1, 1, 0>(
            n, VecArgs<1, 1>{{r}, {V0}}, [=] __device__() { return s->beta; },
            [] __device__(double beta, const double(&in)[1], double(&out)[1], double(&)[1]) { out[0] = in[0] / beta; },
            NoEpi<1>{}, nullptr, &s->done, st);
    else
        rc = launch_masked_map(n, [=] __device__(int64_t i) { V0[i] = r[i] / s->beta; }, &s->done, st);
    if (rc) return rc;
    return launch_scalar([=] __device__() {
        if (s->done) return;
        for (int i = 0; i <= s->restart; ++i) g[i] = 0.0;
        g[0] = s->beta;
        s->j_done = 0;
        s->cycle_done = 0;
    }, st);
}

template <int K>
static int gmres_multidot_k(int64_t n, int k, const double* V, int64_t ld, const double* w, double* Hj, GS* s,
                            void* ws, cudaStream_t st) {
    return launch_map_reduce_n<K>(
        n,
        [=] __device__(int64_t i, double(&acc)[K]) {
            const double wi = w[i];
#pragma unroll
            for (int q = 0; q < K; ++q)
                if (q < k) acc[q] += __dmul_rn(V[int64_t(q) * ld + i], wi);
        },
        [=] __device__(double(&tot)[K]) {
            for (int q = 0; q < k; ++q) Hj[q] = tot[q];
        },
        ws, &s->cycle_done, st);
}

// Vectorised classical Gram-Schmidt kernels: double2 loads of w and of the
// k <= K basis vectors (all issued before any use: k+1 independent 16-byte
// loads in flight per thread), one pass over the basis per kernel. Same
// per-element arithmetic as the scalar lambdas (kept for unaligned operands).
constexpr int kCgsGroup = 8;  // basis vectors loaded together (16-byte loads in flight per thread)

static int cgs_grid(int64_t n, int K) {
    int64_t g = ceil_div(ceil_div(n, 2), 256);
    const int64_t cap = int64_t(sm_count()) * (K > 16 ? 2 : 4);
    if (g > cap) g = cap;
    if (g > kRedMaxBlocks) g = kRedMaxBlocks;
    return int(g < 1 ? 1 : g);
}

static int orth_grid(int64_t n) {
    int64_t g = ceil_div(ceil_div(n, 2), 256);
    const int64_t cap = int64_t(sm_count()) * 4;
    if (g > cap) g = cap;
    if (g > kRedMaxBlocks) g = kRedMaxBlocks;
    return int(g < 1 ? 1 : g);
}

static bool cgs_vec_ok(const double* V, int64_t ld, const double* w) {
    return ((reinterpret_cast<uintptr_t>(V) | reinterpret_cast<uintptr_t>(w)) & 15) == 0 && (ld & 1) == 0;
}

template <int K>
__global__ void __launch_bounds__(256)
gmres_multidot_vec(int64_t n, int k, const double* __restrict__ V, int64_t ld, const double* __restrict__ w,
                   double* __restrict__ Hj, const int* __restrict__ skip, RedWorkspace ws) {
    if (*skip) return;
    double acc[K];
#pragma unroll
    for (int q = 0; q < K; ++q) acc[q] = 0.0;
    const int64_t np = n >> 1, T = int64_t(gridDim.x) * 256;
    for (int64_t i = int64_t(blockIdx.x) * 256 + threadIdx.x; i < np; i += T) {
        const double2 wv = reinterpret_cast<const double2*>(w)[i];
#pragma unroll
        for (int g = 0; g < K; g += kCgsGroup) {
            double2 v[kCgsGroup];
#pragma unroll
            for (int u = 0; u < kCgsGroup; ++u)
                if (g + u < k) v[u] = __ldcs(reinterpret_cast<const double2*>(V + int64_t(g + u) * ld) + i);
#pragma unroll
            for (int u = 0; u < kCgsGroup; ++u)
                if (g + u < k) {
                    acc[g + u] += __dmul_rn(v[u].x, wv.x);
                    acc[g + u] += __dmul_rn(v[u].y, wv.y);
                }
        }
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < K; ++q)
            if (q < k) acc[q] += __dmul_rn(V[int64_t(q) * ld + n - 1], w[n - 1]);
    }
    double tot[K];
    if (grid_reduce_last_n<K>(acc, ws, tot) && threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < K; ++q)
            if (q < k) Hj[q] = tot[q];
    }
}

// (256, 4): at most 64 registers, so 4 blocks per SM of the orthogonalisation
// (which keeps no accumulators) instead of the 2 its K = 32 variant got with
// every basis load hoisted: 5.5-6.0 -> 6.2-6.4 TB/s (tools/orth_probe.py)
template <int K>
__global__ void __launch_bounds__(256, 4)
gmres_orth_vec(int64_t n, int k, const double* __restrict__ V, int64_t ld, double* __restrict__ w,
               const double* __restrict__ Hj, GS* s, RedWorkspace ws) {
    if (s->cycle_done) return;
    // projections in shared memory (broadcast reads): keeps K doubles out of
    // the register file, so more blocks stay resident
    __shared__ double h[K];
    if (threadIdx.x < K) h[threadIdx.x] = int(threadIdx.x) < k ? Hj[threadIdx.x] : 0.0;
    __syncthreads();
    double acc = 0.0;
    const int64_t np = n >> 1, T = int64_t(gridDim.x) * 256;
    for (int64_t i = int64_t(blockIdx.x) * 256 + threadIdx.x; i < np; i += T) {
        double2 wv = reinterpret_cast<const double2*>(w)[i];
#pragma unroll
        for (int g = 0; g < K; g += kCgsGroup) {
            double2 v[kCgsGroup];
#pragma unroll
            for (int u = 0; u < kCgsGroup; ++u)
                if (g + u < k) v[u] = __ldcs(reinterpret_cast<const double2*>(V + int64_t(g + u) * ld) + i);
#pragma unroll
            for (int u = 0; u < kCgsGroup; ++u)
                if (g + u < k) {
                    wv.x = __dadd_rn(wv.x, -__dmul_rn(h[g + u], v[u].x));
                    wv.y = __dadd_rn(wv.y, -__dmul_rn(h[g + u], v[u].y));
                }
        }
        reinterpret_cast<double2*>(w)[i] = wv;
        acc += __dmul_rn(wv.x, wv.x);
        acc += __dmul_rn(wv.y, wv.y);
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        double wi = w[n - 1];
#pragma unroll
        for (int q = 0; q < K; ++q)
            if (q < k) wi = __dadd_rn(wi, -__dmul_rn(h[q], V[int64_t(q) * ld + n - 1]));
        w[n - 1] = wi;
        acc += __dmul_rn(wi, wi);
    }
    double total;
    if (grid_reduce_last(acc, ws, total) && threadIdx.x == 0) s->sq = total;
}

// Deferred normalisation (single-GPU wk_gmres_solve): basis slot i holds
// u_i with v_i = sig[i] u_i, so the new direction is never rescaled in a
// separate pass. The SpMV writes z = A u_j straight into slot j+1 and the
// multidot leaves d_i = u_i . z in Hj; this kernel forms h_i = sig_i sig_j d_i
// (= v_i . A v_j), w = sig_j z - sum_i (h_i sig_i) u_i in place in slot j+1
// and ||w||^2; the Givens step then sets sig[j+1] = 1 / ||w||. Two vector
// passes (read w, write v_{j+1}) fewer per iteration; the same algorithm up
// to rounding (w is formed from sig_j z instead of A fl(w / h)).
template <int K>
__global__ void __launch_bounds__(256, 4)
gmres_orth_scaled_vec(int64_t n, int k, const double* __restrict__ V, int64_t ld, double* __restrict__ w,
                      double* __restrict__ Hj, const double* __restrict__ sig, GS* s, RedWorkspace ws) {
    if (s->cycle_done) return;
    __shared__ double c[K];
    __shared__ double hs[K];
    const double sj = sig[k - 1];
    if (threadIdx.x < K) {
        const int q = threadIdx.x;
        const double h = q < k ? __dmul_rn(__dmul_rn(sig[q], sj), Hj[q]) : 0.0;
        hs[q] = h;
        c[q] = q < k ? __dmul_rn(h, sig[q]) : 0.0;
    }
    __syncthreads();
    double acc = 0.0;
    const int64_t np = n >> 1, T = int64_t(gridDim.x) * 256;
    for (int64_t i = int64_t(blockIdx.x) * 256 + threadIdx.x; i < np; i += T) {
        double2 wv = reinterpret_cast<const double2*>(w)[i];
        wv.x = __dmul_rn(sj, wv.x);
        wv.y = __dmul_rn(sj, wv.y);
#pragma unroll
        for (int g = 0; g < K; g += kCgsGroup) {
            double2 v[kCgsGroup];
#pragma unroll
            for (int u = 0; u < kCgsGroup; ++u)
                if (g + u < k) v[u] = __ldcs(reinterpret_cast<const double2*>(V + int64_t(g + u) * ld) + i);
#pragma unroll
            for (int u = 0; u < kCgsGroup; ++u)
                if (g + u < k) {
                    wv.x = __dadd_rn(wv.x, -__dmul_rn(c[g + u], v[u].x));
                    wv.y = __dadd_rn(wv.y, -__dmul_rn(c[g + u], v[u].y));
                }
        }
        reinterpret_cast<double2*>(w)[i] = wv;
        acc += __dmul_rn(wv.x, wv.x);
        acc += __dmul_rn(wv.y, wv.y);
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        double wi = __dmul_rn(sj, w[n - 1]);
#pragma unroll
        for (int q = 0; q < K; ++q)
            if (q < k) wi = __dadd_rn(wi, -__dmul_rn(c[q], V[int64_t(q) * ld + n - 1]));
        w[n - 1] = wi;
        acc += __dmul_rn(wi, wi);
    }
    double total;
    if (grid_reduce_last(acc, ws, total) && threadIdx.x == 0) {  // every block has read the raw d_i
        for (int q = 0; q < k; ++q) Hj[q] = hs[q];
        s->sq = total;
    }
}

static int gmres_orth_scaled(int64_t n, int j, const double* V, int64_t ld, double* w, double* Hj, const double* sig,
                             GS* s, void* ws, cudaStream_t st) {
    const int k = j + 1;
    const RedWorkspace rw = red_ws(ws);
#define WK_ORTH_S(KK)                                                                             \
    do {                                                                                          \
        gmres_orth_scaled_vec<KK><<<orth_grid(n), 256, 0, st>>>(n, k, V, ld, w, Hj, sig, s, rw);  \
        WK_LAUNCH_CHECK();                                                                        \
        return 0;                                                                                 \
    } while (0)
    if (k <= 2) WK_ORTH_S(2);
    if (k <= 4) WK_ORTH_S(4);
    if (k <= 8) WK_ORTH_S(8);
    if (k <= 16) WK_ORTH_S(16);
    WK_ORTH_S(kRedMaxVec);
#undef WK_ORTH_S
}

#define WK_CGS_LAUNCH(KERN, KK, ...)                                                         \
    do {                                                                                   \
        KERN<KK><<<cgs_grid(n, KK), 256, 0, st>>>(__VA_ARGS__);                            \
        WK_LAUNCH_CHECK();                                                                 \
        return 0;                                                                          \
    } while (0)

static int gmres_multidot(int64_t n, int j, const double* V, int64_t ld, const double* w, double* Hj, GS* s, void* ws,
                          cudaStream_t st) {
    const int k = j + 1;
    WK_REQUIRE(k <= kRedMaxVec, WK_ERR_INVALID, "GMRES restart must be < %d", kRedMaxVec);
    if (n == 0)
        return launch_scalar([=] __device__() {
            if (!s->cycle_done)
                for (int q = 0; q < k; ++q) Hj[q] = 0.0;
        }, st);
    if (cgs_vec_ok(V, ld, w)) {
        const RedWorkspace rw = red_ws(ws);
        const int* skip = &s->cycle_done;
        if (k <= 2) WK_CGS_LAUNCH(gmres_multidot_vec, 2, n, k, V, ld, w, Hj, skip, rw);
        if (k <= 4) WK_CGS_LAUNCH(gmres_multidot_vec, 4, n, k, V, ld, w, Hj, skip, rw);
        if (k <= 8) WK_CGS_LAUNCH(gmres_multidot_vec, 8, n, k, V, ld, w, Hj, skip, rw);
        if (k <= 16) WK_CGS_LAUNCH(gmres_multidot_vec, 16, n, k, V, ld, w, Hj, skip, rw);
        // k > 16: two passes of 16 vectors (w is read twice, but 32 register
        // accumulators would leave one block per SM)
        gmres_multidot_vec<16><<<cgs_grid(n, 16), 256, 0, st>>>(n, 16, V, ld, w, Hj, skip, rw);
        WK_LAUNCH_CHECK();
        WK_CGS_LAUNCH(gmres_multidot_vec, 16, n, k - 16, V + 16 * ld, ld, w, Hj + 16, skip, rw);
    }
    if (k <= 8) return gmres_multidot_k<8>(n, k, V, ld, w, Hj, s, ws, st);
    if (k <= 16) return gmres_multidot_k<16>(n, k, V, ld, w, Hj, s, ws, st);
    return gmres_multidot_k<kRedMaxVec>(n, k, V, ld, w, Hj, s, ws, st);
}

static int gmres_orth(int64_t n, int j, const double* V, int64_t ld, double* w, const double* Hj, GS* s, void* ws,
                      cudaStream_t st) {
    if (n == 0)
        return launch_scalar([=] __device__() {
            if (!s->cycle_done) s->sq = 0.0;
        }, st);
    const int k = j + 1;
    if (cgs_vec_ok(V, ld, w) && k <= kRedMaxVec) {
        const RedWorkspace rw = red_ws(ws);
#define WK_ORTH(KK)                                                                        \
    do {                                                                                   \
        gmres_orth_vec<KK><<<orth_grid(n), 256, 0, st>>>(n, k, V, ld, w, Hj, s, rw);        \
        WK_LAUNCH_CHECK();                                                                 \
        return 0;                                                                          \
    } while (0)
        if (k <= 2) WK_ORTH(2);
        if (k <= 4) WK_ORTH(4);
        if (k <= 8) WK_ORTH(8);
        if (k <= 16) WK_ORTH(16);
        WK_ORTH(kRedMaxVec);
#undef WK_ORTH
    }
    return launch_map_reduce(
        n,
        [=] __device__(int64_t i) {
            double wi = w[i];
            for (int q = 0; q <= j; ++q) wi = __dadd_rn(wi, -__dmul_rn(Hj[q], V[int64_t(q) * ld + i]));
            w[i] = wi;
            return __dmul_rn(wi, wi);
        },
        [=] __device__(double t) { s->sq = t; }, ws, &s->cycle_done, st);
}

static int gmres_givens(int j, double* H, double* cs_, double* sn_, double* g, GS* s, double* hist, cudaStream_t st,
                        double* sig = nullptr) {
    return launch_scalar([=] __device__() {
        if (s->cycle_done) return;
        const int m = s->restart;
        double* Hj = H + int64_t(j) * (m + 1);
        const double hn = sqrt(s->sq);
        s->hn = hn;
        if (sig != nullptr) sig[j + 1] = hn != 0.0 ? 1.0 / hn : 0.0;  // the scale of basis slot j + 1
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
    }, st);
}

static int gmres_next_basis(int64_t n, const double* w, double* Vn, GS* s, cudaStream_t st) {
    if (n > 0 && vmap_ok({w, Vn}))
        return launch_vmap<1, 1, 0>(
            n, VecArgs<1, 1>{{w}, {Vn}}, [=] __device__() { return s->hn; },
            [] __device__(double hn, const double(&in)[1], double(&out)[1], double(&)[1]) { out[0] = in[0] / hn; },
            NoEpi<1>{}, nullptr, &s->cycle_done, st);
    return launch_masked_map(n, [=] __device__(int64_t i) { Vn[i] = w[i] / s->hn; }, &s->cycle_done, st);
}

static int gmres_update_x(int64_t n, const double* V, int64_t ld, const double* H, const double* g, double* y, double* x,
                          GS* s, cudaStream_t st, const double* sig = nullptr) {
    WK_TRY(launch_scalar([=] __device__() {
        if (s->done) return;
        const int m = s->restart, jd = s->j_done;
        for (int i = jd - 1; i >= 0; --i) {
            double acc = g[i];
            for (int k = i + 1; k < jd; ++k) acc = __dadd_rn(acc, -__dmul_rn(H[i + int64_t(k) * (m + 1)], y[k]));
            y[i] = acc / H[i + int64_t(i) * (m + 1)];
        }
        // deferred normalisation: x += sum y_i v_i = sum (y_i sig_i) u_i
        if (sig != nullptr)
            for (int i = 0; i < jd; ++i) y[i] = __dmul_rn(y[i], sig[i]);
    }, st));
    return launch_masked_map(
        n,
        [=] __device__(int64_t i) {
            const int jd = s->j_done;
            double xi = x[i];
            for (int q = 0; q < jd; ++q) xi = __dadd_rn(xi, __dmul_rn(y[q], V[int64_t(q) * ld + i]));
            x[i] = xi;
        },
        &s->done, st);
}

static int gmres_residual(int64_t n, const double* b, const double* w, double* r, GS* s, void* ws, cudaStream_t st) {
    if (n == 0)
        return launch_scalar([=] __device__() {
            if (!s->done) s->sq = 0.0;
        }, st);
    if (vmap_ok({b, w, r}))
        return launch_vmap<2, 1, 1>(
            n, VecArgs<2, 1>{{b, w}, {r}}, NoScalars{},
            [] __device__(int, const double(&in)[2], double(&out)[1], double(&red)[1]) {
                const double ri = __dadd_rn(in[0], -in[1]);
                out[0] = ri;
                red[0] = __dmul_rn(ri, ri);
            },
            [=] __device__(double(&t)[1]) { s->sq = t[0]; }, ws, &s->done, st);
    return launch_map_reduce(
        n,
        [=] __device__(int64_t i) {
            const double ri = __dadd_rn(b[i], -w[i]);
            r[i] = ri;
            return __dmul_rn(ri, ri);
        },
        [=] __device__(double t) { s->sq = t; }, ws, &s->done, st);
}

static int gmres_restart(GS* s, double* hist, cudaStream_t st) {
    return launch_scalar([=] __device__() {
        if (s->done) return;
        const double bt = sqrt(s->sq);
        s->beta = bt;
        hist[s->iteration] = bt;
        s->done = !(s->iteration < s->max_iters && bt > s->threshold);
        s->cycle_done = s->done;
    }, st);
}

}  // namespace wk

using namespace wk;

extern "C" {

// ---- exported steps (distributed driver) --------------------------------------------

int wk_bicg_init(int64_t n, const double* b, double* x, double* r, double* rh, double* p, double* v,
                 wk_bicg_state* s, void* ws, wk_stream_t stream) {
    clear_error();
    return bicg_init(n, b, x, r, rh, p, v, s, ws, as_stream(stream));
}
int wk_bicg_init_finish(wk_bicg_state* s, double tol, int64_t max_iters, double* hist, wk_stream_t stream) {
    clear_error();
    return bicg_init_finish(s, tol, max_iters, hist, as_stream(stream));
}
int wk_bicg_rho(int64_t n, const double* rh, const double* r, wk_bicg_state* s, void* ws, wk_stream_t stream) {
    clear_error();
    return bicg_rho(n, rh, r, s, ws, as_stream(stream));
}
int wk_bicg_step_beta(wk_bicg_state* s, wk_stream_t stream) {
    clear_error();
    return bicg_step_beta(s, as_stream(stream));
}
int wk_bicg_update_p(int64_t n, const double* r, const double* v, double* p, wk_bicg_state* s, wk_stream_t stream) {
    clear_error();
    return bicg_update_p(n, r, v, p, s, as_stream(stream));
}
int wk_bicg_rv(int64_t n, const double* rh, const double* v, wk_bicg_state* s, void* ws, wk_stream_t stream) {
    clear_error();
    return bicg_rv(n, rh, v, s, ws, as_stream(stream));
}
int wk_bicg_step_alpha(wk_bicg_state* s, wk_stream_t stream) {
    clear_error();
    return bicg_step_alpha(s, as_stream(stream));
}
int wk_bicg_update_s(int64_t n, const double* r, const double* v, double* sv, wk_bicg_state* s, void* ws,
                     wk_stream_t stream) {
    clear_error();
    return bicg_update_s(n, r, v, sv, s, ws, as_stream(stream));
}
int wk_bicg_step_s(wk_bicg_state* s, double* hist, wk_stream_t stream) {
    clear_error();
    return bicg_step_s(s, hist, as_stream(stream));
}
int wk_bicg_half_x(int64_t n, const double* p, double* x, wk_bicg_state* s, void* ws, wk_stream_t stream) {
    clear_error();
    return bicg_half_x(n, p, x, s, ws, as_stream(stream));
}
int wk_bicg_tt_ts(int64_t n, const double* t, const double* sv, wk_bicg_state* s, void* ws, wk_stream_t stream) {
    clear_error();
    return bicg_tt_ts(n, t, sv, s, ws, as_stream(stream));
}
int wk_bicg_step_omega(wk_bicg_state* s, wk_stream_t stream) {
    clear_error();
    return bicg_step_omega(s, as_stream(stream));
}
int wk_bicg_update_xr(int64_t n, const double* p, const double* sv, const double* t, double* x, double* r,
                      wk_bicg_state* s, void* ws, wk_stream_t stream) {
    clear_error();
    return bicg_update_xr(n, p, sv, t, x, r, s, ws, as_stream(stream));
}
// Fused steps of wk_bicgstab_solve for the distributed solver: v = A p with
// r-hat.v (mode 1) / t = A s with t.t and t.s (mode 2) summed in the SpMV when
// the operand takes it (SELL-P(64), aligned), else SpMV + dot kernel; the x/r
// update with the next r-hat.r summed in the same pass (all-reduce rr and
// rho_next together afterwards), and the rho hand-over.
int wk_bicg_spmv_dots(const wk_matrix* A, const double* x, double* y, wk_bicg_state* s, const double* w, int32_t mode,
                      void* ws, wk_stream_t stream) {
    clear_error();
    WK_REQUIRE(mode == 1 || mode == 2, WK_ERR_INVALID, "mode must be 1 (r-hat.v) or 2 (t.t, t.s)");
    cudaStream_t st = as_stream(stream);
    const int rc = spmv_bicg_fused(A, x, y, s, w, mode, ws, st);
    if (rc != 1) return rc;
    WK_TRY(wk_spmv_masked(A, x, y, &s->done, stream));
    return mode == 1 ? bicg_rv(A->nrows, w, y, s, ws, st) : bicg_tt_ts(A->nrows, y, x, s, ws, st);
}
int wk_bicg_rho_first(int64_t n, const double* rh, const double* r, wk_bicg_state* s, void* ws, wk_stream_t stream) {
    clear_error();
    WK_REQUIRE(n > 0 && vmap_ok({rh, r}), WK_ERR_INVALID, "wk_bicg_rho_first needs 16-byte aligned vectors");
    return bicg_rho_first(n, rh, r, s, ws, as_stream(stream));
}
int wk_bicg_take_rho(wk_bicg_state* s, wk_stream_t stream) {
    clear_error();
    return bicg_take_rho(s, as_stream(stream));
}
int wk_bicg_update_xr_rho(int64_t n, const double* p, const double* sv, const double* t, const double* rh, double* x,
                          double* r, wk_bicg_state* s, void* ws, wk_stream_t stream) {
    clear_error();
    WK_REQUIRE(n > 0 && vmap_ok({p, sv, t, rh, x, r}), WK_ERR_INVALID,
               "wk_bicg_update_xr_rho needs 16-byte aligned vectors");
    return bicg_update_xr_rho(n, p, sv, t, rh, x, r, s, ws, as_stream(stream));
}
int wk_bicg_step_r(wk_bicg_state* s, double* hist, wk_stream_t stream) {
    clear_error();
    return bicg_step_r(s, hist, as_stream(stream));
}

int wk_gmres_init(int64_t n, const double* b, double* x, double* r, wk_gmres_state* s, void* ws, wk_stream_t stream) {
    clear_error();
    return gmres_init(n, b, x, r, s, ws, as_stream(stream));
}
int wk_gmres_init_finish(wk_gmres_state* s, double tol, int64_t max_iters, int32_t restart, double* hist,
                         wk_stream_t stream) {
    clear_error();
    WK_REQUIRE(restart >= 1 && restart <= kRedMaxVec - 1, WK_ERR_INVALID, "restart must be in [1, %d]",
               kRedMaxVec - 1);
    return gmres_init_finish(s, tol, max_iters, restart, hist, as_stream(stream));
}
int wk_gmres_cycle_start(int64_t n, const double* r, double* V0, double* g, wk_gmres_state* s, wk_stream_t stream) {
    clear_error();
    return gmres_cycle_start(n, r, V0, g, s, as_stream(stream));
}
int wk_gmres_multidot(int64_t n, int32_t j, const double* V, int64_t ld, const double* w, double* Hj,
                      wk_gmres_state* s, void* ws, wk_stream_t stream) {
    clear_error();
    return gmres_multidot(n, j, V, ld, w, Hj, s, ws, as_stream(stream));
}
int wk_gmres_orth(int64_t n, int32_t j, const double* V, int64_t ld, double* w, const double* Hj, wk_gmres_state* s,
                  void* ws, wk_stream_t stream) {
    clear_error();
    return gmres_orth(n, j, V, ld, w, Hj, s, ws, as_stream(stream));
}
int wk_gmres_givens(int32_t j, double* H, double* cs, double* sn, double* g, wk_gmres_state* s, double* hist,
                    wk_stream_t stream) {
    clear_error();
    return gmres_givens(j, H, cs, sn, g, s, hist, as_stream(stream));
}
// deferred normalisation (basis slot i holds u_i, v_i = sig[i] u_i; sig[0] = 1)
int wk_gmres_orth_scaled(int64_t n, int32_t j, const double* V, int64_t ld, double* w, double* Hj, const double* sig,
                         wk_gmres_state* s, void* ws, wk_stream_t stream) {
    clear_error();
    WK_REQUIRE(j >= 0 && j + 1 <= kRedMaxVec, WK_ERR_INVALID, "GMRES restart must be < %d", kRedMaxVec);
    WK_REQUIRE(cgs_vec_ok(V, ld, w), WK_ERR_INVALID, "wk_gmres_orth_scaled needs 16-byte aligned V, w and even ld");
    return gmres_orth_scaled(n, j, V, ld, w, Hj, sig, s, ws, as_stream(stream));
}
int wk_gmres_givens_scaled(int32_t j, double* H, double* cs, double* sn, double* g, double* sig, wk_gmres_state* s,
                           double* hist, wk_stream_t stream) {
    clear_error();
    return gmres_givens(j, H, cs, sn, g, s, hist, as_stream(stream), sig);
}
int wk_gmres_update_x_scaled(int64_t n, const double* V, int64_t ld, const double* H, const double* g, double* y,
                             double* x, const double* sig, wk_gmres_state* s, wk_stream_t stream) {
    clear_error();
    return gmres_update_x(n, V, ld, H, g, y, x, s, as_stream(stream), sig);
}
int wk_gmres_next_basis(int64_t n, const double* w, double* Vn, wk_gmres_state* s, wk_stream_t stream) {
    clear_error();
    return gmres_next_basis(n, w, Vn, s, as_stream(stream));
}
int wk_gmres_update_x(int64_t n, const double* V, int64_t ld, const double* H, const double* g, double* y, double* x,
                      wk_gmres_state* s, wk_stream_t stream) {
    clear_error();
    return gmres_update_x(n, V, ld, H, g, y, x, s, as_stream(stream));
}
int wk_gmres_residual(int64_t n, const double* b, const double* w, double* r, wk_gmres_state* s, void* ws,
                      wk_stream_t stream) {
    clear_error();
    return gmres_residual(n, b, w, r, s, ws, as_stream(stream));
}
int wk_gmres_restart(wk_gmres_state* s, double* hist, wk_stream_t stream) {
    clear_error();
    return gmres_restart(s, hist, as_stream(stream));
}

// ---- single-GPU solvers composed of the same steps (no all-reduce) -------------------

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
    BS* s = cv.take<BS>(1);
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
    WK_TRY(bicg_init(n, b, x, r, rh, p, v, s, red, st));
    WK_TRY(bicg_init_finish(s, tol, max_iters, hist, st));
    const int* done = &s->done;
    constexpr int kChunk = 10;
    // fused rho (rh.r summed in the x/r step of the previous iteration) when
    // every vector is 16-byte aligned
    const bool fused = n > 0 && vmap_ok({b, x, r, rh, p, v, sv, t});
    if (fused) WK_TRY(bicg_rho_first(n, rh, r, s, red, st));
    int rc = capture(g, [&](cudaStream_t cs) -> int {
        for (int i = 0; i < kChunk; ++i) {
            if (fused)
                WK_TRY(bicg_take_rho(s, cs));
            else
                WK_TRY(bicg_rho(n, rh, r, s, red, cs));
            WK_TRY(bicg_step_beta(s, cs));
            WK_TRY(bicg_update_p(n, r, v, p, s, cs));
            // v = A p with rv = r-hat.v fused into the SpMV when it can take it
            if (!fused || spmv_bicg_fused(A, p, v, s, rh, 1, red, cs) != 0) {
                WK_TRY(wk_spmv_masked(A, p, v, done, cs));
                WK_TRY(bicg_rv(n, rh, v, s, red, cs));
            }
            WK_TRY(bicg_step_alpha(s, cs));
            WK_TRY(bicg_update_s(n, r, v, sv, s, red, cs));
            WK_TRY(bicg_step_s(s, hist, cs));
            WK_TRY(bicg_half_x(n, p, x, s, red, cs));
            // t = A s with t.t and t.s fused into the SpMV when it can take them
            if (!fused || spmv_bicg_fused(A, sv, t, s, nullptr, 2, red, cs) != 0) {
                WK_TRY(wk_spmv_masked(A, sv, t, done, cs));
                WK_TRY(bicg_tt_ts(n, t, sv, s, red, cs));
            }
            WK_TRY(bicg_step_omega(s, cs));
            if (fused)
                WK_TRY(bicg_update_xr_rho(n, p, sv, t, rh, x, r, s, red, cs));
            else
                WK_TRY(bicg_update_xr(n, p, sv, t, x, r, s, red, cs));
            WK_TRY(bicg_step_r(s, hist, cs));
        }
        return 0;
    });
    if (rc) {
        cudaEventDestroy(ev);
        return rc;
    }
    BS h{};
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

int64_t wk_gmres_workspace_bytes(int64_t n, int32_t restart) {
    const int64_t m = restart;
    const int64_t vec = ceil_div(n * 8, 256) * 256;
    return 256 + red_ws_bytes() + 256 + (m + 1) * vec + 2 * vec + ceil_div((m + 1) * m * 8 + 5 * (m + 1) * 8, 256) * 256 +
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
    GS* s = cv.take<GS>(1);
    void* red = cv.take<char>(red_ws_bytes());
    const int64_t ld = ceil_div(n * 8, 256) * 256 / 8;
    double* V = cv.take<double>(ld * (m + 1));
    double* w = cv.take<double>(n);
    double* r = cv.take<double>(n);
    double* small = cv.take<double>((m + 1) * m + 5 * (m + 1));
    double* H = small;
    double* cs_ = H + (m + 1) * m;
    double* sn_ = cs_ + (m + 1);
    double* g = sn_ + (m + 1);
    double* y = g + (m + 1);
    double* sig = y + (m + 1);
    cudaStream_t user = as_stream(stream);
    GraphRunner gr;
    WK_CUDA(cudaStreamCreateWithFlags(&gr.cs, cudaStreamNonBlocking));
    cudaEvent_t ev;
    WK_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    WK_CUDA(cudaEventRecord(ev, user));
    WK_CUDA(cudaStreamWaitEvent(gr.cs, ev, 0));
    cudaStream_t st = gr.cs;
    WK_CUDA(cudaMemsetAsync(red, 0, size_t(red_ws_bytes()), st));
    WK_TRY(gmres_init(n, b, x, r, s, red, st));
    WK_TRY(gmres_init_finish(s, tol, max_iters, m, hist, st));
    const int* done = &s->done;
    const int* cdone = &s->cycle_done;
    // deferred normalisation (gmres_orth_scaled_vec) when the basis takes
    // 16-byte vector access; otherwise w, then v_{j+1} = w / h (next_basis)
    const bool scaled = n > 1 && cgs_vec_ok(V, ld, V);
    int rc = capture(gr, [&](cudaStream_t cs) -> int {
        WK_TRY(gmres_cycle_start(n, r, V, g, s, cs));
        if (scaled) WK_TRY(launch_scalar([=] __device__() { sig[0] = 1.0; }, cs));
        for (int j = 0; j < m; ++j) {
            double* Vj = V + int64_t(j) * ld;
            double* Hj = H + int64_t(j) * (m + 1);
            if (scaled) {
                double* z = V + int64_t(j + 1) * ld;
                WK_TRY(wk_spmv_masked(A, Vj, z, cdone, cs));
                WK_TRY(gmres_multidot(n, j, V, ld, z, Hj, s, red, cs));
                WK_TRY(gmres_orth_scaled(n, j, V, ld, z, Hj, sig, s, red, cs));
                WK_TRY(gmres_givens(j, H, cs_, sn_, g, s, hist, cs, sig));
                continue;
            }
            WK_TRY(wk_spmv_masked(A, Vj, w, cdone, cs));
            WK_TRY(gmres_multidot(n, j, V, ld, w, Hj, s, red, cs));
            WK_TRY(gmres_orth(n, j, V, ld, w, Hj, s, red, cs));
            WK_TRY(gmres_givens(j, H, cs_, sn_, g, s, hist, cs));
            if (j + 1 < m) WK_TRY(gmres_next_basis(n, w, V + int64_t(j + 1) * ld, s, cs));
        }
        WK_TRY(gmres_update_x(n, V, ld, H, g, y, x, s, cs, scaled ? sig : nullptr));
        WK_TRY(wk_spmv_masked(A, x, w, done, cs));
        WK_TRY(gmres_residual(n, b, w, r, s, red, cs));
        WK_TRY(gmres_restart(s, hist, cs));
        return 0;
    });
    if (rc) {
        cudaEventDestroy(ev);
        return rc;
    }
    GS h{};
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
    (void)cdone;
    return 0;
}

}  // extern "C"
