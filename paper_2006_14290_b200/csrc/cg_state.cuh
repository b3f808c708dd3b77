// CG scalar steps on the device (kernels.py:315-330), shared by the reduction
// epilogues of the fused kernels and by the 1-thread step kernels of the
// distributed path.
#pragma once

#include "common.cuh"
#include "peer_dev.cuh"

namespace wk {

constexpr int kReplaceEvery = 50;  // kernels.py:322

__device__ __forceinline__ void cg_alpha_step(wk_cg_state* s) {
    if (s->done) return;
    const double pq = s->pq;
    if (pq <= 0.0) {  // kernels.py:317-318 (NaN falls through, as in Python)
        s->breakdown = 1;
        s->done = 1;
        s->iteration += 1;
        return;
    }
    s->alpha = s->rho / pq;
    s->iteration += 1;
}

__device__ __forceinline__ void cg_beta_step(wk_cg_state* s, double* hist) {
    if (s->done) return;
    const double rr = s->rr;
    const double rn = sqrt(rr);
    hist[s->iteration] = rn;
    s->beta = rr / s->rho;
    s->rho = rr;
    s->done = !(s->iteration < s->max_iters && rn > s->threshold);
}

__device__ __forceinline__ bool cg_replacing(const wk_cg_state* s) { return s->iteration % kReplaceEvery == 0; }

// Epilogue target of an SpMV with a fused p.q reduction (CG q = A p):
// state->pq = sum over the rank's rows of p[r] * q[r]; with `finalize` the
// alpha step runs in the same epilogue (single GPU), otherwise the caller
// all-reduces state->pq first (distributed).
struct DotEpilogue {
    double* partials;   // reduction workspace (reduce.cuh RedWorkspace)
    unsigned* ticket;
    wk_cg_state* state;
    int finalize;
    PeerCtx* peer;      // non-null: push the local p.q to every rank (fused all-reduce)
    const PeerHalo* halo;  // non-null: wait for the pushed halo of x before the first gather
};

// Epilogue of an SpMV with BiCGSTAB's dots fused (wk_bicgstab_solve):
// mode 1 (v = A p): rv = sum w[r] * y[r] with w = r-hat;
// mode 2 (t = A s): tt = sum y[r]^2, ts = sum y[r] * x[r] (x = s).
struct BicgEpilogue {
    double* partials;
    unsigned* ticket;
    wk_bicg_state* state;
    const double* w;
    int mode;
};

}  // namespace wk
