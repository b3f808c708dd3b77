// Deterministic device-wide reductions and scans (header-only templates).
//
// Reductions: a fixed grid (a function of n and the SM count only) folds its
// grid-stride slice per thread, reduces per block with warp butterflies
// (reduce_subwarp, kernels.py:35-49), writes one partial per block; the last
// block to arrive (atomic ticket) folds the partials in block order. The same
// input on the same GPU therefore always gives the same bits. The summation
// order differs from OpenBLAS ddot (as the reference's own ddot differs
// between thread counts), so solver parity uses the residual tolerance of
// BASELINE.md §2.
#pragma once

#include <initializer_list>

#include "common.cuh"

namespace wk {

constexpr int kRedThreads = 256;
constexpr int kRedMaxBlocks = 1024;
constexpr int kRedMaxVec = 32;  // multidot width

struct RedWorkspace {
    double* partials;  // kRedMaxVec * kRedMaxBlocks
    unsigned* ticket;
};

inline RedWorkspace red_ws(void* ws) {
    RedWorkspace w;
    w.partials = reinterpret_cast<double*>(ws);
    w.ticket = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(ws) + sizeof(double) * kRedMaxVec * kRedMaxBlocks);
    return w;
}

inline int64_t red_ws_bytes() { return int64_t(sizeof(double)) * kRedMaxVec * kRedMaxBlocks + 256; }

inline int red_grid(int64_t n) {
    int64_t g = ceil_div(n, int64_t(kRedThreads) * 8);
    const int64_t cap = int64_t(sm_count()) * 4;
    if (g > cap) g = cap;
    if (g > kRedMaxBlocks) g = kRedMaxBlocks;
    if (g < 1) g = 1;
    return int(g);
}

// Block-level: reduce `v`, publish the partial, and return true in the (single)
// last-arriving block, where `total` (thread 0) holds the grid total.
template <int kThreads = kRedThreads>
__device__ __forceinline__ bool grid_reduce_last(double v, RedWorkspace ws, double& total) {
    __shared__ double red[kThreads / 32];
    __shared__ bool is_last;
    const double bsum = block_sum<kThreads>(v, red);
    if (threadIdx.x == 0) {
        ws.partials[blockIdx.x] = bsum;
        __threadfence();
        const unsigned t = atomicAdd(ws.ticket, 1u);
        is_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!is_last) return false;
    __threadfence();
    double acc = 0.0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += kThreads) acc += __ldcg(ws.partials + b);
    __syncthreads();  // `red` reuse
    total = block_sum<kThreads>(acc, red);
    if (threadIdx.x == 0) *ws.ticket = 0;
    return true;
}

// Two values, any block size: partial slot v of block b at partials[v *
// kRedMaxBlocks + b]; returns true in the last-arriving block (thread 0 holds
// both grid totals).
template <int kThreads>
__device__ __forceinline__ bool grid_reduce_last2(double v0, double v1, RedWorkspace ws, double& t0, double& t1) {
    __shared__ double red[kThreads / 32];
    __shared__ bool is_last;
    const double b0 = block_sum<kThreads>(v0, red);
    __syncthreads();  // `red` reuse
    const double b1 = block_sum<kThreads>(v1, red);
    if (threadIdx.x == 0) {
        ws.partials[blockIdx.x] = b0;
        ws.partials[kRedMaxBlocks + blockIdx.x] = b1;
        __threadfence();
        is_last = atomicAdd(ws.ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!is_last) return false;
    __threadfence();
    double a0 = 0.0, a1 = 0.0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += kThreads) {
        a0 += __ldcg(ws.partials + b);
        a1 += __ldcg(ws.partials + kRedMaxBlocks + b);
    }
    __syncthreads();
    t0 = block_sum<kThreads>(a0, red);
    __syncthreads();
    t1 = block_sum<kThreads>(a1, red);
    if (threadIdx.x == 0) *ws.ticket = 0;
    return true;
}

// N-value variant: f(i, acc) adds into acc[0..N-1]; partial slot v of block b
// lives at partials[v * kRedMaxBlocks + b]. Returns true in the last block,
// where total[] (thread 0) holds the grid totals.
template <int N>
__device__ __forceinline__ bool grid_reduce_last_n(const double (&v)[N], RedWorkspace ws, double (&total)[N]) {
    __shared__ double red[kRedThreads / 32];
    __shared__ bool is_last;
#pragma unroll
    for (int q = 0; q < N; ++q) {
        const double bsum = block_sum<kRedThreads>(v[q], red);
        if (threadIdx.x == 0) ws.partials[q * kRedMaxBlocks + blockIdx.x] = bsum;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        __threadfence();
        is_last = atomicAdd(ws.ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!is_last) return false;
    __threadfence();
#pragma unroll
    for (int q = 0; q < N; ++q) {
        double acc = 0.0;
        for (unsigned b = threadIdx.x; b < gridDim.x; b += kRedThreads) acc += __ldcg(ws.partials + q * kRedMaxBlocks + b);
        total[q] = block_sum<kRedThreads>(acc, red);
        __syncthreads();
    }
    if (threadIdx.x == 0) *ws.ticket = 0;
    return true;
}

template <int N, typename F, typename Epi>
__global__ void __launch_bounds__(kRedThreads)
map_reduce_n_kernel(int64_t n, F f, Epi epi, RedWorkspace ws, const int* __restrict__ skip) {
    if (skip != nullptr && *skip) return;
    double acc[N];
#pragma unroll
    for (int q = 0; q < N; ++q) acc[q] = 0.0;
    const int64_t stride = int64_t(gridDim.x) * kRedThreads;
    for (int64_t i = int64_t(blockIdx.x) * kRedThreads + threadIdx.x; i < n; i += stride) f(i, acc);
    double total[N];
    if (grid_reduce_last_n<N>(acc, ws, total) && threadIdx.x == 0) epi(total);
}

template <int N, typename F, typename Epi>
int launch_map_reduce_n(int64_t n, F f, Epi epi, void* ws, const int* skip, cudaStream_t st) {
    map_reduce_n_kernel<N><<<red_grid(n), kRedThreads, 0, st>>>(n, f, epi, red_ws(ws), skip);
    WK_LAUNCH_CHECK();
    return 0;
}

// Generic map-reduce: total = sum_i f(i); Epi(total) runs on thread 0 of the
// last block. Skips entirely when *skip != 0.
template <typename F, typename Epi>
__global__ void __launch_bounds__(kRedThreads)
map_reduce_kernel(int64_t n, F f, Epi epi, RedWorkspace ws, const int* __restrict__ skip) {
    if (skip != nullptr && *skip) return;
    double acc = 0.0;
    const int64_t stride = int64_t(gridDim.x) * kRedThreads;
    for (int64_t i = int64_t(blockIdx.x) * kRedThreads + threadIdx.x; i < n; i += stride) acc += f(i);
    double total = 0.0;
    if (grid_reduce_last(acc, ws, total) && threadIdx.x == 0) epi(total);
}

template <typename F, typename Epi>
int launch_map_reduce(int64_t n, F f, Epi epi, void* ws, const int* skip, cudaStream_t st) {
    map_reduce_kernel<<<red_grid(n), kRedThreads, 0, st>>>(n, f, epi, red_ws(ws), skip);
    WK_LAUNCH_CHECK();
    return 0;
}

// ---------------------------------------------------------------------------
// Vectorised element-wise step with optional fused reductions (the Krylov
// BLAS-1 updates): NIN input vectors, NOUT output vectors (may alias inputs:
// every load of an iteration precedes its stores), NRED sums. Each thread
// handles U double2 pairs per iteration (k, k + T, ...; U = 4 for one input,
// 2 otherwise), so 2U elements of every vector are in flight per thread; the solver scalars are read ONCE per
// thread by `pro()` instead of once per element (a scalar read through the
// state pointer cannot be hoisted past the vector stores). Per-thread sums run
// in a fixed element order and are folded by grid_reduce_last_n: deterministic.
//   f(c, const double (&in)[NIN], double (&out)[NOUT], double (&red)[NRED])
// All vectors 16-byte aligned (vmap_ok); the callers fall back to the scalar
// map_reduce kernels otherwise.
// ---------------------------------------------------------------------------
template <int NIN, int NOUT>
struct VecArgs {
    const double* in[NIN > 0 ? NIN : 1];
    double* out[NOUT > 0 ? NOUT : 1];
};

inline int vmap_grid(int64_t n) {
    int64_t g = ceil_div(ceil_div(n, 2), int64_t(kRedThreads) * 2);
    const int64_t cap = int64_t(sm_count()) * 8;
    if (g > cap) g = cap;
    if (g > kRedMaxBlocks) g = kRedMaxBlocks;
    return int(g < 1 ? 1 : g);
}

// kRunIf: run only while *skip != 0 (instead of skipping then)
// (kRedThreads, 4): at most 64 registers, so the grid's 8 blocks per SM are
// not cut to 3 by the one-in / one-out instances (GMRES basis scaling: 80
// registers, 4.8 TB/s)
template <int NIN, int NOUT, int NRED, bool kRunIf, typename Pro, typename F, typename Epi>
__global__ void __launch_bounds__(kRedThreads, 4)
vmap_kernel(int64_t n, VecArgs<NIN, NOUT> a, Pro pro, F f, Epi epi, RedWorkspace ws, const int* __restrict__ skip) {
    constexpr int NR = NRED > 0 ? NRED : 1, NO = NOUT > 0 ? NOUT : 1;
    if (skip != nullptr && (kRunIf ? *skip == 0 : *skip != 0)) return;
    const auto c = pro();
    double acc[NR];
#pragma unroll
    for (int q = 0; q < NR; ++q) acc[q] = 0.0;
    auto elem = [&](const double (&in)[NIN > 0 ? NIN : 1], double (&out)[NO]) {
        double red[NR];
        f(c, in, out, red);
#pragma unroll
        for (int q = 0; q < NRED; ++q) acc[q] += red[q];
    };
    // U pairs of every vector in flight per thread: 4 for one input (a copy-
    // shaped step needs the bytes in flight: 2 pairs ran the GMRES basis
    // scaling at 4.9 TB/s), 2 otherwise
    constexpr int U = NIN <= 1 ? 4 : 2;
    constexpr int NI = NIN > 0 ? NIN : 1;
    const int64_t np = n >> 1, T = int64_t(gridDim.x) * kRedThreads;
    for (int64_t k = int64_t(blockIdx.x) * kRedThreads + threadIdx.x; k < np; k += U * T) {
        double2 v[U][NI];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int q = 0; q < NIN; ++q)
                v[u][q] = k + u * T < np ? reinterpret_cast<const double2*>(a.in[q])[k + u * T]
                                         : make_double2(0.0, 0.0);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (u > 0 && k + u * T >= np) break;
            double i0[NI], i1[NI], o0[NO], o1[NO];
#pragma unroll
            for (int q = 0; q < NIN; ++q) {
                i0[q] = v[u][q].x;
                i1[q] = v[u][q].y;
            }
            elem(i0, o0);
            elem(i1, o1);
#pragma unroll
            for (int q = 0; q < NOUT; ++q)
                reinterpret_cast<double2*>(a.out[q])[k + u * T] = make_double2(o0[q], o1[q]);
        }
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        double i0[NIN > 0 ? NIN : 1], o0[NO];
#pragma unroll
        for (int q = 0; q < NIN; ++q) i0[q] = a.in[q][n - 1];
        elem(i0, o0);
#pragma unroll
        for (int q = 0; q < NOUT; ++q) a.out[q][n - 1] = o0[q];
    }
    if (NRED > 0) {
        double total[NR];
        if (grid_reduce_last_n<NR>(acc, ws, total) && threadIdx.x == 0) epi(total);
    }
}

inline bool vmap_ok(std::initializer_list<const void*> ptrs) {
    for (const void* p : ptrs)
        if (reinterpret_cast<uintptr_t>(p) & 15) return false;
    return true;
}

template <int NIN, int NOUT, int NRED, bool kRunIf = false, typename Pro, typename F, typename Epi>
int launch_vmap(int64_t n, VecArgs<NIN, NOUT> a, Pro pro, F f, Epi epi, void* ws, const int* skip, cudaStream_t st) {
    vmap_kernel<NIN, NOUT, NRED, kRunIf><<<vmap_grid(n), kRedThreads, 0, st>>>(n, a, pro, f, epi, red_ws(ws), skip);
    WK_LAUNCH_CHECK();
    return 0;
}

// ---------------------------------------------------------------------------
// Exclusive scan, three passes over tiles of kScanTile elements:
//   1. tile sums  2. single-block scan of tile sums  3. tile-local scan + base.
// Input is produced by a functor `f(i)` (i < n) so callers scan derived
// quantities (row lengths, slice widths, flags) without materialising them.
// out[0] = 0, out[i+1] = out[i] + f(i).
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int64_t kScanTile = int64_t(kScanThreads) * kScanItems;

inline int64_t scan_ws_bytes(int64_t n) { return (ceil_div(n, kScanTile) + 2) * 8 + 256; }

template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* smem /* kScanThreads/32 + 1 */, T& block_total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T incl = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const T o = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += o;
    }
    if (lane == 31) smem[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        T w = lane < kScanThreads / 32 ? smem[lane] : T(0);
        T wi = w;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const T o = __shfl_up_sync(0xffffffffu, wi, d);
            if (lane >= d) wi += o;
        }
        if (lane < kScanThreads / 32) smem[lane] = wi - w;  // exclusive warp offsets
        if (lane == kScanThreads / 32 - 1) smem[kScanThreads / 32] = wi;
    }
    __syncthreads();
    block_total = smem[kScanThreads / 32];
    const T r = smem[wid] + incl - v;
    __syncthreads();
    return r;
}

template <typename F>
__global__ void __launch_bounds__(kScanThreads) scan_tile_sums(int64_t n, F f, int64_t* __restrict__ sums) {
    __shared__ int64_t smem[kScanThreads / 32 + 1];
    const int64_t base = int64_t(blockIdx.x) * kScanTile + int64_t(threadIdx.x) * kScanItems;
    int64_t s = 0;
#pragma unroll
    for (int u = 0; u < kScanItems; ++u)
        if (base + u < n) s += int64_t(f(base + u));
    int64_t tot;
    block_exclusive_scan<int64_t>(s, smem, tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanThreads) scan_tile_sums_exclusive(int64_t ntiles, int64_t* __restrict__ sums);

template <typename F, typename OutT>
__global__ void __launch_bounds__(kScanThreads)
scan_tiles(int64_t n, F f, const int64_t* __restrict__ tile_base, OutT* __restrict__ out) {
    __shared__ int64_t smem[kScanThreads / 32 + 1];
    const int64_t base = int64_t(blockIdx.x) * kScanTile + int64_t(threadIdx.x) * kScanItems;
    int64_t v[kScanItems];
    int64_t s = 0;
#pragma unroll
    for (int u = 0; u < kScanItems; ++u) {
        v[u] = (base + u < n) ? int64_t(f(base + u)) : 0;
        s += v[u];
    }
    int64_t tot;
    int64_t run = block_exclusive_scan<int64_t>(s, smem, tot) + tile_base[blockIdx.x];
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = OutT(0);
#pragma unroll
    for (int u = 0; u < kScanItems; ++u) {
        run += v[u];
        if (base + u < n) out[base + u + 1] = OutT(run);
    }
}

int scan_tile_sums_exclusive_launch(int64_t ntiles, int64_t* sums, cudaStream_t st);

template <typename F, typename OutT>
int exclusive_scan(int64_t n, F f, OutT* out, void* ws, cudaStream_t st) {
    if (n == 0) {
        WK_CUDA(cudaMemsetAsync(out, 0, sizeof(OutT), st));
        return 0;
    }
    const int64_t ntiles = ceil_div(n, kScanTile);
    int64_t* sums = reinterpret_cast<int64_t*>(ws);
    scan_tile_sums<<<(unsigned)ntiles, kScanThreads, 0, st>>>(n, f, sums);
    WK_LAUNCH_CHECK();
    int rc = scan_tile_sums_exclusive_launch(ntiles, sums, st);
    if (rc) return rc;
    scan_tiles<<<(unsigned)ntiles, kScanThreads, 0, st>>>(n, f, sums, out);
    WK_LAUNCH_CHECK();
    return 0;
}

}  // namespace wk
