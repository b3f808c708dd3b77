// BLAS-1 kernels: dot / norm2 (deterministic two-level reduction with
// subwarp butterflies), axpy-style updates (separately rounded like numpy's
// `x + alpha * p`, kernels.py:320-329), batched dots for classical
// Gram-Schmidt, halo gather, and the device-wide scan support.
#include "reduce.cuh"

namespace wk {

__global__ void __launch_bounds__(kScanThreads) scan_tile_sums_exclusive(int64_t ntiles, int64_t* __restrict__ sums) {
    __shared__ int64_t smem[kScanThreads / 32 + 1];
    int64_t carry = 0;
    for (int64_t base = 0; base < ntiles; base += kScanTile) {
        int64_t v[kScanItems];
        int64_t s = 0;
        const int64_t b = base + int64_t(threadIdx.x) * kScanItems;
#pragma unroll
        for (int u = 0; u < kScanItems; ++u) {
            v[u] = (b + u < ntiles) ? sums[b + u] : 0;
            s += v[u];
        }
        int64_t tot;
        int64_t run = block_exclusive_scan<int64_t>(s, smem, tot) + carry;
#pragma unroll
        for (int u = 0; u < kScanItems; ++u) {
            if (b + u < ntiles) sums[b + u] = run;
            run += v[u];
        }
        carry += tot;
        __syncthreads();
    }
}

int scan_tile_sums_exclusive_launch(int64_t ntiles, int64_t* sums, cudaStream_t st) {
    scan_tile_sums_exclusive<<<1, kScanThreads, 0, st>>>(ntiles, sums);
    WK_LAUNCH_CHECK();
    return 0;
}

// result[i] = V_i . w for i < k (k <= kRedMaxVec); w is read once per element.
template <int K>
__global__ void __launch_bounds__(kRedThreads)
multidot_kernel(int64_t n, int k, const double* __restrict__ V, int64_t ld, const double* __restrict__ w,
                double* __restrict__ result, RedWorkspace ws) {
    double acc[K];
#pragma unroll
    for (int i = 0; i < K; ++i) acc[i] = 0.0;
    const int64_t stride = int64_t(gridDim.x) * kRedThreads;
    for (int64_t j = int64_t(blockIdx.x) * kRedThreads + threadIdx.x; j < n; j += stride) {
        const double wj = __ldcs(w + j);
#pragma unroll
        for (int i = 0; i < K; ++i)
            if (i < k) acc[i] += __dmul_rn(__ldcs(V + i * ld + j), wj);
    }
    __shared__ double red[kRedThreads / 32];
    __shared__ bool is_last;
    for (int i = 0; i < k; ++i) {
        const double b = block_sum<kRedThreads>(acc[i], red);
        if (threadIdx.x == 0) ws.partials[int64_t(i) * kRedMaxBlocks + blockIdx.x] = b;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        __threadfence();
        is_last = atomicAdd(ws.ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    for (int i = 0; i < k; ++i) {
        double a = 0.0;
        for (unsigned b = threadIdx.x; b < gridDim.x; b += kRedThreads)
            a += __ldcg(ws.partials + int64_t(i) * kRedMaxBlocks + b);
        const double t = block_sum<kRedThreads>(a, red);
        if (threadIdx.x == 0) result[i] = t;
        __syncthreads();
    }
    if (threadIdx.x == 0) *ws.ticket = 0;
}

template <typename F>
__global__ void __launch_bounds__(256) elementwise_kernel(int64_t n, F f) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) f(i);
}

template <typename F>
int launch_elementwise(int64_t n, F f, cudaStream_t st) {
    if (n == 0) return 0;
    int64_t blocks = ceil_div(n, 256);
    const int64_t cap = int64_t(sm_count()) * 16;
    if (blocks > cap) blocks = cap;
    elementwise_kernel<<<(unsigned)blocks, 256, 0, st>>>(n, f);
    WK_LAUNCH_CHECK();
    return 0;
}

}  // namespace wk

using namespace wk;

extern "C" {

int64_t wk_reduce_workspace_bytes(void) { return red_ws_bytes(); }

int64_t wk_scan_workspace_bytes(int64_t n) { return scan_ws_bytes(n); }

int wk_exclusive_scan_i64(int64_t n, const int64_t* in, int64_t* out, void* ws, wk_stream_t stream) {
    clear_error();
    return exclusive_scan(n, [in] __device__(int64_t i) { return in[i]; }, out, ws, as_stream(stream));
}

int wk_dot_f64(int64_t n, const double* x, const double* y, double* result, void* workspace, wk_stream_t stream) {
    clear_error();
    if (n == 0) {
        WK_CUDA(cudaMemsetAsync(result, 0, sizeof(double), as_stream(stream)));
        return 0;
    }
    return launch_map_reduce(
        n, [x, y] __device__(int64_t i) { return __dmul_rn(__ldcs(x + i), __ldcs(y + i)); },
        [result] __device__(double t) { *result = t; }, workspace, nullptr, as_stream(stream));
}

int wk_norm2_f64(int64_t n, const double* x, double* result, void* workspace, wk_stream_t stream) {
    clear_error();
    if (n == 0) {
        WK_CUDA(cudaMemsetAsync(result, 0, sizeof(double), as_stream(stream)));
        return 0;
    }
    return launch_map_reduce(
        n, [x] __device__(int64_t i) { const double v = __ldcs(x + i); return __dmul_rn(v, v); },
        [result] __device__(double t) { *result = sqrt(t); }, workspace, nullptr, as_stream(stream));
}

int wk_axpy_f64(int64_t n, double alpha, const double* x, double* y, wk_stream_t stream) {
    clear_error();
    return launch_elementwise(
        n, [=] __device__(int64_t i) { y[i] = __dadd_rn(y[i], __dmul_rn(alpha, x[i])); }, as_stream(stream));
}

int wk_xpby_f64(int64_t n, const double* x, double beta, double* y, wk_stream_t stream) {
    clear_error();
    return launch_elementwise(
        n, [=] __device__(int64_t i) { y[i] = __dadd_rn(x[i], __dmul_rn(beta, y[i])); }, as_stream(stream));
}

int wk_scal_f64(int64_t n, double alpha, double* x, wk_stream_t stream) {
    clear_error();
    return launch_elementwise(n, [=] __device__(int64_t i) { x[i] = __dmul_rn(alpha, x[i]); }, as_stream(stream));
}

int wk_gather_f64(int64_t n, const int32_t* idx, const double* src, double* dst, wk_stream_t stream) {
    clear_error();
    return launch_elementwise(n, [=] __device__(int64_t i) { dst[i] = src[idx[i]]; }, as_stream(stream));
}

int wk_multidot_f64(int64_t n, int64_t k, const double* V, int64_t ld, const double* w, double* result,
                    void* workspace, wk_stream_t stream) {
    clear_error();
    WK_REQUIRE(k >= 0 && k <= kRedMaxVec, WK_ERR_INVALID, "multidot supports up to %d vectors", kRedMaxVec);
    cudaStream_t st = as_stream(stream);
    if (k == 0) return 0;
    if (n == 0) {
        WK_CUDA(cudaMemsetAsync(result, 0, sizeof(double) * size_t(k), st));
        return 0;
    }
    const int g = red_grid(n);
    if (k <= 8)
        multidot_kernel<8><<<g, kRedThreads, 0, st>>>(n, int(k), V, ld, w, result, red_ws(workspace));
    else if (k <= 16)
        multidot_kernel<16><<<g, kRedThreads, 0, st>>>(n, int(k), V, ld, w, result, red_ws(workspace));
    else
        multidot_kernel<32><<<g, kRedThreads, 0, st>>>(n, int(k), V, ld, w, result, red_ws(workspace));
    WK_LAUNCH_CHECK();
    return 0;
}

}  // extern "C"
