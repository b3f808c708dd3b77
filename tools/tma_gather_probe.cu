// Measurement scratch (not product): can the TMA engine's tile::gather4 move
// the random x gathers of the R-MAT SpMV off the L1TEX data pipe (one
// wavefront per random LDG gather: the bound of seg8_kernel)?
//
// Same R-MAT scale-24 COO as gather_probe.cu. x is described to the TMA as
// a 2-D tensor of n/2 rows x 2 doubles (16-byte rows); one gather4 fetches
// the 4 rows holding 4 entries' x values into shared memory. Kernels fold
// y_partial += v[k] * x[col[k]] over 8 consecutive entries per lane:
//   lsu      plain __ldg gathers (the gather_probe mode-0 baseline)
//   tma      all 8 gathers per lane through 2 gather4 per window, two
//            windows in flight per warp (shared-memory double buffer)
//   mix      entries 0..3 through one gather4, 4..7 through __ldg
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tma_gather_probe tools/tma_gather_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <thrust/device_ptr.h>
#include <thrust/sort.h>
#include <thrust/unique.h>

#include <cstdint>
#include <cstdio>

#define CK(x)                                                                 \
    do {                                                                      \
        cudaError_t e = (x);                                                  \
        if (e != cudaSuccess) {                                               \
            printf("%s: %s (%d)\n", #x, cudaGetErrorString(e), __LINE__);     \
            return 1;                                                         \
        }                                                                     \
    } while (0)

__device__ __forceinline__ uint64_t splitmix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void rmat_keys(int scale, int64_t m, uint64_t* keys) {
    int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= m) return;
    uint64_t r = 0, c = 0;
    for (int l = 0; l < scale; ++l) {
        double u = (splitmix(uint64_t(e) * 64 + l) >> 11) * (1.0 / 9007199254740992.0);
        int q = u < 0.57 ? 0 : (u < 0.76 ? 1 : (u < 0.95 ? 2 : 3));
        r = (r << 1) | (q >> 1);
        c = (c << 1) | (q & 1);
    }
    keys[e] = (r << 32) | c;
}

__global__ void split_keys(int64_t nnz, const uint64_t* keys, int* row, int* col, double* val) {
    int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= nnz) return;
    row[e] = int(keys[e] >> 32);
    col[e] = int(keys[e] & 0xffffffffu);
    val[e] = (splitmix(uint64_t(e) ^ 0x1234) >> 11) * (1.0 / 9007199254740992.0);
}

__device__ __forceinline__ uint32_t sa(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* tm, uint64_t* bar, int r0, int r1, int r2,
                                        int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(sa(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(sa(bar)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}

__device__ __forceinline__ void bar_init(uint64_t* b, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(n));
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t ph) {
    uint32_t done = 0;
    while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(sa(b)), "r"(ph)
            : "memory");
}

constexpr int kWarps = 12;  // 2 stages x 12 warps x 8 KB (each gather4 lands in its own 128-byte slot)

__global__ void __launch_bounds__(256) fold_lsu(int64_t nnz, const int* __restrict__ col,
                                                const double* __restrict__ val, const double* __restrict__ x,
                                                double* __restrict__ out) {
    const int64_t T = int64_t(gridDim.x) * blockDim.x;
    double acc = 0.0;
    for (int64_t kb = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 8; kb + 8 <= nnz; kb += T * 8) {
        const int4 c0 = __ldcs(reinterpret_cast<const int4*>(col + kb));
        const int4 c1 = __ldcs(reinterpret_cast<const int4*>(col + kb + 4));
        int c[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; u += 2) {
            double2 t = __ldcs(reinterpret_cast<const double2*>(val + kb + u));
            v[u] = t.x;
            v[u + 1] = t.y;
        }
        double g[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) g[u] = __ldg(x + c[u]);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, __dmul_rn(v[u], g[u]));
    }
    atomicAdd(out, acc);
}

// MODE 0: all 8 through TMA; MODE 1: 4 through TMA, 4 through LSU
template <int MODE>
__global__ void __launch_bounds__(kWarps * 32, 1) fold_tma(int64_t nnz, const int* __restrict__ col,
                                                           const double* __restrict__ val, const double* __restrict__ x,
                                                           const __grid_constant__ CUtensorMap tm,
                                                           double* __restrict__ out) {
    constexpr int NG = MODE == 0 ? 8 : 4;  // gathered through TMA per lane
    extern __shared__ __align__(128) double2 dsm[];  // [2][kWarps][32 * NG]
    __shared__ __align__(8) uint64_t bars[2][kWarps];
    // gather4 destinations must be 128-byte aligned: 8 double2 slots per gather4 (4 used)
    auto BUF = [&](int s_, int w_) { return dsm + (size_t(s_) * kWarps + w_) * 32 * NG * 2; };
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        bar_init(&bars[0][warp], 1);
        bar_init(&bars[1][warp], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int64_t nwin = nnz / 256;  // whole windows only (probe)
    const int64_t gw = int64_t(blockIdx.x) * kWarps + warp, nw = int64_t(gridDim.x) * kWarps;
    double acc = 0.0;
    double vp[8];
    int cp[8];
    uint32_t ph[2] = {0u, 0u};
    auto issue = [&](int64_t w, int s, double (&v)[8], int (&c)[8]) {
        const int64_t kb = w * 256 + 8 * lane;
        const int4 c0 = __ldcs(reinterpret_cast<const int4*>(col + kb));
        const int4 c1 = __ldcs(reinterpret_cast<const int4*>(col + kb + 4));
        c[0] = c0.x, c[1] = c0.y, c[2] = c0.z, c[3] = c0.w, c[4] = c1.x, c[5] = c1.y, c[6] = c1.z, c[7] = c1.w;
#pragma unroll
        for (int u = 0; u < 8; u += 2) {
            double2 t = __ldcs(reinterpret_cast<const double2*>(val + kb + u));
            v[u] = t.x;
            v[u + 1] = t.y;
        }
        if (lane == 0) bar_expect(&bars[s][warp], 32u * NG * 16u);
        __syncwarp();
        double2* d = BUF(s, warp) + lane * NG * 2;
        gather4(d, &tm, &bars[s][warp], c[0] >> 1, c[1] >> 1, c[2] >> 1, c[3] >> 1);
        if (NG == 8) gather4(d + 8, &tm, &bars[s][warp], c[4] >> 1, c[5] >> 1, c[6] >> 1, c[7] >> 1);
    };
    auto fold = [&](int s, const double (&v)[8], const int (&c)[8]) {
        double g[8];
        if (NG == 4) {
#pragma unroll
            for (int u = 4; u < 8; ++u) g[u] = __ldg(x + c[u]);
        }
        bar_wait(&bars[s][warp], ph[s]);
        ph[s] ^= 1u;
        const double2* d = BUF(s, warp) + lane * NG * 2;
#pragma unroll
        for (int u = 0; u < NG; ++u) {
            const double2 t = d[(u >> 2) * 8 + (u & 3)];
            g[u] = (c[u] & 1) ? t.y : t.x;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, __dmul_rn(v[u], g[u]));
        __syncwarp();  // every lane has read its stage before it is refilled
    };
    int s = 0;
    int64_t w = gw;
    if (w < nwin) issue(w, 0, vp, cp);
    for (; w < nwin; w += nw) {
        double vn[8];
        int cn[8];
        const bool more = w + nw < nwin;
        if (more) issue(w + nw, s ^ 1, vn, cn);
        fold(s, vp, cp);
        if (more) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                vp[u] = vn[u];
                cp[u] = cn[u];
            }
        }
        s ^= 1;
    }
    atomicAdd(out, acc);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int scale = 24;
    const int64_t n = int64_t(1) << scale, m = n * 16;
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint64_t* keys;
    CK(cudaMalloc(&keys, m * 8));
    rmat_keys<<<(m + 255) / 256, 256>>>(scale, m, keys);
    CK(cudaDeviceSynchronize());
    thrust::sort(thrust::device_ptr<uint64_t>(keys), thrust::device_ptr<uint64_t>(keys + m));
    int64_t nnz = thrust::unique(thrust::device_ptr<uint64_t>(keys), thrust::device_ptr<uint64_t>(keys + m)) -
                  thrust::device_ptr<uint64_t>(keys);
    nnz &= ~int64_t(255);
    int *row, *col;
    double *val, *x, *out;
    CK(cudaMalloc(&row, nnz * 4));
    CK(cudaMalloc(&col, nnz * 4));
    CK(cudaMalloc(&val, nnz * 8));
    CK(cudaMalloc(&x, n * 8));
    CK(cudaMalloc(&out, 2048 * 8));
    split_keys<<<(nnz + 255) / 256, 256>>>(nnz, keys, row, col, val);
    CK(cudaMemcpy(x, val, n * 8, cudaMemcpyDeviceToDevice));
    CK(cudaFree(keys));

    EncodeFn encode = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q));
    CUtensorMap tm;
    cuuint64_t dims[2] = {2, cuuint64_t(n / 2)};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {2, 1};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d, nnz %lld\n", int(r), (long long)nnz);
    if (r != CUDA_SUCCESS) return 1;

    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double ref = 0;
    auto timeit = [&](const char* name, auto launch) {
        for (int i = 0; i < 3; ++i) launch();
        cudaEventRecord(a);
        for (int i = 0; i < 10; ++i) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 10;
        cudaMemset(out, 0, 8);
        launch();
        double s = 0;
        cudaMemcpy(&s, out, 8, cudaMemcpyDeviceToHost);
        cudaError_t e = cudaGetLastError();
        printf("%-28s %.4f ms  %.1f Ggather/s  checksum %.6e %s\n", name, ms, nnz / ms / 1e6, s,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
        (void)ref;
    };
    timeit("lsu 4 blocks/SM", [&] { fold_lsu<<<sms * 4, 256>>>(nnz, col, val, x, out); });
    timeit("lsu 8 blocks/SM", [&] { fold_lsu<<<sms * 8, 256>>>(nnz, col, val, x, out); });
    const int sm0 = 2 * kWarps * 32 * 8 * 16 * 2, sm1 = sm0 / 2;
    CK(cudaFuncSetAttribute(fold_tma<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm0));
    CK(cudaFuncSetAttribute(fold_tma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm1));
    timeit("tma gather4 (all 8)", [&] { fold_tma<0><<<sms, kWarps * 32, sm0>>>(nnz, col, val, x, tm, out); });
    timeit("mix (4 tma + 4 lsu)", [&] { fold_tma<1><<<sms, kWarps * 32, sm1>>>(nnz, col, val, x, tm, out); });
    return 0;
}
