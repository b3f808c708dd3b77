// Microbenchmark (measurement scratch, not product): the x-gather paths for
// the R-MAT SpMV. Builds an R-MAT scale-24 edge-factor-16 COO (Graph500
// parameters, sorted by (row, col)), then times a COO-shaped fold
// y_partial += v[k] * x[col[k]] (8 consecutive entries per lane, streaming
// row/col/val loads as in seg8_kernel) with different instructions for the
// x gather:
//   0 ld.global.nc (__ldg, L1-allocating)    1 ld.global.cg (L2 only)
//   2 tex1Dfetch<int2> (texture pipe)         3 entries alternate 0 / 2
//   4 ld.global.nc.L1::no_allocate            5 ld.global.ca (L1 allocate, coherent)
// ncu's l1tex__data_pipe_lsu_wavefronts showed the LSU data pipe at 87% on
// the production kernel: one wavefront per random gather.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_probe tools/gather_probe.cu
#include <cuda_runtime.h>
#include <thrust/device_ptr.h>
#include <thrust/sort.h>
#include <thrust/unique.h>
#include <thrust/sequence.h>
#include <thrust/functional.h>

#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e = (x);                                                               \
        if (e != cudaSuccess) {                                                            \
            printf("%s: %s (%d)\n", #x, cudaGetErrorString(e), __LINE__);                  \
            return 1;                                                                      \
        }                                                                                  \
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

template <int MODE>
__device__ __forceinline__ double gx(const double* __restrict__ x, cudaTextureObject_t tx, int c, int u) {
    if (MODE == 0) return __ldg(x + c);
    if (MODE == 1) return __ldcg(x + c);
    if (MODE == 2 || (MODE == 3 && (u & 1))) {
        int2 t = tex1Dfetch<int2>(tx, c);
        return __hiloint2double(t.y, t.x);
    }
    if (MODE == 3) return __ldg(x + c);
    if (MODE == 4) {
        double v;
        asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(x + c));
        return v;
    }
    return __ldca(x + c);
}

template <int MODE, int MINB>
__global__ void __launch_bounds__(256, MINB)
fold(int64_t nnz, const int* __restrict__ row, const int* __restrict__ col, const double* __restrict__ val,
     const double* __restrict__ x, cudaTextureObject_t tx, double* __restrict__ out) {
    const int64_t T = int64_t(gridDim.x) * 256;
    double acc = 0.0;
    int rsum = 0;
    for (int64_t kb = (int64_t(blockIdx.x) * 256 + threadIdx.x) * 8; kb + 8 <= nnz; kb += T * 8) {
        const int4 c0 = __ldcs(reinterpret_cast<const int4*>(col + kb));
        const int4 c1 = __ldcs(reinterpret_cast<const int4*>(col + kb + 4));
        const int4 r0 = __ldcs(reinterpret_cast<const int4*>(row + kb));
        const int4 r1 = __ldcs(reinterpret_cast<const int4*>(row + kb + 4));
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
        for (int u = 0; u < 8; ++u) g[u] = gx<MODE>(x, tx, c[u], u);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, __dmul_rn(v[u], g[u]));
        rsum += r0.x ^ r1.w;
    }
    if (acc == 12345.0 || rsum == 7) out[0] = acc;
    out[1 + (blockIdx.x * 256 + threadIdx.x) % 1024] = acc;
}

template <int MODE, int MINB>
float run(int64_t nnz, const int* row, const int* col, const double* val, const double* x, cudaTextureObject_t tx,
          double* out, int blocks_per_sm, int sms) {
    int grid = sms * blocks_per_sm;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) fold<MODE, MINB><<<grid, 256>>>(nnz, row, col, val, x, tx, out);
    cudaEventRecord(a);
    const int reps = 10;
    for (int i = 0; i < reps; ++i) fold<MODE, MINB><<<grid, 256>>>(nnz, row, col, val, x, tx, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
    return ms / reps;
}


// Hot-column cache: the K most frequent columns' x values are packed (hx,
// one gather pass per launch) and copied into shared memory by every CTA of a
// persistent grid; col2[k] = ~slot for a cached column, col otherwise.
__global__ void pack_hot(int K, const int* __restrict__ hot, const double* __restrict__ x, double* __restrict__ hx) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < K) hx[i] = __ldg(x + hot[i]);
}

template <int K>
__global__ void __launch_bounds__(1024, 1)
fold_hot(int64_t nnz, const int* __restrict__ row, const int* __restrict__ col2, const double* __restrict__ val,
         const double* __restrict__ x, const double* __restrict__ hxg, double* __restrict__ out) {
    extern __shared__ double hx[];
    for (int i = threadIdx.x; i < K; i += blockDim.x) hx[i] = hxg[i];
    __syncthreads();
    const int64_t T = int64_t(gridDim.x) * blockDim.x;
    double acc = 0.0;
    int rsum = 0;
    for (int64_t kb = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 8; kb + 8 <= nnz; kb += T * 8) {
        const int4 c0 = __ldcs(reinterpret_cast<const int4*>(col2 + kb));
        const int4 c1 = __ldcs(reinterpret_cast<const int4*>(col2 + kb + 4));
        const int4 r0 = __ldcs(reinterpret_cast<const int4*>(row + kb));
        const int4 r1 = __ldcs(reinterpret_cast<const int4*>(row + kb + 4));
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
        for (int u = 0; u < 8; ++u) g[u] = c[u] < 0 ? hx[~c[u]] : __ldg(x + c[u]);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, __dmul_rn(v[u], g[u]));
        rsum += r0.x ^ r1.w;
    }
    if (acc == 12345.0 || rsum == 7) out[0] = acc;
    out[1 + (blockIdx.x * 1024 + threadIdx.x) % 1024] = acc;
}

__global__ void col_hist(int64_t nnz, const int* __restrict__ col, int* __restrict__ cnt) {
    int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e < nnz) atomicAdd(cnt + col[e], 1);
}
__global__ void make_slot(int K, const int* __restrict__ hot, int* __restrict__ slot) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < K) slot[hot[i]] = i;
}
__global__ void remap(int64_t nnz, const int* __restrict__ col, const int* __restrict__ slot, int* __restrict__ col2) {
    int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e < nnz) {
        int s = slot[col[e]];
        col2[e] = s >= 0 ? ~s : col[e];
    }
}

template <int K>
int run_hot(int64_t n, int64_t nnz, const int* row, const int* col, const double* val, const double* x, double* out,
            int sms, int* cnt_sorted_cols, int* slot, int* col2, double* hx, const char* tag) {
    CK(cudaMemset(slot, 0xff, n * 4));
    make_slot<<<(K + 255) / 256, 256>>>(K, cnt_sorted_cols, slot);
    remap<<<(nnz + 255) / 256, 256>>>(nnz, col, slot, col2);
    CK(cudaFuncSetAttribute(fold_hot<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, K * 8));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto go = [&] {
        pack_hot<<<(K + 255) / 256, 256>>>(K, cnt_sorted_cols, x, hx);
        fold_hot<K><<<sms, 1024, K * 8>>>(nnz, row, col2, val, x, hx, out);
    };
    for (int i = 0; i < 3; ++i) go();
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) go();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 10;
    cudaError_t e = cudaGetLastError();
    const double bytes = 16.0 * nnz + 8.0 * n;
    printf("hot K=%d %s: %.4f ms  %.1f GB/s  %s\n", K, tag, ms, bytes / ms / 1e6, e == cudaSuccess ? "" : cudaGetErrorString(e));
    return 0;
}

__global__ void fold_cols(int64_t nnz, int* col, int mask) {
    int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e < nnz) col[e] &= mask;
}

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
    nnz &= ~int64_t(7);
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
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = x;
    rd.res.linear.desc = cudaCreateChannelDesc<int2>();
    rd.res.linear.sizeInBytes = n * 8;
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tx;
    CK(cudaCreateTextureObject(&tx, &rd, &td, nullptr));
    const double bytes = 16.0 * nnz + 8.0 * n;
    printf("nnz %lld, bytes %.3f GB (16 B/entry + x)\n", (long long)nnz, bytes / 1e9);
#define R(MODE, MINB, BPS)                                                                                  \
    {                                                                                                       \
        float ms = run<MODE, MINB>(nnz, row, col, val, x, tx, out, BPS, sms);                              \
        printf("mode %d minb %d blocks/SM %d: %.4f ms  %.1f GB/s  %.2f Ggather/s\n", MODE, MINB, BPS, ms,    \
               bytes / ms / 1e6, nnz / ms / 1e6);                                                            \
    }
    R(0, 1, 4) R(0, 1, 8) R(0, 4, 4) R(0, 4, 8)
    R(1, 4, 8) R(2, 4, 8) R(3, 4, 8) R(4, 4, 8) R(5, 4, 8)
    R(2, 4, 4) R(3, 4, 4) R(1, 4, 4)
    {
        int *cnt, *ids, *slot, *col2;
        double* hx;
        CK(cudaMalloc(&cnt, n * 4));
        CK(cudaMalloc(&ids, n * 4));
        CK(cudaMalloc(&slot, n * 4));
        CK(cudaMalloc(&col2, nnz * 4));
        CK(cudaMalloc(&hx, 32768 * 8));
        CK(cudaMemset(cnt, 0, n * 4));
        col_hist<<<(nnz + 255) / 256, 256>>>(nnz, col, cnt);
        thrust::sequence(thrust::device_ptr<int>(ids), thrust::device_ptr<int>(ids + n));
        thrust::sort_by_key(thrust::device_ptr<int>(cnt), thrust::device_ptr<int>(cnt + n), thrust::device_ptr<int>(ids),
                            thrust::greater<int>());
        std::vector<int> hc(65536);
        CK(cudaMemcpy(hc.data(), cnt, 65536 * 4, cudaMemcpyDeviceToHost));
        long long s = 0;
        for (int k = 0; k < 65536; ++k) {
            s += hc[k];
            if (k + 1 == 4096 || k + 1 == 8192 || k + 1 == 16384 || k + 1 == 24576 || k + 1 == 32768 || k + 1 == 65536)
                printf("top %d columns: %.4f of entries\n", k + 1, double(s) / nnz);
        }
        run_hot<8192>(n, nnz, row, col, val, x, out, sms, ids, slot, col2, hx, "");
        run_hot<4096>(n, nnz, row, col, val, x, out, sms, ids, slot, col2, hx, "");
    }
    // sensitivity to the x footprint: fold the column ids into n/2, n/4, n/8
    for (int sh = 1; sh <= 3; ++sh) {
        fold_cols<<<(nnz + 255) / 256, 256>>>(nnz, col, int((n >> sh) - 1));
        printf("x footprint %lld MB:\n", (long long)((n >> sh) * 8 >> 20));
        R(0, 1, 4) R(0, 1, 8)
    }
    return 0;
}
