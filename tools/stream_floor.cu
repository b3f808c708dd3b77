// Measurement scratch (not product): the cold-cache streaming floor for
// BASELINE config 1 (CSR SpMV of the 5-point 1000^2 Poisson matrix: 80 MB of
// algorithmic traffic, smaller than the 126 MB L2, so every timed launch
// follows a 512 MB L2-flushing write, as in bench.py).
//
// Kernels, each reading the same byte count the CSR SpMV reads (col 20 MB +
// val 40 MB + row_ptrs 4 MB + x 8 MB) and writing 8 MB:
//   vec<B,U>   grid-stride 16-byte loads, U loads in flight per thread, B
//              blocks of 256 threads per SM
//   bulk<K>    one CTA per SM, thread 0 issues cp.async.bulk copies of K KB
//              chunks into a 4-stage shared ring (TMA streaming floor)
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o stream_floor tools/stream_floor.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                 \
    do {                                                                      \
        cudaError_t e = (x);                                                  \
        if (e != cudaSuccess) {                                               \
            printf("%s: %s (%d)\n", #x, cudaGetErrorString(e), __LINE__);     \
            return 1;                                                         \
        }                                                                     \
    } while (0)

__global__ void flush_kernel(int4* buf, int64_t n16) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n16; i += int64_t(gridDim.x) * blockDim.x)
        buf[i] = make_int4(int(i), 0, 0, 0);
}

template <int U>
__global__ void __launch_bounds__(256) vec_kernel(const int4* __restrict__ in, int64_t n16, int4* __restrict__ out,
                                                  int64_t o16) {
    const int64_t T = int64_t(gridDim.x) * blockDim.x;
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    int acc = 0;
    for (int64_t i = t; i < n16; i += T * U) {
        int4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = (i + u * T < n16) ? __ldcs(in + i + u * T) : make_int4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].w;
    }
    for (int64_t i = t; i < o16; i += T) __stcs(out + i, make_int4(acc, 0, 0, 0));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

template <int KB>
__global__ void __launch_bounds__(256, 1) bulk_kernel(const char* __restrict__ in, int64_t nbytes,
                                                      int4* __restrict__ out, int64_t o16) {
    extern __shared__ __align__(128) char smem[];
    constexpr int S = 4;
    constexpr int CH = KB * 1024;
    __shared__ __align__(8) uint64_t bar[S];
    const int64_t nch = (nbytes + CH - 1) / CH;
    if (threadIdx.x == 0)
        for (int s = 0; s < S; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    __syncthreads();
    auto issue = [&](int64_t c, int s) {
        const int64_t off = c * CH;
        const int len = int(nbytes - off < CH ? nbytes - off : CH);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(len));
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(smem + s * CH)),
            "l"(in + off), "r"(len), "r"(smem_u32(&bar[s]))
            : "memory");
    };
    int acc = 0;
    int64_t my = 0;
    for (int64_t c = blockIdx.x; c < nch && my < S; c += gridDim.x, ++my)
        if (threadIdx.x == 0) issue(c, int(my));
    int64_t k = 0;
    for (int64_t c = blockIdx.x; c < nch; c += gridDim.x, ++k) {
        const int s = int(k % S);
        const uint32_t ph = uint32_t((k / S) & 1);
        uint32_t done = 0;
        while (!done)
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(smem_u32(&bar[s])), "r"(ph));
        acc ^= reinterpret_cast<const int*>(smem + s * CH)[threadIdx.x];
        __syncthreads();
        const int64_t cn = c + int64_t(S) * gridDim.x;
        if (threadIdx.x == 0 && cn < nch) issue(cn, s);
    }
    const int64_t T = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < o16; i += T)
        __stcs(out + i, make_int4(acc, 0, 0, 0));
}

// usage: stream_floor [read_bytes write_bytes]; the default is config 1. The
// config-2 headline (SELL-P 27-point 200^3: 2,640,093,256 B read, 64,000,000
// B written) is `stream_floor 2640093256 64000000`.
int main(int argc, char** argv) {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int64_t in_bytes = 72000000;  // col 20 MB + val 40 MB + ptrs 4 MB + x 8 MB
    int64_t out_bytes = 8000000;  // y
    if (argc == 3) {
        in_bytes = (atoll(argv[1]) + 15) / 16 * 16;
        out_bytes = (atoll(argv[2]) + 15) / 16 * 16;
    }
    const int64_t flush_bytes = int64_t(512) << 20;
    char *in, *out, *fl;
    CK(cudaMalloc(&in, in_bytes + 4096));
    CK(cudaMalloc(&out, out_bytes));
    CK(cudaMalloc(&fl, flush_bytes));
    CK(cudaMemset(in, 1, in_bytes));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const double total = double(in_bytes + out_bytes);
    printf("bytes %.1f MB (read %.1f, write %.1f)\n", total / 1e6, in_bytes / 1e6, out_bytes / 1e6);
    auto timeit = [&](const char* name, auto launch) {
        float best = 1e9, sum = 0;
        const int reps = 30;
        for (int r = 0; r < reps + 3; ++r) {
            flush_kernel<<<sms * 4, 512>>>(reinterpret_cast<int4*>(fl), flush_bytes / 16);
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r >= 3) {
                sum += ms;
                best = ms < best ? ms : best;
            }
        }
        cudaError_t e = cudaGetLastError();
        printf("%-28s mean %.2f us  min %.2f us  %.0f GB/s (mean)  %s\n", name, sum / reps * 1e3, best * 1e3,
               total / (sum / reps) / 1e6, e == cudaSuccess ? "" : cudaGetErrorString(e));
    };
    char nm[64];
#define VEC(U, B)                                                                                              \
    snprintf(nm, sizeof nm, "vec U=%d blocks/SM=%d", U, B);                                                    \
    timeit(nm, [&] {                                                                                           \
        vec_kernel<U><<<sms * B, 256>>>(reinterpret_cast<const int4*>(in), in_bytes / 16,                      \
                                        reinterpret_cast<int4*>(out), out_bytes / 16);                         \
    });
    VEC(1, 8) VEC(2, 8) VEC(4, 8) VEC(8, 8) VEC(4, 4) VEC(8, 4) VEC(4, 2) VEC(8, 2) VEC(16, 2) VEC(16, 4)
#define BULK(KB, G)                                                                                            \
    CK(cudaFuncSetAttribute(bulk_kernel<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * KB * 1024));     \
    snprintf(nm, sizeof nm, "bulk %d KB x4, %d CTA/SM", KB, G);                                                \
    timeit(nm, [&] {                                                                                           \
        bulk_kernel<KB><<<sms * G, 256, 4 * KB * 1024>>>(in, in_bytes, reinterpret_cast<int4*>(out),           \
                                                         out_bytes / 16);                                      \
    });
    BULK(8, 1) BULK(16, 1) BULK(32, 1) BULK(48, 1) BULK(8, 2) BULK(16, 2) BULK(24, 2)
    // empty-kernel launch + event overhead
    timeit("empty (launch overhead)", [&] { vec_kernel<1><<<sms, 256>>>(reinterpret_cast<const int4*>(in), 0,
                                                                        reinterpret_cast<int4*>(out), 0); });
    return 0;
}
