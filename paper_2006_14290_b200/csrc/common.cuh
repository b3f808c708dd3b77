// Shared helpers for the wk_* C-ABI library (sm_100a only).
#pragma once

#include <cooperative_groups.h>
#include <cooperative_groups/reduce.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/wk_sparse.h"

namespace cg = cooperative_groups;

namespace wk {

// ---- error plumbing: every C entry point returns a status and records a
// thread-local message retrievable through wk_last_error() --------------------
void set_error(const char* fmt, ...);
void clear_error();

#define WK_CUDA(expr)                                                                   \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess) {                                                        \
            ::wk::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),     \
                            __FILE__, __LINE__);                                        \
            return (int)_e;                                                             \
        }                                                                               \
    } while (0)

#define WK_REQUIRE(cond, code, ...)                                                     \
    do {                                                                                \
        if (!(cond)) {                                                                  \
            ::wk::set_error(__VA_ARGS__);                                               \
            return (code);                                                              \
        }                                                                               \
    } while (0)

#define WK_LAUNCH_CHECK()                                                               \
    do {                                                                                \
        cudaError_t _e = cudaGetLastError();                                            \
        if (_e != cudaSuccess) {                                                        \
            ::wk::set_error("kernel launch failed: %s (%s:%d)", cudaGetErrorString(_e), \
                            __FILE__, __LINE__);                                        \
            return (int)_e;                                                             \
        }                                                                               \
    } while (0)

#define WK_TRY(expr)          \
    do {                      \
        int _rc = (expr);     \
        if (_rc) return _rc;  \
    } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Number of SMs of the current device (cached per device).
int sm_count();

// CG q = A p with the p.q reduction fused into the SpMV (spmv.cu); returns 1
// if A cannot take the fused path.
int spmv_dot_fused(const wk_matrix* A, const double* p, double* q, wk_cg_state* s, void* red_ws, int finalize,
                   cudaStream_t st, void* peer = nullptr, const void* halo = nullptr, int rev = 0);

// BiCGSTAB SpMV with its dot(s) fused: mode 1 rv = w.y, mode 2 tt = y.y, ts =
// y.x (spmv.cu); returns 1 if A cannot take the fused path.
int spmv_bicg_fused(const wk_matrix* A, const double* x, double* y, wk_bicg_state* s, const double* w, int mode,
                    void* red_ws, cudaStream_t st);

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---- device helpers ------------------------------------------------------------

// Streaming loads for matrix data that is touched exactly once per SpMV:
// evict-first in L2 so the x vector (gathered, reused) stays resident.
__device__ __forceinline__ double ld_stream(const double* p) { return __ldcs(p); }
__device__ __forceinline__ int ld_stream(const int* p) { return __ldcs(p); }
__device__ __forceinline__ double2 ld_stream(const double2* p) { return __ldcs(p); }
__device__ __forceinline__ int2 ld_stream(const int2* p) { return __ldcs(p); }
__device__ __forceinline__ int4 ld_stream(const int4* p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(double* p, double v) { __stcs(p, v); }

// Gathered x: read-only path (L1-allocating) — neighbouring rows reuse it.
__device__ __forceinline__ double ld_x(const double* x, int c) { return __ldg(x + c); }

// Separately rounded multiply-add, matching the reference's Python floats
// (sparse.py:391-395). The library is also compiled with -fmad=false.
__device__ __forceinline__ double mul_add_rn(double acc, double v, double xv) {
    return __dadd_rn(acc, __dmul_rn(v, xv));
}

// ---- Hopper+/Blackwell async bulk copy (TMA 1-D) + mbarrier, inline PTX ------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

// make mbarrier inits visible to the async (TMA) proxy
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// order this thread's prior generic-proxy shared-memory accesses before
// subsequent async-proxy (bulk copy) writes to the same buffer
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// try_wait with a suspend-time hint: a waiting warp sleeps in hardware until
// the phase completes (or the hint expires) instead of spinning on issue slots.
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// 1-D bulk async copy global -> shared (TMA engine), completion counted on `bar`.
// dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

// same with an L2 evict-first cache hint (matrix data is streamed once)
__device__ __forceinline__ void bulk_g2s_evict_first(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                                     uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
        "%4;" ::"r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
        : "memory");
}

// 1-D bulk async copy shared -> global (TMA engine), tracked by bulk groups of
// the issuing thread. dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

// wait until at most N of this thread's committed bulk groups still read shared memory
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

template <int N>
__device__ __forceinline__ void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// Butterfly all-reduce over a power-of-two tile: exactly log2(size)
// shfl_xor rounds (kernels.py:35-49, reduce.cuh:8-16) expressed with
// cooperative-groups tiles.
template <unsigned Size, typename T, typename Parent>
__device__ __forceinline__ T reduce_subwarp(const cg::thread_block_tile<Size, Parent>& tile, T v) {
#pragma unroll
    for (unsigned mask = Size / 2; mask > 0; mask >>= 1) v += tile.shfl_xor(v, mask);
    return v;
}

// Deterministic block sum (fixed tree for a fixed blockDim): warp
// butterflies, then warp 0 reduces the per-warp partials.
template <int kThreads>
__device__ __forceinline__ double block_sum(double v, double* smem /* >= kThreads/32 */) {
    auto block = cg::this_thread_block();
    auto warp = cg::tiled_partition<32>(block);
    v = reduce_subwarp(warp, v);
    if (warp.thread_rank() == 0) smem[warp.meta_group_rank()] = v;
    block.sync();
    double r = 0.0;
    if (warp.meta_group_rank() == 0) {
        r = warp.thread_rank() < kThreads / 32 ? smem[warp.thread_rank()] : 0.0;
        r = reduce_subwarp(warp, r);
    }
    return r;  // valid in thread 0
}

}  // namespace wk
