// Shared helpers of the Krylov solvers: masked element-wise launches, 1-thread
// scalar kernels, workspace carving and CUDA-graph capture of an iteration
// period (krylov.cu, krylov_steps.cu).
#pragma once

#include "reduce.cuh"

namespace wk {

template <typename F>
__global__ void __launch_bounds__(256) masked_map_kernel(int64_t n, F f, const int* __restrict__ skip) {
    if (skip != nullptr && *skip) return;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) f(i);
}

template <typename F>
int launch_masked_map(int64_t n, F f, const int* skip, cudaStream_t st) {
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
int launch_scalar(F f, cudaStream_t st) {
    scalar_kernel<<<1, 1, 0, st>>>(f);
    WK_LAUNCH_CHECK();
    return 0;
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
int capture(GraphRunner& g, Body body) {
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


inline int check_square(const wk_matrix* A) {
    WK_REQUIRE(A->nrows == A->ncols, WK_ERR_DIMENSION, "solver needs a square matrix, got %lldx%lld",
               (long long)A->nrows, (long long)A->ncols);
    return 0;
}

}  // namespace wk
