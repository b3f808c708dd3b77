// Peer-memory communication for the row-block distributed solvers: one-shot
// scalar all-reduce and halo exchange by direct stores into the other ranks'
// memory (NVLink / NVSwitch peer access between GPUs; CUDA IPC maps each
// rank's arena into every other rank's address space), replacing the NCCL
// calls of the distributed CG / BiCGSTAB / GMRES with single small kernels
// that can be captured in the same CUDA graph as the compute kernels.
//
// Arena (one per rank, cudaMalloc'd, IPC-exported; identical layout on all
// ranks so a rank addresses a peer's vector by its own offset):
//   [0, 512)          all-reduce flags, u64 per source rank (monotone seq)
//   [512, 1024)       halo flags, u64 per source rank
//   [1024, 33792)     all-reduce slots: [2 parities][64 ranks][32 doubles]
//   [33792, ...)      distributed vectors [owned | halo], same offsets on all
//                     ranks (sized by the largest rank)
// Protocol (writer): plain stores of the payload to the peer, then
// __threadfence_system and st.release.sys of the peer's flag[me] = seq.
// Reader: ld.acquire.sys of its own flag[src] until >= seq. Sequence numbers
// live in device memory and are advanced by the kernels, so graph replays
// stay in step. All-reduce slots alternate between two parities and every
// rank sums the P slots in rank order: bit-identical results everywhere (the
// device-side convergence flags of the solvers then agree, as with NCCL).
// Spins are bounded (~10 s): on timeout the kernel sets an error word
// instead of hanging the GPU.
#include "peer_dev.cuh"

namespace wk {

__global__ void peer_allreduce_kernel(PeerCtx ctx, const double* __restrict__ src, double* __restrict__ dst,
                                      int count) {
    if (threadIdx.x != 0) return;
    const unsigned long long seq = (unsigned long long)ctx.seq[0] + 1ull;
    const int par = int(seq & 1ull);
    double v[kPeerSlots];
    for (int i = 0; i < count; ++i) v[i] = src[i];
    for (int q = 0; q < ctx.world; ++q) {
        double* slot = reinterpret_cast<double*>(ctx.arena[q] + kSlots) + (par * kPeerMax + ctx.rank) * kPeerSlots;
        for (int i = 0; i < count; ++i) slot[i] = v[i];
    }
    __threadfence_system();
    for (int q = 0; q < ctx.world; ++q)
        st_release_sys(reinterpret_cast<unsigned long long*>(ctx.arena[q] + kArFlags) + ctx.rank, seq);
    const unsigned long long* mine = reinterpret_cast<const unsigned long long*>(ctx.arena[ctx.rank] + kArFlags);
    for (int q = 0; q < ctx.world; ++q)
        if (!wait_flag(mine + q, seq)) {
            *ctx.error = 1;
            break;
        }
    const double* slots = reinterpret_cast<const double*>(ctx.arena[ctx.rank] + kSlots) + par * kPeerMax * kPeerSlots;
    for (int i = 0; i < count; ++i) {
        double acc = 0.0;
        for (int q = 0; q < ctx.world; ++q) acc = __dadd_rn(acc, __ldcv(slots + q * kPeerSlots + i));
        dst[i] = acc;
    }
    ctx.seq[0] = (long long)seq;
}

constexpr int kPeerMaxSends = 8;

struct PeerSends {
    int n;
    int peer[kPeerMaxSends];
    const int* idx[kPeerMaxSends];       // local owned indices to send
    long long count[kPeerMaxSends];
    long long dst_off[kPeerMaxSends];    // byte offset of the destination in the peer's arena
    int nrecv;
    int recv_peer[kPeerMaxSends];
};

// gather + store into the peers' vectors (grid-stride), then the last block to
// finish releases the flags and waits for every incoming halo
__global__ void __launch_bounds__(256)
peer_exchange_kernel(PeerCtx ctx, PeerSends s, const double* __restrict__ x, unsigned* __restrict__ ticket) {
    const unsigned long long seq = (unsigned long long)ctx.seq[1] + 1ull;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (int j = 0; j < s.n; ++j) {
        double* dst = reinterpret_cast<double*>(ctx.arena[s.peer[j]] + s.dst_off[j]);
        const int* idx = s.idx[j];
        for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < s.count[j]; i += stride)
            dst[i] = x[idx[i]];
    }
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    __threadfence_system();
    for (int j = 0; j < s.n; ++j)
        st_release_sys(reinterpret_cast<unsigned long long*>(ctx.arena[s.peer[j]] + kHaloFlags) + ctx.rank, seq);
    const unsigned long long* mine = reinterpret_cast<const unsigned long long*>(ctx.arena[ctx.rank] + kHaloFlags);
    for (int j = 0; j < s.nrecv; ++j)
        if (!wait_flag(mine + s.recv_peer[j], seq)) {
            *ctx.error = 2;
            break;
        }
    *ticket = 0;
    ctx.seq[1] = (long long)seq;
}

}  // namespace wk

using namespace wk;

extern "C" {

int wk_sym_alloc(int64_t bytes, void** ptr, void* handle) {
    clear_error();
    WK_CUDA(cudaMalloc(ptr, size_t(bytes)));
    WK_CUDA(cudaMemset(*ptr, 0, size_t(bytes)));
    cudaIpcMemHandle_t h;
    WK_CUDA(cudaIpcGetMemHandle(&h, *ptr));
    memcpy(handle, &h, sizeof(h));
    return 0;
}

int wk_sym_open(const void* handle, void** ptr) {
    clear_error();
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    WK_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return 0;
}

int wk_sym_close(void* ptr) {
    clear_error();
    WK_CUDA(cudaIpcCloseMemHandle(ptr));
    return 0;
}

int wk_sym_free(void* ptr) {
    clear_error();
    WK_CUDA(cudaFree(ptr));
    return 0;
}

int64_t wk_peer_arena_header_bytes(void) { return kArenaHeader; }

static int make_ctx(const wk_peer_ctx* c, PeerCtx& k) {
    WK_REQUIRE(c->world >= 1 && c->world <= kPeerMax && c->rank >= 0 && c->rank < c->world, WK_ERR_INVALID,
               "peer context: rank %d of %d (at most %d ranks)", c->rank, c->world, kPeerMax);
    k.rank = c->rank;
    k.world = c->world;
    for (int q = 0; q < kPeerMax; ++q) k.arena[q] = q < c->world ? reinterpret_cast<char*>(c->arena[q]) : nullptr;
    k.seq = reinterpret_cast<long long*>(c->seq);
    k.error = c->error;
    return 0;
}

int wk_peer_allreduce(const wk_peer_ctx* ctx, const double* src, double* dst, int32_t count, wk_stream_t stream) {
    clear_error();
    WK_REQUIRE(count >= 1 && count <= kPeerSlots, WK_ERR_INVALID, "peer all-reduce of %d values (1..%d)", count,
               kPeerSlots);
    PeerCtx k;
    WK_TRY(make_ctx(ctx, k));
    peer_allreduce_kernel<<<1, 32, 0, as_stream(stream)>>>(k, src, dst, count);
    WK_LAUNCH_CHECK();
    return 0;
}

int wk_peer_exchange(const wk_peer_ctx* ctx, const double* x, int32_t nsend, const int32_t* send_peer,
                     const int32_t* const* send_idx, const int64_t* send_count, const int64_t* send_dst_offset,
                     int32_t nrecv, const int32_t* recv_peer, void* ticket, wk_stream_t stream) {
    clear_error();
    WK_REQUIRE(nsend >= 0 && nsend <= kPeerMaxSends && nrecv >= 0 && nrecv <= kPeerMaxSends, WK_ERR_INVALID,
               "peer exchange with %d sends / %d receives (at most %d)", nsend, nrecv, kPeerMaxSends);
    PeerCtx k;
    WK_TRY(make_ctx(ctx, k));
    PeerSends s{};
    s.n = nsend;
    long long most = 1;
    for (int j = 0; j < nsend; ++j) {
        s.peer[j] = send_peer[j];
        s.idx[j] = send_idx[j];
        s.count[j] = send_count[j];
        s.dst_off[j] = send_dst_offset[j];
        if (send_count[j] > most) most = send_count[j];
    }
    s.nrecv = nrecv;
    for (int j = 0; j < nrecv; ++j) s.recv_peer[j] = recv_peer[j];
    int64_t blocks = ceil_div(most, 256);
    if (blocks > int64_t(sm_count()) * 4) blocks = int64_t(sm_count()) * 4;
    peer_exchange_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(k, s, x, reinterpret_cast<unsigned*>(ticket));
    WK_LAUNCH_CHECK();
    return 0;
}

}  // extern "C"
