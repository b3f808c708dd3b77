// Device side of the peer-memory protocol (csrc/peer.cu): the arena layout,
// release / acquire flags, and the scalar all-reduce split into a producer
// half (push: the last block of a reduction stores its partial into every
// peer's slot and releases the flags) and a consumer half (wait: a block's
// thread 0 waits for every rank's flag and sums the slots in rank order).
// The fused CG kernels (krylov.cu, sellp_tma.cuh) call the two halves in their
// epilogues / prologues, so an all-reduce costs no extra kernel.
#pragma once

#include "common.cuh"

namespace wk {

constexpr int kPeerMax = 64;
constexpr int kPeerSlots = 32;
constexpr int64_t kArFlags = 0, kHaloFlags = 512, kSlots = 1024, kArenaHeader = 1024 + 2 * kPeerMax * kPeerSlots * 8;

struct PeerCtx {
    int rank, world;
    char* arena[kPeerMax];  // every rank's arena, mapped into this process (own included)
    long long* seq;         // device: [0] all-reduce seq, [1] halo seq
    int* error;             // device: set on a wait timeout
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// wait until flag >= seq (bounded); returns false on timeout
__device__ __forceinline__ bool wait_flag(const unsigned long long* flag, unsigned long long seq) {
    for (long long it = 0; it < (1ll << 27); ++it) {
        if (ld_acquire_sys(flag) >= seq) return true;
        __nanosleep(64);
    }
    return false;
}

// one scalar all-reduce, producer half (thread 0 of the last block): seq
// advances here, so the consumer kernel (next in the stream) reads the new value
__device__ __forceinline__ void peer_push_scalar(PeerCtx* c, double v) {
    const unsigned long long seq = (unsigned long long)c->seq[0] + 1ull;
    const int par = int(seq & 1ull);
    for (int q = 0; q < c->world; ++q)
        reinterpret_cast<double*>(c->arena[q] + kSlots)[(par * kPeerMax + c->rank) * kPeerSlots] = v;
    __threadfence_system();
    for (int q = 0; q < c->world; ++q)
        st_release_sys(reinterpret_cast<unsigned long long*>(c->arena[q] + kArFlags) + c->rank, seq);
    c->seq[0] = (long long)seq;
}

// consumer half (thread 0): the rank-order sum of the all-reduce just pushed
__device__ __forceinline__ double peer_wait_sum(const PeerCtx* c) {
    const unsigned long long seq = (unsigned long long)c->seq[0];
    const int par = int(seq & 1ull);
    const unsigned long long* flags = reinterpret_cast<const unsigned long long*>(c->arena[c->rank] + kArFlags);
    for (int q = 0; q < c->world; ++q)
        if (!wait_flag(flags + q, seq)) *c->error = 1;
    const double* slots = reinterpret_cast<const double*>(c->arena[c->rank] + kSlots) + par * kPeerMax * kPeerSlots;
    double acc = 0.0;
    for (int q = 0; q < c->world; ++q) acc = __dadd_rn(acc, __ldcv(slots + q * kPeerSlots));
    return acc;
}

// block-wide: every thread gets the all-reduced value
__device__ __forceinline__ double peer_wait_sum_block(const PeerCtx* c) {
    __shared__ double g;
    if (threadIdx.x == 0) g = peer_wait_sum(c);
    __syncthreads();
    return g;
}

// Halo of one distributed vector pushed by the kernel that produces it:
// owned rows [lo_j, hi_j) go to rank peer_j at byte offset dst_off_j of its
// arena (the receiver's copy of the vector); the receiving kernel waits for
// the flags of recv_peer[] (slab partitions: contiguous boundary planes).
constexpr int kHaloMax = 8;
struct PeerHalo {
    int n;
    int peer[kHaloMax];
    long long lo[kHaloMax], hi[kHaloMax];
    long long dst_off[kHaloMax];
    int nrecv;
    int recv_peer[kHaloMax];
    long long int_lo, int_hi;  // SELL-P slices [int_lo, int_hi) of the local matrix gather no halo column
};

__device__ __forceinline__ void halo_store(const PeerCtx* c, const PeerHalo* h, long long i, double v) {
    for (int j = 0; j < h->n; ++j)
        if (i >= h->lo[j] && i < h->hi[j])
            reinterpret_cast<double*>(c->arena[h->peer[j]] + h->dst_off[j])[i - h->lo[j]] = v;
}

// last block, thread 0, after every block's system fence: release the halo
// flags at the receivers (seq[1] advances)
__device__ __forceinline__ void halo_release(PeerCtx* c, const PeerHalo* h) {
    const unsigned long long seq = (unsigned long long)c->seq[1] + 1ull;
    __threadfence_system();
    for (int j = 0; j < h->n; ++j)
        st_release_sys(reinterpret_cast<unsigned long long*>(c->arena[h->peer[j]] + kHaloFlags) + c->rank, seq);
    c->seq[1] = (long long)seq;
}

// consumer (thread 0): the halos pushed under the current seq[1] have landed
__device__ __forceinline__ void halo_wait(const PeerCtx* c, const PeerHalo* h) {
    const unsigned long long seq = (unsigned long long)c->seq[1];
    const unsigned long long* flags = reinterpret_cast<const unsigned long long*>(c->arena[c->rank] + kHaloFlags);
    for (int j = 0; j < h->nrecv; ++j)
        if (!wait_flag(flags + h->recv_peer[j], seq)) *c->error = 2;
}

}  // namespace wk
