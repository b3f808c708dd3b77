// Stable LSD radix sort of (uint64 key, f64 value) pairs — the device half of
// CooMatrix.from_entries (sparse.py:63-80: np.lexsort by (row, col), then
// duplicates summed with np.add.at in input order). The key is row * ncols +
// col, so only bit_length(nrows * ncols - 1) bits are sorted: 48 bits (6
// passes of 8) for R-MAT scale 24, against the 8 passes a generic 64-bit sort
// makes. Values travel with their keys (no permutation array and no final
// gather).
//
// One pass = three kernels over chunks of kRsChunk = 32768 pairs:
//   rs_upsweep    per-chunk digit histogram (per-warp shared histograms)
//                 -> counts[digit * nchunks + chunk]
//   exclusive scan of the digit-major counts -> the global output offset of
//                 every (digit, chunk)
//   rs_downsweep  the chunk in 16 sub-tiles of 2048 pairs, in order, each
//                 streamed into shared memory by cp.async.bulk one sub-tile
//                 ahead (two stages; a stage doubles as the reorder buffer of
//                 its sub-tile: 3 CTAs per SM instead of 4 with register
//                 loads, but no load latency on the ranking path). Stable
//                 ranking inside a sub-tile: each warp owns 256 consecutive
//                 pairs (warp-striped: item j of lane l = 32 j + l, so the
//                 (j, lane) order is the input order); per item, eight ballots
//                 give the lanes with equal digits, the rank among
//                 them, and one running per-warp digit count; per-digit
//                 prefixes over the 8 warps and a block scan over the 256
//                 digits give every pair its rank in the sub-tile. The sub-tile
//                 is reordered in shared memory and written out with
//                 consecutive threads on consecutive addresses of each digit
//                 run (coalesced), continuing the chunk's running digit bases.
// Every step preserves input order among equal digits, so the sort is stable:
// duplicates reach the fold in input order, as np.add.at sums them.
#include "reduce.cuh"

namespace wk {

constexpr int kRsThreads = 256;
constexpr int kRsWarps = kRsThreads / 32;
constexpr int kRsItems = 8;                       // per lane per sub-tile
constexpr int kRsTile = kRsThreads * kRsItems;    // 2048 pairs
constexpr int kRsTilesPerChunk = 16;
constexpr int64_t kRsChunk = int64_t(kRsTile) * kRsTilesPerChunk;  // 32768 pairs
constexpr int kRsDigits = 256;

// Lanes of the warp whose (valid) digit equals this lane's: eight ballots
// (match.any.sync is far slower: the first version spent 1.6 ms per pass of
// the histogram kernel stalled on it).
__device__ __forceinline__ unsigned digit_peers(unsigned d, bool valid) {
    const unsigned vmask = __ballot_sync(0xffffffffu, valid);
    unsigned peers = vmask;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const unsigned bit = (d >> b) & 1u;
        const unsigned bal = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? bal : ~bal;
    }
    return valid ? peers : 0u;
}

__global__ void __launch_bounds__(kRsThreads)
rs_upsweep(int64_t n, const unsigned long long* __restrict__ keys, int shift, int64_t nchunks,
           unsigned* __restrict__ counts) {
    __shared__ unsigned h[kRsWarps][kRsDigits];  // per-warp histograms
    const int t = threadIdx.x, w = t >> 5;
#pragma unroll
    for (int q = 0; q < kRsWarps; ++q) h[q][t] = 0u;
    __syncthreads();
    const int64_t lo = int64_t(blockIdx.x) * kRsChunk;
    const int64_t hi = lo + kRsChunk < n ? lo + kRsChunk : n;
    for (int64_t i0 = lo; i0 < hi; i0 += kRsThreads * 4) {
        unsigned d[4];
        bool ok[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = i0 + u * kRsThreads + t;
            ok[u] = i < hi;
            d[u] = ok[u] ? unsigned(__ldcs(keys + i) >> shift) & 255u : 0u;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (ok[u]) atomicAdd(&h[w][d[u]], 1u);  // shared atomics: replays only on equal digits
    }
    __syncthreads();
    unsigned tot = 0;
#pragma unroll
    for (int q = 0; q < kRsWarps; ++q) tot += h[q][t];
    counts[int64_t(t) * nchunks + blockIdx.x] = tot;
}

// Sub-tile staging: keys | values of one sub-tile (16 KB + 16 KB) per stage,
// two stages; the next sub-tile streams in (cp.async.bulk, one mbarrier per
// stage) while the current one is ranked, and the current stage is then
// reused as the reorder buffer.
constexpr int kRsStageBytes = kRsTile * 16;
constexpr int kRsSmem = 2 * kRsStageBytes + 64;

// The downsweep runs 512 threads (16 warps, 4 pairs each) on a 2048-pair
// sub-tile: every serial phase of a sub-tile (the per-warp ranking chain, the
// writes) is half as long as with 256 threads x 8 pairs, and two CTAs fit an
// SM (32 warps instead of 24); the 256 digit-indexed steps use threads 0..255.
constexpr int kDsThreads = 512;
constexpr int kDsWarps = kDsThreads / 32;
constexpr int kDsItems = kRsTile / kDsThreads;

__global__ void __launch_bounds__(kDsThreads, 2)
rs_downsweep(int64_t n, const unsigned long long* __restrict__ kin, const double* __restrict__ vin,
             unsigned long long* __restrict__ kout, double* __restrict__ vout, int shift, int64_t nchunks,
             const int64_t* __restrict__ offs) {
    extern __shared__ __align__(128) unsigned char rs_smem[];
    __shared__ int64_t base[kRsDigits];
    __shared__ unsigned short wcnt[kDsWarps][kRsDigits];  // <= 128 per warp and digit
    __shared__ unsigned dstart[kRsDigits];
    __shared__ unsigned dcount[kRsDigits];
    __shared__ unsigned wsum[kRsDigits / 32];
    uint64_t* full = reinterpret_cast<uint64_t*>(rs_smem + 2 * kRsStageBytes);
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const bool dig = t < kRsDigits;  // thread t owns digit t in the digit-indexed steps
    const unsigned lt = (1u << lane) - 1u;
    if (dig) base[t] = offs[int64_t(t) * nchunks + blockIdx.x];
    const int64_t clo = int64_t(blockIdx.x) * kRsChunk;
    const int64_t chi = clo + kRsChunk < n ? clo + kRsChunk : n;
    const int ntile = int((chi - clo + kRsTile - 1) / kRsTile);
    const uint64_t pol = policy_evict_first();
    if (t == 0) {
        mbar_init(full, 1);
        mbar_init(full + 1, 1);
        fence_mbar_init();
    }
    __syncthreads();
    // bulk part of sub-tile i: an even number of pairs (16-byte multiples)
    auto issue = [&](int i) {
        const int64_t s0 = clo + int64_t(i) * kRsTile;
        const int cnt = int(chi - s0 < kRsTile ? chi - s0 : kRsTile);
        const uint32_t nb = uint32_t(cnt & ~1) * 8u;
        unsigned char* st = rs_smem + (i & 1) * kRsStageBytes;
        mbar_arrive_expect_tx(full + (i & 1), 2 * nb);
        if (nb) {
            bulk_g2s_evict_first(st, kin + s0, nb, full + (i & 1), pol);
            bulk_g2s_evict_first(st + kRsTile * 8, vin + s0, nb, full + (i & 1), pol);
        }
    };
    if (t == 0) issue(0);
    unsigned short* wflat = &wcnt[0][0];
    for (int it = 0; it < ntile; ++it) {
        const int64_t s0 = clo + int64_t(it) * kRsTile;
        const int cnt = int(chi - s0 < kRsTile ? chi - s0 : kRsTile);
        unsigned long long* sk = reinterpret_cast<unsigned long long*>(rs_smem + (it & 1) * kRsStageBytes);
        double* sv = reinterpret_cast<double*>(rs_smem + (it & 1) * kRsStageBytes + kRsTile * 8);
        if (t == 0 && it + 1 < ntile) issue(it + 1);  // the other stage was released at the end of it - 1
#pragma unroll
        for (int q = 0; q < kDsWarps * kRsDigits / kDsThreads; ++q) wflat[q * kDsThreads + t] = 0;
        mbar_wait(full + (it & 1), uint32_t((it >> 1) & 1));
        if ((cnt & 1) && t == 0) {  // odd tail pair: not part of the bulk copy
            sk[cnt - 1] = kin[s0 + cnt - 1];
            sv[cnt - 1] = vin[s0 + cnt - 1];
        }
        __syncthreads();
        unsigned long long k[kDsItems];
        double v[kDsItems];
        unsigned d[kDsItems];  // digit (256: no pair), then | rank << 9
#pragma unroll
        for (int j = 0; j < kDsItems; ++j) {
            const int li = w * (32 * kDsItems) + j * 32 + lane;
            const bool ok = li < cnt;
            k[j] = ok ? sk[li] : 0ull;
            v[j] = ok ? sv[li] : 0.0;
            d[j] = ok ? unsigned(k[j] >> shift) & 255u : 256u;
        }
#pragma unroll
        for (int j = 0; j < kDsItems; ++j) {
            const unsigned dj = d[j];
            const unsigned peers = digit_peers(dj & 255u, dj < 256u);
            const unsigned before = dj < 256u ? wcnt[w][dj] : 0u;
            d[j] = dj | ((before + __popc(peers & lt)) << 9);
            __syncwarp();
            if (dj < 256u && lane == __ffs(peers) - 1) wcnt[w][dj] = (unsigned short)(before + __popc(peers));
            __syncwarp();
        }
        __syncthreads();  // every pair of the stage is in registers: the stage becomes the reorder buffer
        // digit t: exclusive prefix over the warps, total count, block scan of the totals
        unsigned run = 0, incl = 0;
        if (dig) {
#pragma unroll
            for (int q = 0; q < kDsWarps; ++q) {
                const unsigned c = wcnt[q][t];
                wcnt[q][t] = (unsigned short)run;  // < 2048: the sub-tile offset of warp q's first pair
                run += c;
            }
            dcount[t] = run;
            incl = run;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) wsum[w] = incl;
        }
        __syncthreads();
        if (dig) {
            unsigned wpre = 0;
            for (int q = 0; q < w; ++q) wpre += wsum[q];
            dstart[t] = wpre + incl - run;
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kDsItems; ++j) {
            const unsigned dj = d[j] & 511u;
            if (dj < 256u) {
                const unsigned pos = dstart[dj] + wcnt[w][dj] + (d[j] >> 9);
                sk[pos] = k[j];
                sv[pos] = v[j];
            }
        }
        __syncthreads();
        for (int i = t; i < cnt; i += kDsThreads) {
            const unsigned long long key = sk[i];
            const unsigned dd = unsigned(key >> shift) & 255u;
            const int64_t dst = base[dd] + (i - int(dstart[dd]));
            __stcs(kout + dst, key);
            __stcs(vout + dst, sv[i]);
        }
        __syncthreads();  // stage free: the next iteration's bulk copy may overwrite it
        if (t == 0) fence_proxy_async_smem();
        if (dig) base[t] += dcount[t];
    }
}

}  // namespace wk

using namespace wk;

extern "C" {

int64_t wk_sort_pairs_workspace(int64_t n) {
    const int64_t nchunks = ceil_div(n, kRsChunk);
    const int64_t m = nchunks * kRsDigits;
    return ceil_div(m * 4, 256) * 256 + ceil_div((m + 1) * 8, 256) * 256 + ceil_div(scan_ws_bytes(m), 256) * 256;
}

int wk_sort_pairs_u64_f64(int64_t n, int32_t key_bits, uint64_t* keys, double* values, uint64_t* keys_alt,
                          double* values_alt, void* work, int64_t work_bytes, wk_stream_t stream) {
    clear_error();
    WK_REQUIRE(n >= 0 && key_bits >= 0 && key_bits <= 64, WK_ERR_INVALID, "bad sort shape (n %lld, key_bits %d)",
               (long long)n, key_bits);
    WK_REQUIRE(work_bytes >= wk_sort_pairs_workspace(n), WK_ERR_INVALID, "sort workspace too small");
    const int passes = (key_bits + 7) / 8;
    if (n <= 1 || passes == 0) return 0;
    auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
    WK_REQUIRE(al16(keys) && al16(values) && al16(keys_alt) && al16(values_alt), WK_ERR_INVALID,
               "sort buffers must be 16-byte aligned");
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev & 63]) {
        WK_CUDA(cudaFuncSetAttribute(rs_downsweep, cudaFuncAttributeMaxDynamicSharedMemorySize, kRsSmem));
        attr_set[dev & 63] = true;
    }
    cudaStream_t st = as_stream(stream);
    const int64_t nchunks = ceil_div(n, kRsChunk);
    const int64_t m = nchunks * kRsDigits;
    char* p = reinterpret_cast<char*>(work);
    unsigned* counts = reinterpret_cast<unsigned*>(p);
    p += ceil_div(m * 4, 256) * 256;
    int64_t* offs = reinterpret_cast<int64_t*>(p);
    p += ceil_div((m + 1) * 8, 256) * 256;
    void* scan_ws = p;
    auto* ka = reinterpret_cast<unsigned long long*>(keys);
    auto* kb = reinterpret_cast<unsigned long long*>(keys_alt);
    double* va = values;
    double* vb = values_alt;
    for (int pass = 0; pass < passes; ++pass) {
        const int shift = 8 * pass;
        rs_upsweep<<<unsigned(nchunks), kRsThreads, 0, st>>>(n, ka, shift, nchunks, counts);
        WK_LAUNCH_CHECK();
        const unsigned* c = counts;
        WK_TRY(exclusive_scan(m, [=] __device__(int64_t i) { return int64_t(c[i]); }, offs, scan_ws, st));
        rs_downsweep<<<unsigned(nchunks), kDsThreads, kRsSmem, st>>>(n, ka, va, kb, vb, shift, nchunks, offs);
        WK_LAUNCH_CHECK();
        unsigned long long* tk = ka;
        ka = kb;
        kb = tk;
        double* tv = va;
        va = vb;
        vb = tv;
    }
    // an odd number of passes leaves the result in the alternate buffers: copy back
    if (passes & 1) {
        WK_CUDA(cudaMemcpyAsync(keys, keys_alt, size_t(n) * 8, cudaMemcpyDeviceToDevice, st));
        WK_CUDA(cudaMemcpyAsync(values, values_alt, size_t(n) * 8, cudaMemcpyDeviceToDevice, st));
    }
    return 0;
}

}  // extern "C"
