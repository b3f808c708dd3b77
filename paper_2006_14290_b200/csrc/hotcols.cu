// Gather plan: the hot columns of a power-law matrix, for the COO and CSR
// load_balance kernels (segwarp.cuh seg8_hot_kernel).
//
// A random x gather costs one L2 sector request; on R-MAT those requests, not
// DRAM bytes, bound the SpMV (tools/gather_probe.cu). Columns are far from
// uniform there: the top 8192 columns of R-MAT scale 24 hold 20.8% of the
// entries. The plan, built once per matrix on the device:
//   1. counts[c]   entries per column (one atomic per entry)
//   2. hist[b]     columns per count value (counts >= min_count only: the
//                  many low counts are never candidates)
//   3. threshold   the smallest t >= min_count with #{c : counts[c] >= t}
//                  <= kHotMax (one block, suffix scan of hist)
//   4. slots       hot columns in column order (exclusive scan of the flags),
//                  slot[c] = rank or -1; the first kHotMax are kept
//   5. col2[k]     ~slot[col[k]] for a hot column, col[k] otherwise
// Every CTA of the SpMV gathers x of the hot columns into shared memory once
// per launch, so a column pays off when it has more entries than there are
// CTAs; the default min_count (wk_gather_plan_build) is 2 * SM count.
// The plan changes where x[c] is read from, never the value or the fold order:
// results are bitwise those of the plain kernels.
#include "hotcols.cuh"
#include "reduce.cuh"

namespace wk {

constexpr int kHotBins = 1 << 16;  // count values 0 .. 65535 (last bin: >= 65535)

struct GatherPlanHeader {
    int nhot;        // cached columns (<= kHotMax)
    int threshold;   // count threshold t
    long long covered;  // entries in cached columns
};
static_assert(sizeof(GatherPlanHeader) == 16, "plan header is 16 bytes");

static int64_t plan_col2_offset() { return 16 + int64_t(kHotMax) * 4; }

__global__ void col_count_kernel(int64_t nnz, const int* __restrict__ col, unsigned* __restrict__ counts) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < nnz; e += stride)
        atomicAdd(counts + __ldcs(col + e), 1u);
}

__global__ void count_hist_kernel(int64_t ncols, unsigned min_count, const unsigned* __restrict__ counts,
                                  unsigned* __restrict__ hist) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < ncols; c += stride) {
        const unsigned n = counts[c];
        if (n >= min_count) atomicAdd(hist + (n < unsigned(kHotBins - 1) ? n : unsigned(kHotBins - 1)), 1u);
    }
}

// one block of 1024 threads, 64 bins each (bin b = count value b)
__global__ void __launch_bounds__(1024) threshold_kernel(unsigned min_count, const unsigned* __restrict__ hist,
                                                         GatherPlanHeader* __restrict__ h) {
    constexpr int kPer = kHotBins / 1024;
    __shared__ long long scols[1024];
    __shared__ int best;
    const int t = threadIdx.x;
    long long mine = 0;
    for (int i = 0; i < kPer; ++i) mine += hist[t * kPer + i];
    scols[t] = mine;
    if (t == 0) best = kHotBins;
    __syncthreads();
    // suffix sums over threads (Hillis-Steele on shared memory)
    for (int d = 1; d < 1024; d <<= 1) {
        const long long o = (t + d < 1024) ? scols[t + d] : 0;
        __syncthreads();
        scols[t] += o;
        __syncthreads();
    }
    // columns with count >= the first bin of the next thread
    long long above = (t + 1 < 1024) ? scols[t + 1] : 0;
    for (int i = kPer - 1; i >= 0; --i) {
        const int b = t * kPer + i;
        above += hist[b];
        if (b >= int(min_count) && b >= 1 && above <= kHotMax) atomicMin(&best, b);
    }
    __syncthreads();
    if (t == 0) {
        h->threshold = best;
        h->nhot = 0;
        h->covered = 0;
    }
}

__global__ void slot_kernel(int64_t ncols, const int* __restrict__ offs, unsigned* __restrict__ counts_to_slots,
                            GatherPlanHeader* __restrict__ h, int* __restrict__ hot) {
    const unsigned t = unsigned(h->threshold);
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    long long cov = 0;
    for (int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < ncols; c += stride) {
        const unsigned n = counts_to_slots[c];
        const int o = offs[c];
        int slot = -1;
        if (n >= t && o < kHotMax) {
            slot = o;
            hot[o] = int(c);
            cov += n;
        }
        counts_to_slots[c] = unsigned(slot);
        if (c == ncols - 1) h->nhot = offs[ncols] < kHotMax ? offs[ncols] : kHotMax;
    }
    for (int d = 16; d > 0; d >>= 1) cov += __shfl_xor_sync(0xffffffffu, cov, d);
    if ((threadIdx.x & 31) == 0 && cov) atomicAdd(reinterpret_cast<unsigned long long*>(&h->covered),
                                                  (unsigned long long)cov);
}

__global__ void remap_kernel(int64_t nnz, const int* __restrict__ col, const int* __restrict__ slots,
                             int* __restrict__ col2) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < nnz; e += stride) {
        const int c = __ldcs(col + e);
        const int s = __ldg(slots + c);
        __stcs(col2 + e, s >= 0 ? ~s : c);
    }
}

GatherPlan gather_plan_view(const void* plan) {
    const char* p = reinterpret_cast<const char*>(plan);
    return GatherPlan{reinterpret_cast<const int*>(p), reinterpret_cast<const int*>(p + 16),
                      reinterpret_cast<const int*>(p + plan_col2_offset())};
}

}  // namespace wk

using namespace wk;

extern "C" {

int64_t wk_gather_plan_bytes(int64_t nnz) { return plan_col2_offset() + ceil_div(nnz * 4, 16) * 16; }

int64_t wk_gather_plan_scratch_bytes(int64_t ncols) {
    // counts/slots u32[ncols] | hist u32[kHotBins] | offsets i32[ncols + 1] | scan workspace
    return ceil_div(ncols * 4, 256) * 256 + int64_t(kHotBins) * 4 + ceil_div((ncols + 1) * 4, 256) * 256 +
           ceil_div(scan_ws_bytes(ncols), 256) * 256;
}

int wk_gather_plan_build(int64_t ncols, int64_t nnz, const int32_t* col_idx, int64_t min_count, void* plan,
                         void* scratch, wk_stream_t stream) {
    clear_error();
    WK_REQUIRE(ncols >= 0 && ncols < (int64_t(1) << 31) && nnz >= 0, WK_ERR_INVALID, "bad gather plan shape");
    WK_REQUIRE((reinterpret_cast<uintptr_t>(plan) & 15) == 0 && (reinterpret_cast<uintptr_t>(scratch) & 15) == 0,
               WK_ERR_INVALID, "gather plan and scratch must be 16-byte aligned");
    cudaStream_t st = as_stream(stream);
    if (min_count <= 0) min_count = 2 * int64_t(sm_count());
    if (min_count > kHotBins - 1) min_count = kHotBins - 1;
    char* s = reinterpret_cast<char*>(scratch);
    unsigned* counts = reinterpret_cast<unsigned*>(s);
    s += ceil_div(ncols * 4, 256) * 256;
    unsigned* hist = reinterpret_cast<unsigned*>(s);
    s += int64_t(kHotBins) * 4;
    int* offs = reinterpret_cast<int*>(s);
    s += ceil_div((ncols + 1) * 4, 256) * 256;
    void* scan_ws = s;
    auto* h = reinterpret_cast<GatherPlanHeader*>(plan);
    int* hot = reinterpret_cast<int*>(reinterpret_cast<char*>(plan) + 16);
    int* col2 = reinterpret_cast<int*>(reinterpret_cast<char*>(plan) + plan_col2_offset());
    WK_CUDA(cudaMemsetAsync(plan, 0, size_t(plan_col2_offset()), st));
    if (ncols == 0) return 0;
    WK_CUDA(cudaMemsetAsync(counts, 0, size_t(ncols) * 4, st));
    WK_CUDA(cudaMemsetAsync(hist, 0, size_t(kHotBins) * 4, st));
    const int grid = sm_count() * 8;
    if (nnz) {
        col_count_kernel<<<grid, 256, 0, st>>>(nnz, col_idx, counts);
        WK_LAUNCH_CHECK();
    }
    count_hist_kernel<<<grid, 256, 0, st>>>(ncols, unsigned(min_count), counts, hist);
    WK_LAUNCH_CHECK();
    threshold_kernel<<<1, 1024, 0, st>>>(unsigned(min_count), hist, h);
    WK_LAUNCH_CHECK();
    const unsigned* cnt = counts;
    const GatherPlanHeader* hc = h;
    WK_TRY(exclusive_scan(ncols, [=] __device__(int64_t c) { return int(cnt[c] >= unsigned(hc->threshold)); }, offs,
                          scan_ws, st));
    slot_kernel<<<grid, 256, 0, st>>>(ncols, offs, counts, h, hot);
    WK_LAUNCH_CHECK();
    if (nnz) {
        remap_kernel<<<grid, 256, 0, st>>>(nnz, col_idx, reinterpret_cast<const int*>(counts), col2);
        WK_LAUNCH_CHECK();
    }
    return 0;
}

}  // extern "C"
