// CSR "merge" SpMV: merge-path load balancing (the Ginkgo "load_balance"
// strategy's goal — equal work per CTA whatever the row-length skew — reached
// with the merge-path decomposition of Merrill & Garland, SC'16).
//
// The work list is the merge of the row ends (ptrs[1..n]) with the nonzero
// indices 0..nnz-1: n + nnz items. CTA t owns items [t*kMgTile, (t+1)*kMgTile)
// (kMgTile = 2048), whose (row, nonzero) start coordinates are found once per
// matrix by a binary search along the diagonal (the plan). Per tile:
//   1. stage the tile's row ends and the products v*x[col] of its nonzeros in
//      shared memory (coalesced loads, 8 independent loads + gathers in flight
//      per thread);
//   2. each thread finds its own sub-diagonal (binary search in shared
//      memory) and walks kMgItems items sequentially: a nonzero adds its
//      product to the running sum (separately rounded, in column order), a
//      row end emits the row. Rows that lie entirely inside one thread's
//      items are the reference fold (sparse.py:391-395) bit for bit;
//   3. rows cut by thread boundaries are joined by a block-wide segmented
//      scan of the threads' carries (earlier parts first), rows cut by tile
//      boundaries by a second tiny kernel that adds the tiles' carries in
//      tile order. Both are deterministic: same input, same bits.
// Reassociated rows are checked with the 1e-12 scaled tolerance (the
// reference's own CSR kernel reassociates too, kernels.py:186-190).
#pragma once

#include "common.cuh"

namespace wk {

constexpr int kMgThreads = 256;
constexpr int kMgItems = 8;
constexpr int kMgTile = kMgThreads * kMgItems;

inline int64_t csr_merge_tiles(int64_t nrows, int64_t nnz) {
    const int64_t t = ceil_div(nrows + nnz, kMgTile);
    return t < 1 ? 1 : t;
}

// plan: tile_row[ntiles + 1] int32 | carry_row[ntiles] int32 | carry_val[ntiles] f64 (16-byte aligned parts)
struct MergePlan {
    int* tile_row;
    int* carry_row;
    double* carry_val;
};

inline int64_t csr_merge_plan_bytes(int64_t nrows, int64_t nnz) {
    const int64_t t = csr_merge_tiles(nrows, nnz);
    return ceil_div((t + 1) * 4, 16) * 16 + ceil_div(t * 4, 16) * 16 + t * 8;
}

inline MergePlan csr_merge_plan_views(void* plan, int64_t nrows, int64_t nnz) {
    const int64_t t = csr_merge_tiles(nrows, nnz);
    char* p = reinterpret_cast<char*>(plan);
    MergePlan m;
    m.tile_row = reinterpret_cast<int*>(p);
    p += ceil_div((t + 1) * 4, 16) * 16;
    m.carry_row = reinterpret_cast<int*>(p);
    p += ceil_div(t * 4, 16) * 16;
    m.carry_val = reinterpret_cast<double*>(p);
    return m;
}

// Number of rows finished on the merge path at diagonal `diag`: the smallest i
// with row_end[i] > diag - i - 1 (row_end = ptrs + 1), clamped to [diag - nnz, diag].
template <typename P>
__device__ __forceinline__ int64_t merge_path_rows(int64_t diag, P row_end, int64_t a_len, int64_t b_len) {
    int64_t lo = diag - b_len > 0 ? diag - b_len : 0;
    int64_t hi = diag < a_len ? diag : a_len;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (int64_t(row_end[mid]) <= diag - mid - 1)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

__global__ void csr_merge_plan_kernel(int64_t nrows, int64_t nnz, int64_t ntiles, const int* __restrict__ ptrs,
                                      int* __restrict__ tile_row) {
    const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b > ntiles) return;
    const int64_t total = nrows + nnz;
    int64_t d = b * kMgTile;
    if (d > total) d = total;
    tile_row[b] = int(merge_path_rows(d, ptrs + 1, nrows, nnz));
}

// (flag, value) segmented-sum operator: a flagged right operand restarts the sum.
__device__ __forceinline__ void seg_combine(int& f, double& v, int pf, double pv) {
    if (!f) v = __dadd_rn(pv, v);
    f |= pf;
}

// Per-stage shared-memory layout of the persistent kernel: the tile's values
// (products are formed in place), column indices and row ends, each with
// 16-byte alignment slack for the bulk copies.
constexpr int kMgValSlots = kMgTile + 2;
constexpr int kMgColSlots = kMgTile + 4;
constexpr int kMgEndSlots = kMgTile + 1 + 4;
constexpr size_t kMgStageBytes =
    (size_t(kMgValSlots) * 8 + size_t(kMgColSlots) * 4 + size_t(kMgEndSlots) * 4 + 127) / 128 * 128;
// One stage: 33 KB of shared memory per CTA, five CTAs per SM (registers);
// two stages (double-buffered TMA) left three CTAs per SM and fewer tiles'
// x gathers in flight: R-MAT 24 3.93 -> 2.34 ms, 27-point 200^3 1.09 -> 1.00
// ms (tools/merge_probe.py; 1024-item tiles: 2.14 / 1.28 ms, 4096: 2.57 /
// 1.61 ms).
constexpr int kMgStages = 1;
constexpr size_t kMgSmem = kMgStages * kMgStageBytes + kMgStages * 8 + 256;

struct MgTile {
    int64_t i0, i1, j0, j1;
};

__device__ __forceinline__ MgTile mg_tile(int64_t t, int64_t nrows, int64_t nnz, const int* __restrict__ tile_row) {
    MgTile g;
    const int64_t total = nrows + nnz;
    const int64_t d0 = t * kMgTile;
    const int64_t d1 = (d0 + kMgTile < total) ? d0 + kMgTile : total;
    g.i0 = __ldg(tile_row + t);
    g.i1 = __ldg(tile_row + t + 1);
    g.j0 = d0 - g.i0;
    g.j1 = d1 - g.i1;
    return g;
}

// thread 0: bulk-copy the 16-byte aligned body of the tile's values, columns
// and row ends (ptrs[i0+1 .. i0+nstage]) into a stage
__device__ __forceinline__ void mg_issue(const MgTile& g, int64_t nrows, const int* __restrict__ ptrs,
                                         const int* __restrict__ col, const double* __restrict__ val,
                                         unsigned char* stage, uint64_t* bar, uint64_t pol) {
    const int64_t nstage = (g.i1 - g.i0) + (g.i1 < nrows ? 1 : 0);
    const int64_t va = g.j0 & ~int64_t(1), ve = g.j1 & ~int64_t(1);
    const int64_t ca = g.j0 & ~int64_t(3), ce = g.j1 & ~int64_t(3);
    const int64_t ra = (g.i0 + 1) & ~int64_t(3), re = (g.i0 + 1 + nstage) & ~int64_t(3);
    const uint32_t bv = ve > va ? uint32_t((ve - va) * 8) : 0u;
    const uint32_t bc = ce > ca ? uint32_t((ce - ca) * 4) : 0u;
    const uint32_t br = re > ra ? uint32_t((re - ra) * 4) : 0u;
    mbar_arrive_expect_tx(bar, bv + bc + br);
    if (bv) bulk_g2s_evict_first(stage, val + va, bv, bar, pol);
    if (bc) bulk_g2s_evict_first(stage + size_t(kMgValSlots) * 8, col + ca, bc, bar, pol);
    if (br) bulk_g2s(stage + size_t(kMgValSlots) * 8 + size_t(kMgColSlots) * 4, ptrs + ra, br, bar);
}

// Persistent merge-path kernel: CTA b takes tiles b, b + grid, ...; a tile's
// operands stream in with cp.async.bulk (mbarrier complete_tx) as soon as the
// previous tile's stage is free; the five CTAs of an SM overlap each other's
// loads, gathers and folds.
__global__ void __launch_bounds__(kMgThreads)
csr_merge_kernel(int64_t nrows, int64_t nnz, int64_t ntiles, const int* __restrict__ ptrs,
                 const int* __restrict__ col, const double* __restrict__ val, const double* __restrict__ x,
                 double* __restrict__ y, const int* __restrict__ tile_row, int* __restrict__ carry_row,
                 double* __restrict__ carry_val, const int* __restrict__ skip) {
    if (skip != nullptr && *skip) return;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ double s_wv[kMgThreads / 32];
    __shared__ int s_wf[kMgThreads / 32];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kMgStages * kMgStageBytes);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint64_t pol = policy_evict_first();
    if (tid == 0) {
        for (int s = 0; s < kMgStages; ++s) mbar_init(bars + s, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
        for (int s = 0; s < kMgStages; ++s) {
            const int64_t t = blockIdx.x + int64_t(s) * gridDim.x;
            if (t < ntiles)
                mg_issue(mg_tile(t, nrows, nnz, tile_row), nrows, ptrs, col, val, smem + s * kMgStageBytes, bars + s,
                         pol);
        }
    }
    uint32_t n = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++n) {
        const int st = int(n % kMgStages);
        unsigned char* stage = smem + st * kMgStageBytes;
        double* sv = reinterpret_cast<double*>(stage);
        const int* sc = reinterpret_cast<const int*>(stage + size_t(kMgValSlots) * 8);
        int* se = reinterpret_cast<int*>(stage + size_t(kMgValSlots) * 8 + size_t(kMgColSlots) * 4);
        const MgTile g = mg_tile(t, nrows, nnz, tile_row);
        const int nn = int(g.j1 - g.j0);
        const int nfin = int(g.i1 - g.i0);
        const int nstage = nfin + (g.i1 < nrows ? 1 : 0);
        const int ov = int(g.j0 & 1), oc = int(g.j0 & 3), orr = int((g.i0 + 1) & 3);
        const int nv = int((g.j1 & ~int64_t(1)) - g.j0);   // entries [0, nv) of the values arrived by TMA
        const int nc = int((g.j1 & ~int64_t(3)) - g.j0);
        const int ne = int(((g.i0 + 1 + nstage) & ~int64_t(3)) - (g.i0 + 1));
        mbar_wait(bars + st, (n / kMgStages) & 1);
        // row ends past the bulk body: plain loads (visible after the barrier below)
        if (tid < nstage - (ne > 0 ? ne : 0) && tid < 4) {
            const int k = (ne > 0 ? ne : 0) + tid;
            se[orr + k] = __ldg(ptrs + g.i0 + 1 + k);
        }
        {
            double v[kMgItems], xv[kMgItems];
            int c[kMgItems];
#pragma unroll
            for (int u = 0; u < kMgItems; ++u) {
                const int k = u * kMgThreads + tid;
                v[u] = 0.0;
                c[u] = 0;
                if (k < nn) {
                    v[u] = (k < nv) ? sv[ov + k] : ld_stream(val + g.j0 + k);
                    c[u] = (k < nc) ? sc[oc + k] : ld_stream(col + g.j0 + k);
                }
            }
#pragma unroll
            for (int u = 0; u < kMgItems; ++u) xv[u] = (u * kMgThreads + tid < nn) ? ld_x(x, c[u]) : 0.0;
#pragma unroll
            for (int u = 0; u < kMgItems; ++u) {
                const int k = u * kMgThreads + tid;
                if (k < nn) sv[ov + k] = __dmul_rn(v[u], xv[u]);
            }
        }
        __syncthreads();
        const double* prod = sv + ov;
        const int* rend = se + orr;
        const int jbase = int(g.j0);
        // this thread's sub-path: items [ld, le) of the tile
        const int items = nfin + nn;
        const int ld = (tid * kMgItems < items) ? tid * kMgItems : items;
        const int le = (ld + kMgItems < items) ? ld + kMgItems : items;
        int lo = ld - nn > 0 ? ld - nn : 0, hi = ld < nfin ? ld : nfin;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (rend[mid] - jbase <= ld - mid - 1)
                lo = mid + 1;
            else
                hi = mid;
        }
        int ti = lo, tj = ld - lo;
        double acc = 0.0, first_val = 0.0;
        int first_row = -1;
        for (int it = ld; it < le; ++it) {
            if (tj < nn && tj < rend[ti] - jbase) {
                acc = __dadd_rn(acc, prod[tj]);
                ++tj;
            } else {
                if (first_row < 0) {
                    first_row = ti;
                    first_val = acc;
                } else {
                    y[g.i0 + ti] = acc;
                }
                acc = 0.0;
                ++ti;
            }
        }
        // inclusive segmented scan of the carries (flag = the thread closed a row)
        int f = first_row >= 0;
        double v = acc;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const double pv = __shfl_up_sync(0xffffffffu, v, d);
            const int pf = __shfl_up_sync(0xffffffffu, f, d);
            if (lane >= d) seg_combine(f, v, pf, pv);
        }
        if (lane == 31) {
            s_wv[wid] = v;
            s_wf[wid] = f;
        }
        __syncthreads();
        int pf = 0;
        double pv = 0.0;
        for (int w = 0; w < wid; ++w) {
            if (s_wf[w]) {
                pv = s_wv[w];
                pf = 1;
            } else {
                pv = __dadd_rn(pv, s_wv[w]);
            }
        }
        double ex = __shfl_up_sync(0xffffffffu, v, 1);
        int exf = __shfl_up_sync(0xffffffffu, f, 1);
        if (lane == 0) {
            ex = pv;
            exf = pf;
        } else if (wid > 0) {
            seg_combine(exf, ex, pf, pv);
        }
        if (first_row >= 0) y[g.i0 + first_row] = __dadd_rn(ex, first_val);
        if (tid == kMgThreads - 1) {
            double tv = v;
            int tf = f;
            if (wid > 0) seg_combine(tf, tv, pf, pv);
            carry_row[t] = (g.i1 < nrows) ? int(g.i1) : -1;
            carry_val[t] = tv;
        }
        fence_proxy_async_smem();  // this thread's generic writes to the stage before the next bulk copy
        __syncthreads();           // stage and s_wv/s_wf free
        if (tid == 0) {
            const int64_t tn = t + int64_t(kMgStages) * gridDim.x;
            if (tn < ntiles) {
                mg_issue(mg_tile(tn, nrows, nnz, tile_row), nrows, ptrs, col, val, stage, bars + st, pol);
            }
        }
    }
}

// rows cut by tile boundaries: the first tile of each run of equal carry rows
// adds the run's carries (tile order) in front of the completing tile's part
__global__ void csr_merge_fixup_kernel(int64_t ntiles, const int* __restrict__ carry_row,
                                       const double* __restrict__ carry_val, double* __restrict__ y,
                                       const int* __restrict__ skip) {
    if (skip != nullptr && *skip) return;
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= ntiles) return;
    const int r = carry_row[t];
    if (r < 0 || (t > 0 && carry_row[t - 1] == r)) return;
    double s = carry_val[t];
    for (int64_t u = t + 1; u < ntiles && carry_row[u] == r; ++u) s = __dadd_rn(s, carry_val[u]);
    y[r] = __dadd_rn(s, y[r]);
}

inline int launch_csr_merge(int64_t nrows, int64_t nnz, const int* ptrs, const int* col, const double* val,
                            const double* x, double* y, void* plan, const int* skip, cudaStream_t st) {
    const int64_t ntiles = csr_merge_tiles(nrows, nnz);
    const MergePlan p = csr_merge_plan_views(plan, nrows, nnz);
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev & 63]) {
        WK_CUDA(cudaFuncSetAttribute(csr_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kMgSmem)));
        attr_set[dev & 63] = true;
    }
    int per_sm = 0;
    WK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, csr_merge_kernel, kMgThreads, kMgSmem));
    int64_t grid = int64_t(sm_count()) * (per_sm > 0 ? per_sm : 1);
    if (grid > ntiles) grid = ntiles;
    csr_merge_kernel<<<(unsigned)grid, kMgThreads, kMgSmem, st>>>(nrows, nnz, ntiles, ptrs, col, val, x, y,
                                                                  p.tile_row, p.carry_row, p.carry_val, skip);
    WK_LAUNCH_CHECK();
    if (ntiles > 1) {
        csr_merge_fixup_kernel<<<(unsigned)ceil_div(ntiles, 256), 256, 0, st>>>(ntiles, p.carry_row, p.carry_val, y,
                                                                               skip);
        WK_LAUNCH_CHECK();
    }
    return 0;
}

inline int build_csr_merge_plan(int64_t nrows, int64_t nnz, const int* ptrs, void* plan, cudaStream_t st) {
    const int64_t ntiles = csr_merge_tiles(nrows, nnz);
    const MergePlan p = csr_merge_plan_views(plan, nrows, nnz);
    csr_merge_plan_kernel<<<(unsigned)ceil_div(ntiles + 1, 256), 256, 0, st>>>(nrows, nnz, ntiles, ptrs, p.tile_row);
    WK_LAUNCH_CHECK();
    return 0;
}

}  // namespace wk
