// Synthetic matrices generated directly in HBM (no host round trip):
//   * constant-coefficient stencils on nx*ny*nz grids (2-D 5-point Poisson of
//     corpus.py:33-50, 3-D 7/27-point Laplacians, 7-point convection-
//     diffusion) as CSR with ascending columns;
//   * R-MAT / Graph500 edges from a counter-based hash (splitmix64), so the
//     CPU oracle (oracle/corpus_ref.py) regenerates the identical matrix;
//   * duplicate summation in the order of `CooMatrix.from_entries`
//     (sparse.py:73-79: lexsort, then 0.0 + v1 + v2 + ... per (row, col)).
#include <algorithm>
#include <vector>

#include "reduce.cuh"

namespace wk {

constexpr int kMaxStencil = 32;

struct Stencil {
    int n;
    int dx[kMaxStencil], dy[kMaxStencil], dz[kMaxStencil];
    double v[kMaxStencil];
};

__device__ __forceinline__ bool stencil_in(const Stencil& s, int p, int64_t i, int64_t j, int64_t k, int64_t nx,
                                           int64_t ny, int64_t nz) {
    const int64_t a = i + s.dx[p], b = j + s.dy[p], c = k + s.dz[p];
    return a >= 0 && a < nx && b >= 0 && b < ny && c >= 0 && c < nz;
}

__global__ void stencil_fill_kernel(int64_t nx, int64_t ny, int64_t nz, Stencil s, const int* __restrict__ ptrs,
                                    int* __restrict__ col, double* __restrict__ val) {
    const int64_t n = nx * ny * nz;
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int64_t i = r % nx, j = (r / nx) % ny, k = r / (nx * ny);
    int64_t e = ptrs[r];
    for (int p = 0; p < s.n; ++p) {
        if (stencil_in(s, p, i, j, k, nx, ny, nz)) {
            col[e] = int(r + (int64_t(s.dz[p]) * ny + s.dy[p]) * nx + s.dx[p]);
            val[e] = s.v[p];
            ++e;
        }
    }
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ double uniform01(uint64_t seed, uint64_t counter) {
    const uint64_t h = splitmix64(seed * 0xD1B54A32D192ED03ull + counter);
    return double(h >> 11) * (1.0 / 9007199254740992.0);
}

__global__ void rmat_kernel(int scale, double a, double b, double c, uint64_t seed, int64_t edge_lo, int64_t count,
                            int64_t* __restrict__ keys, double* __restrict__ vals) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= count) return;
    const uint64_t e = uint64_t(edge_lo + t);
    const uint64_t L = uint64_t(scale) + 1;
    int64_t row = 0, col = 0;
    const double ab = a + b, abc = a + b + c;
    for (int lvl = 0; lvl < scale; ++lvl) {
        const double u = uniform01(seed, e * L + uint64_t(lvl));
        const int64_t bit = int64_t(1) << (scale - 1 - lvl);
        if (u >= ab) row |= bit;
        if ((u >= a && u < ab) || u >= abc) col |= bit;
    }
    keys[t] = row * (int64_t(1) << scale) + col;
    vals[t] = uniform01(seed, e * L + uint64_t(scale));
}

// Duplicate fold of a sorted key array (from_entries, sparse.py:73-79: the
// values of equal (row, col) keys summed as 0.0 + v1 + v2 + ... in input
// order, np.add.at on zeros). Tiles of 2048 keys, 8 consecutive per thread:
//   dedup_count_kernel    heads (key != previous key) per tile
//   (exclusive scan of the tile counts, total in the last slot)
//   dedup_scatter_kernel  the tile staged in shared memory, heads again,
//                         block scan -> output slot, each head folds its
//                         run; the triples are written out coalesced
// Keys are read twice and values once; the round-1 version materialised an
// int64 offset per input key (three passes over 268M keys on R-MAT 24).
constexpr int kDdThreads = 256, kDdItems = 8;
constexpr int64_t kDdTile = int64_t(kDdThreads) * kDdItems;

__device__ __forceinline__ int tile_heads(int64_t n, const int64_t* __restrict__ keys, int64_t base, int64_t (&k)[kDdItems],
                                          unsigned& hmask) {
    int64_t prev = base > 0 && base < n ? keys[base - 1] : 0;
    int c = 0;
    hmask = 0u;
    if (base + kDdItems <= n) {
#pragma unroll
        for (int u = 0; u < kDdItems; u += 2) {
            const longlong2 t = __ldcs(reinterpret_cast<const longlong2*>(keys + base + u));
            k[u] = t.x;
            k[u + 1] = t.y;
        }
    } else {
#pragma unroll
        for (int u = 0; u < kDdItems; ++u) k[u] = base + u < n ? keys[base + u] : 0;
    }
#pragma unroll
    for (int u = 0; u < kDdItems; ++u) {
        const int64_t i = base + u;
        if (i < n && (i == 0 || k[u] != prev)) {
            hmask |= 1u << u;
            ++c;
        }
        prev = k[u];
    }
    return c;
}

__global__ void __launch_bounds__(kDdThreads)
dedup_count_kernel(int64_t n, const int64_t* __restrict__ keys, int64_t* __restrict__ tile_counts) {
    __shared__ int64_t smem[kDdThreads / 32 + 1];
    int64_t k[kDdItems];
    unsigned hm;
    const int c = tile_heads(n, keys, int64_t(blockIdx.x) * kDdTile + int64_t(threadIdx.x) * kDdItems, k, hm);
    int64_t tot;
    block_exclusive_scan<int64_t>(int64_t(c), smem, tot);
    if (threadIdx.x == 0) tile_counts[blockIdx.x] = tot;
}

// The tile's keys and values are staged in shared memory with coalesced
// 16-byte loads, every thread folds the runs that start in its 8 items from
// there (a run that leaves the tile continues from global memory, in order),
// and the tile's unique (row, col, value) triples are staged again and written
// with consecutive threads on consecutive slots. Shared slots are padded by
// one per 8 (dd_pad) so a warp reading its lanes' items 8 apart hits 32
// distinct banks. (Thread-owned items loaded and stored directly left every
// warp access 8 elements apart: 3.8 ms on R-MAT 24, DRAM traffic 1.3x the
// algorithmic bytes from the partial-sector stores; staged without the
// padding, bank conflicts made it 4.1 ms.)
__device__ __forceinline__ int dd_pad(int i) { return i + (i >> 3); }
constexpr int kDdSlots = kDdTile + kDdTile / 8;

// (256, 5): <= 48 registers, five CTAs per SM instead of the four 64
// registers allowed (2.40 -> 1.97 ms same-box; six CTAs spill: 2.35 ms)
__global__ void __launch_bounds__(kDdThreads, 5)
dedup_scatter_kernel(int64_t n, int64_t ncols, const int64_t* __restrict__ keys, const double* __restrict__ vals,
                     const int64_t* __restrict__ tile_offs, int* __restrict__ row, int* __restrict__ col,
                     double* __restrict__ out) {
    __shared__ __align__(16) int64_t sk[kDdSlots];  // keys, then the staged (row, col) pairs
    __shared__ __align__(16) double sv[kDdSlots];   // values, then the staged sums
    __shared__ int64_t smem[kDdThreads / 32 + 1];
    const int64_t t0 = int64_t(blockIdx.x) * kDdTile;
    const int cnt = int(n - t0 < kDdTile ? n - t0 : kDdTile);
    const bool vv = (reinterpret_cast<uintptr_t>(vals) & 15) == 0;
    if (vv && cnt == kDdTile) {
        // full tile: every load of the thread in flight before the first store
        constexpr int kL = kDdTile / (2 * kDdThreads);
        longlong2 kk[kL];
        double2 v2[kL];
#pragma unroll
        for (int q = 0; q < kL; ++q) {
            const int i = 2 * (threadIdx.x + q * kDdThreads);
            kk[q] = __ldcs(reinterpret_cast<const longlong2*>(keys + t0 + i));
            v2[q] = __ldcs(reinterpret_cast<const double2*>(vals + t0 + i));
        }
#pragma unroll
        for (int q = 0; q < kL; ++q) {
            const int i = 2 * (threadIdx.x + q * kDdThreads);
            sk[dd_pad(i)] = kk[q].x;
            sk[dd_pad(i + 1)] = kk[q].y;
            sv[dd_pad(i)] = v2[q].x;
            sv[dd_pad(i + 1)] = v2[q].y;
        }
    } else {
        for (int i = threadIdx.x; i < cnt; i += kDdThreads) {
            sk[dd_pad(i)] = keys[t0 + i];
            sv[dd_pad(i)] = vals[t0 + i];
        }
    }
    __syncthreads();
    const int b0 = threadIdx.x * kDdItems;
    int64_t prev = b0 > 0 ? (b0 - 1 < cnt ? sk[dd_pad(b0 - 1)] : 0) : (t0 > 0 ? keys[t0 - 1] : 0);
    unsigned hm = 0u;
    int c = 0;
#pragma unroll
    for (int u = 0; u < kDdItems; ++u) {
        const int i = b0 + u;
        const int64_t k = i < cnt ? sk[dd_pad(i)] : 0;
        if (i < cnt && (t0 + i == 0 || k != prev)) {
            hm |= 1u << u;
            ++c;
        }
        prev = k;
    }
    int64_t tot;
    const int64_t o0 = block_exclusive_scan<int64_t>(int64_t(c), smem, tot);
    int64_t rk[kDdItems];
    double rs[kDdItems];
#pragma unroll
    for (int u = 0; u < kDdItems; ++u) {
        rk[u] = 0;
        rs[u] = 0.0;
        if (!((hm >> u) & 1u)) continue;
        const int64_t key = sk[dd_pad(b0 + u)];
        double acc = 0.0;
        int j = b0 + u;
        for (; j < cnt && sk[dd_pad(j)] == key; ++j) acc += sv[dd_pad(j)];
        if (j == cnt)  // the run goes on past the tile
            for (int64_t g = t0 + cnt; g < n && keys[g] == key; ++g) acc += vals[g];
        rk[u] = key;
        rs[u] = acc;
    }
    __syncthreads();  // every read of the staged input is done
    const bool pow2 = (ncols & (ncols - 1)) == 0;  // R-MAT: no 64-bit division
    const int sh = pow2 ? __ffsll(ncols) - 1 : 0;
    int2* rc = reinterpret_cast<int2*>(sk);
    int o = int(o0);
#pragma unroll
    for (int u = 0; u < kDdItems; ++u) {
        if (!((hm >> u) & 1u)) continue;
        const int64_t key = rk[u];
        if (pow2) {
            rc[dd_pad(o)] = make_int2(int(key >> sh), int(key & (ncols - 1)));
        } else {
            const int64_t q = key / ncols;
            rc[dd_pad(o)] = make_int2(int(q), int(key - q * ncols));
        }
        sv[dd_pad(o)] = rs[u];
        ++o;
    }
    __syncthreads();
    const int64_t base = tile_offs[blockIdx.x];
    for (int i = threadIdx.x; i < int(tot); i += kDdThreads) {
        const int2 p = rc[dd_pad(i)];
        __stcs(row + base + i, p.x);
        __stcs(col + base + i, p.y);
        __stcs(out + base + i, sv[dd_pad(i)]);
    }
}

}  // namespace wk

using namespace wk;

extern "C" {

int wk_gen_stencil_csr(int64_t nx, int64_t ny, int64_t nz, int32_t npoints, const int32_t* h_dx,
                       const int32_t* h_dy, const int32_t* h_dz, const double* h_values, int32_t* row_ptrs,
                       int32_t* col_idx, double* values, void* scan_ws, wk_stream_t stream) {
    clear_error();
    WK_REQUIRE(npoints >= 0 && npoints <= kMaxStencil, WK_ERR_INVALID, "at most %d stencil points", kMaxStencil);
    WK_REQUIRE(nx >= 0 && ny >= 0 && nz >= 0, WK_ERR_INVALID, "negative grid size");
    // order points by linear offset so every row's columns ascend
    std::vector<int> order(npoints);
    for (int p = 0; p < npoints; ++p) order[p] = p;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
        const int64_t oa = (int64_t(h_dz[a]) * ny + h_dy[a]) * nx + h_dx[a];
        const int64_t ob = (int64_t(h_dz[b]) * ny + h_dy[b]) * nx + h_dx[b];
        return oa < ob;
    });
    Stencil s;
    s.n = npoints;
    for (int p = 0; p < npoints; ++p) {
        s.dx[p] = h_dx[order[p]];
        s.dy[p] = h_dy[order[p]];
        s.dz[p] = h_dz[order[p]];
        s.v[p] = h_values[order[p]];
    }
    const int64_t n = nx * ny * nz;
    cudaStream_t st = as_stream(stream);
    if (col_idx == nullptr) {
        auto len = [=] __device__(int64_t r) {
            const int64_t i = r % nx, j = (r / nx) % ny, k = r / (nx * ny);
            int c = 0;
            for (int p = 0; p < s.n; ++p) c += stencil_in(s, p, i, j, k, nx, ny, nz);
            return int64_t(c);
        };
        return exclusive_scan(n, len, row_ptrs, scan_ws, st);
    }
    if (n == 0) return 0;
    stencil_fill_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(nx, ny, nz, s, row_ptrs, col_idx, values);
    WK_LAUNCH_CHECK();
    return 0;
}

int wk_gen_rmat_edges(int32_t scale, int32_t edge_factor, double a, double b, double c, uint64_t seed,
                      int64_t edge_lo, int64_t count, int64_t* keys, double* values, wk_stream_t stream) {
    clear_error();
    (void)edge_factor;
    WK_REQUIRE(scale >= 1 && scale <= 30, WK_ERR_INVALID, "R-MAT scale must be in [1, 30]");
    if (count == 0) return 0;
    rmat_kernel<<<(unsigned)ceil_div(count, 256), 256, 0, as_stream(stream)>>>(scale, a, b, c, seed, edge_lo, count,
                                                                             keys, values);
    WK_LAUNCH_CHECK();
    return 0;
}

int64_t wk_coo_dedup_tiles(int64_t n) { return ceil_div(n, kDdTile); }

int64_t wk_coo_dedup_workspace(int64_t n) { return (wk_coo_dedup_tiles(n) + 1) * 8; }

int wk_coo_dedup_count(int64_t n, const int64_t* keys, void* work, wk_stream_t stream) {
    clear_error();
    WK_REQUIRE((reinterpret_cast<uintptr_t>(keys) & 15) == 0 && (reinterpret_cast<uintptr_t>(work) & 7) == 0,
               WK_ERR_INVALID, "dedup keys must be 16-byte aligned");
    cudaStream_t st = as_stream(stream);
    const int64_t nt = wk_coo_dedup_tiles(n);
    int64_t* tc = reinterpret_cast<int64_t*>(work);
    WK_CUDA(cudaMemsetAsync(tc + nt, 0, 8, st));
    if (nt) {
        dedup_count_kernel<<<(unsigned)nt, kDdThreads, 0, st>>>(n, keys, tc);
        WK_LAUNCH_CHECK();
    }
    return scan_tile_sums_exclusive_launch(nt + 1, tc, st);  // tc[nt] = number of unique keys
}

int wk_coo_dedup_scatter(int64_t n, int64_t ncols, const int64_t* keys, const double* values, const void* work,
                         int32_t* row, int32_t* col, double* out_values, wk_stream_t stream) {
    clear_error();
    WK_REQUIRE((reinterpret_cast<uintptr_t>(keys) & 15) == 0, WK_ERR_INVALID, "dedup keys must be 16-byte aligned");
    const int64_t nt = wk_coo_dedup_tiles(n);
    if (nt == 0) return 0;
    dedup_scatter_kernel<<<(unsigned)nt, kDdThreads, 0, as_stream(stream)>>>(
        n, ncols > 0 ? ncols : 1, keys, values, reinterpret_cast<const int64_t*>(work), row, col, out_values);
    WK_LAUNCH_CHECK();
    return 0;
}

}  // extern "C"
