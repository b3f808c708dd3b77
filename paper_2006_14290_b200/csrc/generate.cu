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
//   dedup_scatter_kernel  heads again, block scan -> output slot, each head
//                         folds its run and writes (row, col, value)
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

__global__ void __launch_bounds__(kDdThreads)
dedup_scatter_kernel(int64_t n, int64_t ncols, const int64_t* __restrict__ keys, const double* __restrict__ vals,
                     const int64_t* __restrict__ tile_offs, int* __restrict__ row, int* __restrict__ col,
                     double* __restrict__ out) {
    __shared__ int64_t smem[kDdThreads / 32 + 1];
    const int64_t base = int64_t(blockIdx.x) * kDdTile + int64_t(threadIdx.x) * kDdItems;
    int64_t k[kDdItems];
    unsigned hm;
    const int c = tile_heads(n, keys, base, k, hm);
    int64_t tot;
    int64_t o = block_exclusive_scan<int64_t>(int64_t(c), smem, tot) + tile_offs[blockIdx.x];
    const bool pow2 = (ncols & (ncols - 1)) == 0;  // R-MAT: no 64-bit division
    const int sh = pow2 ? __ffsll(ncols) - 1 : 0;
#pragma unroll
    for (int u = 0; u < kDdItems; ++u) {
        if (!((hm >> u) & 1u)) continue;
        const int64_t key = k[u];
        double acc = 0.0;
        for (int64_t j = base + u; j < n && keys[j] == key; ++j) acc += vals[j];
        if (pow2) {
            row[o] = int(key >> sh);
            col[o] = int(key & (ncols - 1));
        } else {
            const int64_t q = key / ncols;
            row[o] = int(q);
            col[o] = int(key - q * ncols);
        }
        out[o] = acc;
        ++o;
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
