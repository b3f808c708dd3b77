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

__global__ void sum_dups_kernel(int64_t n, int64_t ncols, const int64_t* __restrict__ keys,
                                const double* __restrict__ vals, const int64_t* __restrict__ offsets,
                                int* __restrict__ row, int* __restrict__ col, double* __restrict__ out) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t key = keys[i];
    if (i > 0 && keys[i - 1] == key) return;
    double acc = 0.0;
    for (int64_t j = i; j < n && keys[j] == key; ++j) acc += vals[j];
    const int64_t o = offsets[i];
    if ((ncols & (ncols - 1)) == 0) {  // power of two (R-MAT): no 64-bit division
        const int sh = __ffsll(ncols) - 1;
        row[o] = int(key >> sh);
        col[o] = int(key & (ncols - 1));
    } else {
        row[o] = int(key / ncols);
        col[o] = int(key - (key / ncols) * ncols);
    }
    out[o] = acc;
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

int wk_coo_unique_offsets(int64_t n, const int64_t* keys, int64_t* offsets, void* scan_ws, wk_stream_t stream) {
    clear_error();
    auto head = [=] __device__(int64_t i) { return int64_t(i == 0 || keys[i] != keys[i - 1]); };
    return exclusive_scan(n, head, offsets, scan_ws, as_stream(stream));
}

int wk_coo_sum_duplicates(int64_t n, int64_t ncols, const int64_t* keys, const double* values,
                          const int64_t* offsets, int32_t* row, int32_t* col, double* out_values,
                          wk_stream_t stream) {
    clear_error();
    if (n == 0) return 0;
    sum_dups_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, as_stream(stream)>>>(n, ncols > 0 ? ncols : 1, keys, values, offsets,
                                                                             row, col, out_values);
    WK_LAUNCH_CHECK();
    return 0;
}

}  // extern "C"
