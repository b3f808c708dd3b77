// Format conversions on the device. Every output array is bit-identical to
// the reference's host conversion:
//   coo_to_csr     sparse.py:212-216  (row counts -> cumsum)
//   coo_to_sellp   sparse.py:219-242  (per-slice max length -> cumulative
//                  widths -> zero-filled storage -> k = sets[s]*ss + j*ss + l)
//   CSR -> ELL     the same rule with one slice of stride `stride`
//   CSR -> Hybrid  ELL(width) of each row's leading entries + row-major COO rest
//
// The scatter kernels stage a row block's CSR entries in shared memory with
// coalesced loads and then write the column-major destination with
// consecutive threads on consecutive addresses (the transpose-through-smem
// pattern), so both sides of the conversion stream at full width.
#include "reduce.cuh"

namespace wk {

constexpr int kConvThreads = 256;
constexpr int kStageCap = 2048;  // staged entries per block (24 KB)

// Row lengths and per-slice maximum lengths (sparse.py:225-228) in one pass:
// lengths[r] = ptrs[r+1] - ptrs[r]; out[s + 1] = max over the slice's rows
// (butterfly within ss <= 32 lanes, warp maxima combined in shared memory for
// ss <= 256, atomicMax into a zeroed array beyond).
__global__ void __launch_bounds__(256) slice_widths_kernel(int64_t nrows, int log2ss, const int* __restrict__ ptrs,
                                                           int* __restrict__ lengths, int64_t* __restrict__ out) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t r = int64_t(blockIdx.x) * 256 + tid;
    const int len = r < nrows ? ptrs[r + 1] - ptrs[r] : 0;
    if (r < nrows) lengths[r] = len;
    const int ss = 1 << log2ss;
    const int g = ss < 32 ? ss : 32;
    int m = len;
    for (int d = 1; d < g; d <<= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, d));
    if (ss <= 32) {
        if ((tid & (ss - 1)) == 0 && r < nrows) out[(r >> log2ss) + 1] = m;
        return;
    }
    __shared__ int wm[8];
    if (lane == 0) wm[warp] = m;
    __syncthreads();
    if (ss <= 256) {
        const int per = ss >> 5;
        if (tid < (256 >> log2ss)) {
            const int64_t r0 = int64_t(blockIdx.x) * 256 + int64_t(tid) * ss;
            if (r0 < nrows) {
                int mm = 0;
                for (int k = 0; k < per; ++k) mm = max(mm, wm[tid * per + k]);
                out[(r0 >> log2ss) + 1] = mm;
            }
        }
    } else if (tid == 0) {
        int mm = 0;
        for (int k = 0; k < 8; ++k) mm = max(mm, wm[k]);
        atomicMax(reinterpret_cast<unsigned long long*>(out + ((int64_t(blockIdx.x) * 256) >> log2ss) + 1),
                  (unsigned long long)mm);
    }
}

__global__ void row_lengths_kernel(int64_t nrows, const int* __restrict__ ptrs, int* __restrict__ lengths) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r < nrows) lengths[r] = ptrs[r + 1] - ptrs[r];
}

// Column-major scatter of rows [r0, r0 + nrb) into destination slots
// dst(j, l) = dbase + j * dstride + l for j < width, l < nrb_slots (rows
// beyond nrows or j >= len are padding (0, 0.0)). Rows longer than `width`
// are clipped (the Hybrid ELL part).
__device__ void scatter_block(int64_t nrows, int64_t r0, int64_t nrb_slots, int64_t width, int64_t dbase,
                              int64_t dstride, const int* __restrict__ ptrs, const int* __restrict__ col,
                              const double* __restrict__ val, int* __restrict__ dcol, double* __restrict__ dval,
                              int* s_col, double* s_val, int* s_ptr) {
    const int64_t r_hi = (r0 + nrb_slots < nrows) ? r0 + nrb_slots : nrows;
    const int64_t nreal = r_hi > r0 ? r_hi - r0 : 0;
    const int64_t src_lo = nreal ? ptrs[r0] : 0;
    const int64_t src_hi = nreal ? ptrs[r_hi] : 0;
    const int64_t cnt = src_hi - src_lo;
    const bool staged = cnt <= kStageCap && nrb_slots <= kConvThreads * 4;
    if (staged) {
        // (no row pointers to stage for a block of padding rows only: r0 may lie past nrows)
        for (int64_t i = threadIdx.x; nreal > 0 && i <= nreal; i += kConvThreads) s_ptr[i] = ptrs[r0 + i] - int(src_lo);
        for (int64_t i = threadIdx.x; i < cnt; i += kConvThreads) {
            s_col[i] = __ldcs(col + src_lo + i);
            s_val[i] = __ldcs(val + src_lo + i);
        }
        __syncthreads();
    }
    const int64_t total = width * nrb_slots;
    const bool pow2 = (nrb_slots & (nrb_slots - 1)) == 0;
    const int sh = pow2 ? __ffsll(nrb_slots) - 1 : 0;
    for (int64_t e = threadIdx.x; e < total; e += kConvThreads) {
        const int64_t j = pow2 ? (e >> sh) : e / nrb_slots;
        const int64_t l = e - j * nrb_slots;
        int c = 0;
        double v = 0.0;
        if (l < nreal) {
            if (staged) {
                const int lo = s_ptr[l], hi = s_ptr[l + 1];
                if (j < hi - lo) {
                    c = s_col[lo + j];
                    v = s_val[lo + j];
                }
            } else {
                const int64_t lo = ptrs[r0 + l], hi = ptrs[r0 + l + 1];
                if (j < hi - lo) {
                    c = col[lo + j];
                    v = val[lo + j];
                }
            }
        }
        const int64_t d = dbase + j * dstride + l;
        __stcs(dcol + d, c);
        __stcs(dval + d, v);
    }
}

__global__ void __launch_bounds__(kConvThreads)
sellp_fill_kernel(int64_t nrows, int log2ss, const int* __restrict__ ptrs, const int* __restrict__ col,
                  const double* __restrict__ val, const int64_t* __restrict__ sets, int* __restrict__ dcol,
                  double* __restrict__ dval) {
    __shared__ int s_col[kStageCap];
    __shared__ double s_val[kStageCap];
    __shared__ int s_ptr[kConvThreads * 4 + 1];
    const int64_t s = blockIdx.x;
    const int64_t ss = int64_t(1) << log2ss;
    const int64_t w = sets[s + 1] - sets[s];
    scatter_block(nrows, s * ss, ss, w, sets[s] * ss, ss, ptrs, col, val, dcol, dval, s_col, s_val, s_ptr);
}

// CSR -> SELL-P / ELL fill with TMA-staged input (16-byte aligned CSR arrays,
// 4 <= rows per tile <= 256; the staged-scatter kernels above otherwise). Persistent CTAs (2 per SM) walk tiles of R
// rows (SELL-P: one slice, R = ss; ELL: R = 2^k <= 256 rows with R * width <=
// the stage capacity), t = blockIdx.x + i * gridDim.x. Thread 0 bulk-loads
// the next tile's CSR range (values and column indices are contiguous per
// tile; the range is widened to a multiple of 4 entries for 16-byte
// alignment) into the other stage of a 2-deep ring, one mbarrier per stage;
// the tile's row pointers are loaded into registers one iteration ahead. 256
// threads write the current tile's column-major image from shared memory with
// consecutive threads on consecutive destination addresses (entry j of row l
// at dbase + j * dstride + l, padding (0, 0.0)), plain streaming stores —
// staging the image for a TMA bulk store was slower (the store ring
// serialises the CTA). Tiles whose range exceeds a stage, or whose widened
// range passes nnz, read global memory directly. 27-point 200^3: SELL-P fill
// 1.015 -> 0.876 ms, ELL fill 1.149 -> 0.838 ms (wider ELL tiles: 1 KB
// contiguous stores per column instead of 512 B). (sparse.py:219-242.)
// entries per stage (48 KB). SELL-P fill: one stage, three CTAs per SM
// (0.99 -> 0.90 ms for the 27-point 200^3 conversion: more CTAs beat the
// in-CTA prefetch); ELL fill: two stages, two CTAs (one stage: 0.89 -> 0.95
// ms). Grids are sized by the occupancy calculator.
constexpr int kFillCap = 4096;

template <int NS, bool kEll, int C = kFillCap>
__global__ void __launch_bounds__(kConvThreads, NS == 1 ? 3 : 2)
fill_tma_kernel(int64_t nrows, int log2r, int64_t ntiles, const int* __restrict__ ptrs, const int* __restrict__ col,
                const double* __restrict__ val, const int64_t* __restrict__ sets, int64_t width, int64_t stride,
                int* __restrict__ dcol, double* __restrict__ dval, int* __restrict__ dlen) {
    extern __shared__ __align__(128) unsigned char smem[];
    double* in_val = reinterpret_cast<double*>(smem);                  // [NS][C]
    int* in_col = reinterpret_cast<int*>(in_val + NS * C);             // [NS][C]
    int* s_ptr = in_col + NS * C;                                      // [R + 1], R <= 256
    long long* s_lo4 = reinterpret_cast<long long*>(s_ptr + 260);     // [NS] aligned range start, -1 = direct
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_lo4 + NS);         // [NS]
    const int tid = threadIdx.x;
    const int64_t R = int64_t(1) << log2r;
    if (tid == 0) {
        for (int st = 0; st < NS; ++st) mbar_init(bars + st, 1);
        fence_mbar_init();
    }
    __syncthreads();
    const int64_t nnz = ptrs[nrows];
    const uint64_t pol = policy_evict_first();
    auto real_rows = [&](int64_t r0) -> int64_t { return r0 >= nrows ? 0 : (r0 + R < nrows ? R : nrows - r0); };
    auto issue = [&](int64_t i) {  // thread 0
        const int64_t t = blockIdx.x + i * gridDim.x;
        if (t >= ntiles) return;
        const int st = int(i % NS);
        const int64_t r0 = t * R, nreal = real_rows(r0);
        const int64_t lo = nreal ? ptrs[r0] : 0, hi = nreal ? ptrs[r0 + nreal] : 0;
        const int64_t lo4 = lo & ~int64_t(3), hi4 = (hi + 3) & ~int64_t(3);
        const bool fits = hi4 <= nnz && hi4 - lo4 <= C;
        s_lo4[st] = fits ? lo4 : -1;
        if (fits && hi4 > lo4) {
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(bars + st, uint32_t(hi4 - lo4) * 12u);
            bulk_g2s_evict_first(in_val + st * C, val + lo4, uint32_t(hi4 - lo4) * 8u, bars + st, pol);
            bulk_g2s_evict_first(in_col + st * C, col + lo4, uint32_t(hi4 - lo4) * 4u, bars + st, pol);
        } else {
            mbar_arrive(bars + st);
        }
    };
    if (tid == 0)
        for (int k = 0; k < NS - 1; ++k) issue(k);
    // row pointers of the next tile are loaded one iteration ahead (registers)
    auto load_ptrs = [&](int64_t t, int& p0, int& p1) {
        const int64_t r0 = t * R, nreal = t < ntiles ? real_rows(r0) : 0;
        // nothing to read past the last tile or for tiles of padding rows only
        p0 = (nreal > 0 && tid <= nreal) ? ptrs[r0 + tid] : 0;
        p1 = (tid == 0 && R <= nreal) ? ptrs[r0 + R] : 0;  // entry R (thread 0), R == blockDim
    };
    int p0, p1;
    load_ptrs(blockIdx.x, p0, p1);
    for (int64_t i = 0;; ++i) {
        const int64_t t = blockIdx.x + i * gridDim.x;
        if (t >= ntiles) break;
        const int st = int(i % NS);
        if (tid == 0) issue(i + NS - 1);
        const int64_t r0 = t * R, nreal = real_rows(r0);
        if (tid <= nreal) s_ptr[tid] = p0;
        if (tid == 0 && R <= nreal) s_ptr[R] = p1;
        load_ptrs(t + gridDim.x, p0, p1);
        int64_t w, dbase, dstride, nslots;
        if (kEll) {
            w = width;
            dbase = r0;
            dstride = stride;
            nslots = (r0 + R <= stride) ? R : stride - r0;
        } else {
            const int64_t s0 = sets[t];
            w = sets[t + 1] - s0;
            dbase = s0 * R;
            dstride = R;
            nslots = R;
        }
        mbar_wait(bars + st, uint32_t((i / NS) & 1));
        __syncthreads();
        if (kEll && tid < nreal) {
            const int len = s_ptr[tid + 1] - s_ptr[tid];
            dlen[r0 + tid] = len < width ? len : int(width);
        }
        const long long lo4 = s_lo4[st];
        const double* iv = in_val + st * C;
        const int* ic = in_col + st * C;
        const int64_t total = w << log2r;
        for (int64_t e = tid; e < total; e += kConvThreads) {
            const int64_t j = e >> log2r, l = e & (R - 1);
            if (kEll && l >= nslots) continue;
            int c = 0;
            double v = 0.0;
            if (l < nreal) {
                const int a = s_ptr[l], b = s_ptr[l + 1];
                if (j < b - a) {
                    if (lo4 >= 0) {
                        const int k = int(a + j - lo4);
                        c = ic[k];
                        v = iv[k];
                    } else {
                        c = col[a + j];
                        v = val[a + j];
                    }
                }
            }
            const int64_t d = dbase + j * dstride + l;
            __stcs(dcol + d, c);
            __stcs(dval + d, v);
        }
        __syncthreads();  // in[st], s_ptr free for the next tile
    }
}

template <int NS, bool kEll, int C = kFillCap>
int launch_fill_tma(int64_t nrows, int log2r, int64_t ntiles, const int* ptrs, const int* col, const double* val,
                    const int64_t* sets, int64_t width, int64_t stride, int* dcol, double* dval, int* dlen,
                    cudaStream_t st) {
    constexpr size_t smem = size_t(NS) * C * 12 + 260 * 4 + NS * 8 + NS * 8;
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev & 63]) {
        WK_CUDA(cudaFuncSetAttribute(fill_tma_kernel<NS, kEll, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(smem)));
        attr_set[dev & 63] = true;
    }
    int per_sm = 0;  // persistent grid: every CTA the SM can hold
    WK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fill_tma_kernel<NS, kEll, C>, kConvThreads, smem));
    int64_t grid = int64_t(sm_count()) * (per_sm > 0 ? per_sm : 1);
    if (grid > ntiles) grid = ntiles;
    fill_tma_kernel<NS, kEll, C><<<(unsigned)grid, kConvThreads, smem, st>>>(nrows, log2r, ntiles, ptrs, col, val, sets,
                                                                        width, stride, dcol, dval, dlen);
    WK_LAUNCH_CHECK();
    return 0;
}

static bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// `rpb` rows per block (a power of two <= kConvThreads chosen so that the
// block's CSR range fits the shared-memory stage: width 27 -> 64 rows, 1728
// entries), i.e. coalesced staged reads and 512-byte contiguous value stores.
__global__ void __launch_bounds__(kConvThreads)
ell_fill_kernel(int64_t nrows, int64_t width, int64_t stride, int64_t rpb, const int* __restrict__ ptrs,
                const int* __restrict__ col, const double* __restrict__ val, int* __restrict__ dcol,
                double* __restrict__ dval, int* __restrict__ dlen) {
    __shared__ int s_col[kStageCap];
    __shared__ double s_val[kStageCap];
    __shared__ int s_ptr[kConvThreads * 4 + 1];
    const int64_t r0 = int64_t(blockIdx.x) * rpb;
    const int64_t nslots = (r0 + rpb <= stride) ? rpb : stride - r0;
    if (threadIdx.x < rpb) {
        const int64_t r = r0 + threadIdx.x;
        if (r < nrows) {
            const int len = ptrs[r + 1] - ptrs[r];
            dlen[r] = len < width ? len : int(width);
        }
    }
    scatter_block(nrows, r0, nslots, width, r0, stride, ptrs, col, val, dcol, dval, s_col, s_val, s_ptr);
}

// COO remainder of CSR->Hybrid, in two kernels.
//
// hybrid_coo_fill_kernel: a warp takes 32 consecutive rows (one row-pointer
// pair per lane), scans their overflow counts (entries past `width`) and
// copies the group's overflow as ONE flattened run: the destination is
// contiguous (offsets[r0] ..), so every pass writes 32 consecutive COO entries
// and each lane finds its row by a 5-step binary search over the scanned
// counts in registers. Rows with no overflow (56% of R-MAT rows are empty)
// cost one lane of one load. A row with more than kHybLong overflow entries is
// not copied here: its segments of kHybSeg entries are appended to a work list
// (one atomic per long row), so no single warp walks R-MAT's
// heaviest rows (238k entries) or their 32-row group (~1M entries) alone.
// hybrid_coo_long_kernel: the warps of the whole grid take the listed
// segments round-robin, one contiguous copy of <= kHybSeg entries each.
// (The first version, a warp per row: 4.9 ms on R-MAT scale 24, width 8.)
constexpr int kHybLong = 256;
constexpr int kHybSeg = 4096;

__global__ void __launch_bounds__(256)
hybrid_coo_fill_kernel(int64_t nrows, int64_t width, const int* __restrict__ ptrs, const int* __restrict__ col,
                       const double* __restrict__ val, const int64_t* __restrict__ offsets, int* __restrict__ crow,
                       int* __restrict__ ccol, double* __restrict__ cval, unsigned long long* __restrict__ nseg,
                       int2* __restrict__ segs) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    constexpr int kU = 8;
    for (int64_t r0 = ((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * 32; r0 < nrows; r0 += warps * 32) {
        const int64_t r = r0 + lane;
        int lo = 0, cnt = 0;
        if (r < nrows) {
            const int p0 = __ldcs(ptrs + r), p1 = __ldcs(ptrs + r + 1);
            lo = p0 + int(width < p1 - p0 ? width : p1 - p0);
            cnt = p1 - lo;
        }
        if (cnt > kHybLong) {  // long row: list its segments for the second kernel
            const int ns = (cnt + kHybSeg - 1) / kHybSeg;
            const unsigned long long at = atomicAdd(nseg, (unsigned long long)ns);
            for (int q = 0; q < ns; ++q) segs[at + q] = make_int2(int(r), q);
            cnt = 0;
        }
        int incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int o = __shfl_up_sync(FULL, incl, d);
            if (lane >= d) incl += o;
        }
        const int total = __shfl_sync(FULL, incl, 31);
        if (total == 0) continue;
        const int excl = incl - cnt;
        for (int d0 = 0; d0 < total; d0 += 32 * kU) {
            int src[kU], row[kU];
            int64_t dst[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int d = d0 + u * 32 + lane;
                int j = 0;
#pragma unroll
                for (int s = 16; s > 0; s >>= 1) {
                    const int e = __shfl_sync(FULL, excl, j + s);
                    if (e <= d) j += s;
                }
                const int off = d - __shfl_sync(FULL, excl, j);
                src[u] = __shfl_sync(FULL, lo, j) + off;
                row[u] = int(r0) + j;
                dst[u] = off;  // destination = offsets[row] + off (rows of a group need not be adjacent
                               // in the remainder: a long row between them is copied elsewhere)
            }
            int c[kU];
            double v[kU];
            int64_t o[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const bool ok = d0 + u * 32 + lane < total;
                c[u] = ok ? __ldcs(col + src[u]) : 0;
                v[u] = ok ? __ldcs(val + src[u]) : 0.0;
                o[u] = ok ? __ldg(offsets + row[u]) : 0;
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                if (d0 + u * 32 + lane < total) {
                    const int64_t at = o[u] + dst[u];
                    __stcs(crow + at, row[u]);
                    __stcs(ccol + at, c[u]);
                    __stcs(cval + at, v[u]);
                }
            }
        }
    }
}

__global__ void __launch_bounds__(256)
hybrid_coo_long_kernel(int64_t width, const int* __restrict__ ptrs, const int* __restrict__ col,
                       const double* __restrict__ val, const int64_t* __restrict__ offsets, int* __restrict__ crow,
                       int* __restrict__ ccol, double* __restrict__ cval, const unsigned long long* __restrict__ nseg,
                       const int2* __restrict__ segs) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    const int64_t n = int64_t(*nseg);
    constexpr int kU = 8;
    for (int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
        const int2 sg = segs[i];
        const int p0 = ptrs[sg.x], p1 = ptrs[sg.x + 1];
        const int lo = p0 + int(width), cnt = p1 - lo;
        const int s0 = sg.y * kHybSeg;
        const int s1 = (cnt - s0 < kHybSeg) ? cnt : s0 + kHybSeg;
        const int64_t base = offsets[sg.x];
        for (int k0 = s0; k0 < s1; k0 += 32 * kU) {
            int c[kU];
            double v[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int k = k0 + u * 32 + lane;
                c[u] = k < s1 ? __ldcs(col + lo + k) : 0;
                v[u] = k < s1 ? __ldcs(val + lo + k) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int k = k0 + u * 32 + lane;
                if (k < s1) {
                    __stcs(crow + base + k, sg.x);
                    __stcs(ccol + base + k, c[u]);
                    __stcs(cval + base + k, v[u]);
                }
            }
        }
    }
}

// first[r] style boundary fill: for sorted row indices, row_ptrs[r] =
// lower_bound(row_idx, r), computed from the row changes.
// row_ptrs from sorted row indices: entry k starts rows (row[k-1], row[k]]
// (k = nnz closes the rows up to nrows). Eight entries per thread from two
// 16-byte loads when row_idx is aligned (one entry and two scalar loads per
// thread took 0.73 ms on R-MAT 24).
constexpr int kPtrItems = 8;
__global__ void __launch_bounds__(256)
coo_ptrs_kernel(int64_t nrows, int64_t nnz, const int* __restrict__ row, int* __restrict__ ptrs, int vec) {
    const int64_t k0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * kPtrItems;
    if (k0 > nnz) return;
    int cur[kPtrItems];
    if (vec && k0 + kPtrItems <= nnz) {
        const int4 a = __ldcs(reinterpret_cast<const int4*>(row + k0));
        const int4 b = __ldcs(reinterpret_cast<const int4*>(row + k0 + 4));
        cur[0] = a.x, cur[1] = a.y, cur[2] = a.z, cur[3] = a.w;
        cur[4] = b.x, cur[5] = b.y, cur[6] = b.z, cur[7] = b.w;
    } else {
#pragma unroll
        for (int u = 0; u < kPtrItems; ++u) {
            const int64_t k = k0 + u;
            cur[u] = k < nnz ? row[k] : int(nrows);
        }
    }
    int64_t prev = k0 == 0 ? -1 : row[k0 - 1];
#pragma unroll
    for (int u = 0; u < kPtrItems; ++u) {
        const int64_t k = k0 + u;
        if (k > nnz) break;
        const int64_t c = k == nnz ? nrows : cur[u];
        for (int64_t r = prev + 1; r <= c; ++r) ptrs[r] = int(k);
        prev = c;
    }
}

__global__ void csr_rows_kernel(int64_t nrows, const int* __restrict__ ptrs, int* __restrict__ row) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < nrows; r += warps)
        for (int64_t k = ptrs[r] + lane; k < ptrs[r + 1]; k += 32) row[k] = int(r);
}

static int warp_grid(int64_t nrows) {
    int64_t b = ceil_div(nrows * 32, 256);
    const int64_t cap = int64_t(sm_count()) * 32;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return int(b);
}

__global__ void __launch_bounds__(256) max_len_kernel(int64_t nrows, const int* __restrict__ ptrs,
                                                      unsigned long long* __restrict__ result) {
    unsigned long long m = 0;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < nrows; r += stride) {
        const unsigned long long len = (unsigned long long)(ptrs[r + 1] - ptrs[r]);
        m = len > m ? len : m;
    }
    for (int d = 16; d > 0; d >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, m, d);
        m = o > m ? o : m;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(result, m);
}

// Row-length histogram: bins below kHistSmem are counted in shared memory
// with warp-aggregated increments (one atomic per distinct length per warp:
// R-MAT has 56% empty rows, so per-row global atomics serialised on bin 0 —
// 7 ms for 16.7M rows), flushed with one global atomic per non-empty bin per
// block; longer rows (rare) go straight to global memory.
constexpr int kHistSmem = 4096;

__global__ void __launch_bounds__(512) len_hist_kernel(int64_t nrows, int64_t nbins, const int* __restrict__ ptrs,
                                                       unsigned long long* __restrict__ hist) {
    __shared__ unsigned sh[kHistSmem];
    const int nb_s = nbins < kHistSmem ? int(nbins) : kHistSmem;
    for (int i = threadIdx.x; i < nb_s; i += blockDim.x) sh[i] = 0u;
    __syncthreads();
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < nrows; r += stride) {
        int64_t len = __ldcs(ptrs + r + 1) - __ldcs(ptrs + r);
        if (len > nbins - 1) len = nbins - 1;
        if (len < nb_s) {
            const unsigned peers = __match_any_sync(__activemask(), int(len));
            if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(sh + len, unsigned(__popc(peers)));
        } else {
            atomicAdd(hist + len, 1ull);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nb_s; i += blockDim.x)
        if (sh[i]) atomicAdd(hist + i, (unsigned long long)sh[i]);
}

// Host-uploaded SELL-P / ELL: every slot past a row's length becomes the
// reference padding (col 0, val 0.0, sparse.py:230-232), whatever the
// caller's arrays held there (the SpMV kernels fold full slices).
__global__ void __launch_bounds__(256) sellp_zero_padding_kernel(int64_t nrows, int64_t ss, int64_t nslices,
                                                                 const int64_t* __restrict__ sets,
                                                                 const int* __restrict__ lens, int* __restrict__ col,
                                                                 double* __restrict__ val) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < nslices * ss; t += stride) {
        const int64_t s = t / ss, local = t - s * ss;
        const int64_t base = sets[s] * ss, w = sets[s + 1] - sets[s];
        const int64_t len = t < nrows ? lens[t] : 0;
        for (int64_t j = len; j < w; ++j) {
            col[base + j * ss + local] = 0;
            val[base + j * ss + local] = 0.0;
        }
    }
}

__global__ void __launch_bounds__(256) ell_zero_padding_kernel(int64_t nrows, int64_t width, int64_t stride_,
                                                               const int* __restrict__ lens, int* __restrict__ col,
                                                               double* __restrict__ val) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < stride_; r += stride) {
        const int64_t len = r < nrows ? lens[r] : 0;
        for (int64_t j = len; j < width; ++j) {
            col[j * stride_ + r] = 0;
            val[j * stride_ + r] = 0.0;
        }
    }
}

}  // namespace wk

using namespace wk;

extern "C" {

int wk_csr_row_lengths(int64_t nrows, const int32_t* row_ptrs, int32_t* row_lengths, wk_stream_t stream) {
    clear_error();
    if (nrows == 0) return 0;
    row_lengths_kernel<<<(unsigned)ceil_div(nrows, 256), 256, 0, as_stream(stream)>>>(nrows, row_ptrs, row_lengths);
    WK_LAUNCH_CHECK();
    return 0;
}

int wk_csr_max_row_length(int64_t nrows, const int32_t* row_ptrs, int64_t* result, wk_stream_t stream) {
    clear_error();
    cudaStream_t st = as_stream(stream);
    WK_CUDA(cudaMemsetAsync(result, 0, sizeof(int64_t), st));
    if (nrows == 0) return 0;
    int64_t blocks = ceil_div(nrows, 256);
    if (blocks > int64_t(sm_count()) * 8) blocks = int64_t(sm_count()) * 8;
    max_len_kernel<<<(unsigned)blocks, 256, 0, st>>>(nrows, row_ptrs, reinterpret_cast<unsigned long long*>(result));
    WK_LAUNCH_CHECK();
    return 0;
}

int wk_csr_row_length_histogram(int64_t nrows, const int32_t* row_ptrs, int64_t nbins, int64_t* hist,
                                wk_stream_t stream) {
    clear_error();
    WK_REQUIRE(nbins >= 1, WK_ERR_INVALID, "nbins must be >= 1");
    cudaStream_t st = as_stream(stream);
    WK_CUDA(cudaMemsetAsync(hist, 0, sizeof(int64_t) * size_t(nbins), st));
    if (nrows == 0) return 0;
    int64_t blocks = ceil_div(nrows, 512);
    if (blocks > int64_t(sm_count()) * 4) blocks = int64_t(sm_count()) * 4;
    len_hist_kernel<<<(unsigned)blocks, 512, 0, st>>>(nrows, nbins, row_ptrs,
                                                      reinterpret_cast<unsigned long long*>(hist));
    WK_LAUNCH_CHECK();
    return 0;
}

int wk_sellp_zero_padding(int64_t nrows, int64_t slice_size, const int64_t* slice_sets, const int32_t* row_lengths,
                          int32_t* col_idx, double* values, wk_stream_t stream) {
    clear_error();
    const int64_t nslices = ceil_div(nrows, slice_size);
    if (nslices == 0) return 0;
    int64_t blocks = ceil_div(nslices * slice_size, 256);
    if (blocks > int64_t(sm_count()) * 16) blocks = int64_t(sm_count()) * 16;
    sellp_zero_padding_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(nrows, slice_size, nslices, slice_sets,
                                                                               row_lengths, col_idx, values);
    WK_LAUNCH_CHECK();
    return 0;
}

int wk_ell_zero_padding(int64_t nrows, int64_t width, int64_t stride, const int32_t* row_lengths, int32_t* col_idx,
                        double* values, wk_stream_t stream) {
    clear_error();
    if (stride == 0 || width == 0) return 0;
    int64_t blocks = ceil_div(stride, 256);
    if (blocks > int64_t(sm_count()) * 16) blocks = int64_t(sm_count()) * 16;
    ell_zero_padding_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(nrows, width, stride, row_lengths,
                                                                             col_idx, values);
    WK_LAUNCH_CHECK();
    return 0;
}

int wk_csr_to_sellp_sets(int64_t nrows, int64_t slice_size, const int32_t* row_ptrs, int64_t* slice_sets,
                         int32_t* row_lengths, void* scan_ws, wk_stream_t stream) {
    clear_error();
    WK_REQUIRE(slice_size > 0 && (slice_size & (slice_size - 1)) == 0, WK_ERR_SLICE,
               "slice_size must be a positive power of two, got %lld", (long long)slice_size);
    cudaStream_t st = as_stream(stream);
    const int64_t nslices = ceil_div(nrows, slice_size);
    if (nrows) {
        int l2 = 0;
        while ((int64_t(1) << l2) < slice_size) ++l2;
        if (slice_size > 256) WK_CUDA(cudaMemsetAsync(slice_sets, 0, sizeof(int64_t) * (nslices + 1), st));
        slice_widths_kernel<<<(unsigned)ceil_div(nrows, 256), 256, 0, st>>>(nrows, l2, row_ptrs, row_lengths,
                                                                          slice_sets);
        WK_LAUNCH_CHECK();
    }
    // widths sit at slice_sets[s + 1]; the scan reads each before any block overwrites it
    const int64_t* wsrc = slice_sets;
    auto width = [=] __device__(int64_t s) { return wsrc[s + 1]; };
    return exclusive_scan(nslices, width, slice_sets, scan_ws, st);
}

int wk_csr_to_sellp_fill(int64_t nrows, int64_t slice_size, const int32_t* row_ptrs, const int32_t* col_idx,
                         const double* values, const int64_t* slice_sets, int32_t* s_col, double* s_val,
                         wk_stream_t stream) {
    clear_error();
    WK_REQUIRE(slice_size > 0 && (slice_size & (slice_size - 1)) == 0, WK_ERR_SLICE,
               "slice_size must be a positive power of two, got %lld", (long long)slice_size);
    const int64_t nslices = ceil_div(nrows, slice_size);
    if (nslices == 0) return 0;
    int l2 = 0;
    while ((int64_t(1) << l2) < slice_size) ++l2;
    if (slice_size >= 4 && slice_size <= 256 && al16(col_idx) && al16(values))
        return launch_fill_tma<1, false>(nrows, l2, nslices, row_ptrs, col_idx, values, slice_sets, 0, 0, s_col,
                                               s_val, nullptr, as_stream(stream));
    sellp_fill_kernel<<<(unsigned)nslices, kConvThreads, 0, as_stream(stream)>>>(nrows, l2, row_ptrs, col_idx, values,
                                                                               slice_sets, s_col, s_val);
    WK_LAUNCH_CHECK();
    return 0;
}

int wk_csr_to_ell_fill(int64_t nrows, int64_t width, int64_t stride, const int32_t* row_ptrs,
                       const int32_t* col_idx, const double* values, int32_t* e_col, double* e_val,
                       int32_t* e_row_lengths, wk_stream_t stream) {
    clear_error();
    WK_REQUIRE(stride >= nrows, WK_ERR_INVALID, "ELL stride %lld < nrows %lld", (long long)stride,
               (long long)nrows);
    if (stride == 0) return 0;
    if (al16(col_idx) && al16(values)) {
        int l2 = 8;  // tile rows: 256 down to 32 so that a tile's entries fit a stage
        while (l2 > 5 && (int64_t(1) << l2) * width > kFillCap) --l2;
        return launch_fill_tma<2, true>(nrows, l2, ceil_div(stride, int64_t(1) << l2), row_ptrs, col_idx, values,
                                        nullptr, width, stride, e_col, e_val, e_row_lengths, as_stream(stream));
    }
    int64_t rpb = kConvThreads;
    while (rpb > 32 && rpb * width > kStageCap) rpb >>= 1;
    ell_fill_kernel<<<(unsigned)ceil_div(stride, rpb), kConvThreads, 0, as_stream(stream)>>>(
        nrows, width, stride, rpb, row_ptrs, col_idx, values, e_col, e_val, e_row_lengths);
    WK_LAUNCH_CHECK();
    return 0;
}

int wk_hybrid_coo_offsets(int64_t nrows, int64_t width, const int32_t* row_ptrs, int64_t* offsets, void* scan_ws,
                          wk_stream_t stream) {
    clear_error();
    auto rem = [=] __device__(int64_t r) {
        const int64_t len = row_ptrs[r + 1] - row_ptrs[r];
        return len > width ? len - width : int64_t(0);
    };
    return exclusive_scan(nrows, rem, offsets, scan_ws, as_stream(stream));
}

int64_t wk_hybrid_coo_fill_workspace(int64_t rem) {
    // list length <= rem / kHybSeg + (rows with > kHybLong overflow) <= rem / kHybSeg + rem / kHybLong
    return 16 + 8 * (rem / kHybSeg + rem / kHybLong + 1);
}

int wk_hybrid_coo_fill(int64_t nrows, int64_t width, const int32_t* row_ptrs, const int32_t* col_idx,
                       const double* values, const int64_t* offsets, int32_t* c_row, int32_t* c_col,
                       double* c_val, void* work, int64_t work_bytes, wk_stream_t stream) {
    clear_error();
    if (nrows == 0) return 0;
    WK_REQUIRE(work != nullptr && (reinterpret_cast<uintptr_t>(work) & 15) == 0, WK_ERR_INVALID,
               "hybrid fill workspace must be 16-byte aligned");
    cudaStream_t st = as_stream(stream);
    auto* nseg = reinterpret_cast<unsigned long long*>(work);
    auto* segs = reinterpret_cast<int2*>(reinterpret_cast<char*>(work) + 16);
    (void)work_bytes;  // sized by wk_hybrid_coo_fill_workspace(offsets[nrows])
    WK_CUDA(cudaMemsetAsync(nseg, 0, 8, st));
    int64_t blocks = ceil_div(nrows, 256);  // 8 warps x 32 rows
    const int64_t cap = int64_t(sm_count()) * 8;
    if (blocks > cap) blocks = cap;
    hybrid_coo_fill_kernel<<<unsigned(blocks), 256, 0, st>>>(nrows, width, row_ptrs, col_idx, values, offsets,
                                                            c_row, c_col, c_val, nseg, segs);
    WK_LAUNCH_CHECK();
    hybrid_coo_long_kernel<<<unsigned(cap), 256, 0, st>>>(width, row_ptrs, col_idx, values, offsets, c_row, c_col,
                                                         c_val, nseg, segs);
    WK_LAUNCH_CHECK();
    return 0;
}

int wk_coo_to_csr_ptrs(int64_t nrows, int64_t nnz, const int32_t* row_idx, int32_t* row_ptrs, wk_stream_t stream) {
    clear_error();
    const int vec = (reinterpret_cast<uintptr_t>(row_idx) & 15) == 0;
    coo_ptrs_kernel<<<(unsigned)ceil_div(ceil_div(nnz + 1, kPtrItems), 256), 256, 0, as_stream(stream)>>>(
        nrows, nnz, row_idx, row_ptrs, vec);
    WK_LAUNCH_CHECK();
    return 0;
}

int wk_csr_to_coo_rows(int64_t nrows, const int32_t* row_ptrs, int32_t* row_idx, wk_stream_t stream) {
    clear_error();
    if (nrows == 0) return 0;
    csr_rows_kernel<<<warp_grid(nrows), 256, 0, as_stream(stream)>>>(nrows, row_ptrs, row_idx);
    WK_LAUNCH_CHECK();
    return 0;
}

}  // extern "C"
