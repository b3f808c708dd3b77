// Warp-range segmented-sum SpMV for COO and for load-balanced CSR
// (kernels.py:209-257 semantics: entries in row-major order, per-row segment
// sums by a warp segmented scan, atomics only at the run heads shared between
// work units; CSR: deterministic carries instead of atomics).
#pragma once

#include <climits>

#include "common.cuh"
#include "reduce.cuh"

namespace wk {

// ---------------------------------------------------------------------------
// seg8: the same warp-range semantics with 8 consecutive entries per lane
// (windows of 256 entries). Each lane folds its entries sequentially
// (separately rounded, column order: rows inside one lane's 8 entries are the
// reference fold bit for bit) and ONE warp segmented scan per window joins the
// lanes — about an eighth of the shuffle work of seg_warp_kernel, whose
// per-32-entry scans made it issue-bound. Warp ranges are 2048 entries (8
// windows); atomics only for a range's first and last row.
//
// CSR row ids come from a "head plan" built once per matrix: per 256-entry
// window a 256-bit mask of the positions where a non-empty row starts, the
// number of such heads before each window (hoff, exclusive scan) and the row
// id of every head in order (hrow). It replaces a per-window walk of row_ptrs
// (a serial chain of dependent loads) by independent loads of about the size
// of row_ptrs itself (32 B per window + 4 B per non-empty row).
//
// Each lane loads its 8 entries with 16/32-byte vector loads (scalar loads for
// unaligned arrays and the matrix tail). A TMA-staged persistent variant was
// measured 2x slower (the kernel is bound by the random x gathers, not by the
// matrix stream) and removed.
//
// The kernel is bound by the L1TEX data pipe, not by DRAM: every random x
// gather is one wavefront (R-MAT rows share no x lines between lanes), and a
// bare stream + gather fold of the same matrix (tools/gather_probe.cu) takes
// 1.19 ms, 1.03 ms with x shrunk to 16 MB (all L2 hits) — the seg8 kernel runs
// at 0.95-1.0 of that fold. A shared-memory cache of the 8192 hottest columns'
// x (20.8% of R-MAT's entries) did not pay in the real kernel (the L1 already
// serves those gathers: 28% L1 sector hit rate; profiles/r02) and was removed.
// ---------------------------------------------------------------------------
constexpr int kS8Win = 256;                  // entries per window (8 per lane)
constexpr int kS8PerWarp = 8 * kS8Win;       // entries per warp range
constexpr int kS8Warps = 8;                  // warps per block (direct kernel)

inline int64_t seg8_warps(int64_t nnz) { return ceil_div(nnz, kS8PerWarp); }
inline int64_t seg8_windows(int64_t nnz) { return ceil_div(nnz, kS8Win); }

struct HeadPlan {
    const int* hoff;
    const unsigned* mask;
    const int* hrow;
    int* crow;       // per warp range: the row continuing past the range (-1: none) ...
    double* cval;    // ... and the range's part of it (added in range order by the fix-up)
    const int* rrow; // row of each warp range's first entry (ranges + 1 entries; last = -1)
};

struct HeadPlanMut {
    int* hoff;
    unsigned* mask;
    int* hrow;
    void* scan_ws;
    int* crow;
    double* cval;
    int* rrow;
};

inline int64_t head_plan_bytes(int64_t nrows, int64_t nnz) {
    const int64_t w = seg8_windows(nnz), g = seg8_warps(nnz);
    return ceil_div((w + 1) * 4, 256) * 256 + w * 32 + ceil_div(nrows * 4, 256) * 256 + ceil_div(scan_ws_bytes(w), 256) * 256 +
           ceil_div(g * 4, 256) * 256 + ceil_div(g * 8, 256) * 256 + (g + 1) * 4 + 256;
}

inline HeadPlanMut head_plan_views(void* plan, int64_t nrows, int64_t nnz) {
    const int64_t w = seg8_windows(nnz);
    char* p = reinterpret_cast<char*>(plan);
    HeadPlanMut h;
    h.hoff = reinterpret_cast<int*>(p);
    p += ceil_div((w + 1) * 4, 256) * 256;
    h.mask = reinterpret_cast<unsigned*>(p);
    p += w * 32;
    h.hrow = reinterpret_cast<int*>(p);
    p += ceil_div(nrows * 4, 256) * 256;
    h.scan_ws = p;
    p += ceil_div(scan_ws_bytes(w), 256) * 256;
    h.crow = reinterpret_cast<int*>(p);
    p += ceil_div(seg8_warps(nnz) * 4, 256) * 256;
    h.cval = reinterpret_cast<double*>(p);
    p += ceil_div(seg8_warps(nnz) * 8, 256) * 256;
    h.rrow = reinterpret_cast<int*>(p);
    return h;
}

__global__ void head_mask_kernel(int64_t nrows, const int* __restrict__ ptrs, unsigned* __restrict__ mask) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= nrows) return;
    const int p = ptrs[r];
    if (ptrs[r + 1] > p) atomicOr(mask + (int64_t(p) >> 5), 1u << (p & 31));
}

__device__ __forceinline__ int window_heads(const unsigned* __restrict__ mask, int64_t w) {
    int c = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) c += __popc(mask[w * 8 + k]);
    return c;
}

__global__ void head_rows_kernel(int64_t nrows, const int* __restrict__ ptrs, const unsigned* __restrict__ mask,
                                 const int* __restrict__ hoff, int* __restrict__ hrow) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= nrows) return;
    const int p = ptrs[r];
    if (ptrs[r + 1] <= p) return;
    const int64_t w = int64_t(p) >> 8;
    const int word = (p & 255) >> 5;
    int k = hoff[w];
    for (int q = 0; q < word; ++q) k += __popc(mask[w * 8 + q]);
    k += __popc(mask[w * 8 + word] & ((1u << (p & 31)) - 1u));
    hrow[k] = int(r);
}

__device__ __forceinline__ int head_row_of(const HeadPlan& hp, int64_t e);

// row of the first entry of every warp range (range g starts at g * kS8PerWarp)
__global__ void range_rows_kernel(int64_t nranges, int64_t nnz, HeadPlan hp, int* __restrict__ rrow) {
    const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g > nranges) return;
    const int64_t e = g * kS8PerWarp;
    rrow[g] = e < nnz ? head_row_of(hp, e) : -1;
}

inline int build_head_plan(int64_t nrows, int64_t nnz, const int* ptrs, void* plan, cudaStream_t st) {
    const int64_t nw = seg8_windows(nnz);
    const HeadPlanMut h = head_plan_views(plan, nrows, nnz);
    if (nw > 0) WK_CUDA(cudaMemsetAsync(h.mask, 0, size_t(nw) * 32, st));
    if (nrows > 0) {
        head_mask_kernel<<<(unsigned)ceil_div(nrows, 256), 256, 0, st>>>(nrows, ptrs, h.mask);
        WK_LAUNCH_CHECK();
    }
    const unsigned* mask = h.mask;
    WK_TRY(exclusive_scan(nw, [=] __device__(int64_t w) { return window_heads(mask, w); }, h.hoff, h.scan_ws, st));
    if (nrows > 0) {
        head_rows_kernel<<<(unsigned)ceil_div(nrows, 256), 256, 0, st>>>(nrows, ptrs, h.mask, h.hoff, h.hrow);
        WK_LAUNCH_CHECK();
    }
    const int64_t g = seg8_warps(nnz);
    range_rows_kernel<<<(unsigned)ceil_div(g + 1, 256), 256, 0, st>>>(
        g, nnz, HeadPlan{h.hoff, h.mask, h.hrow, h.crow, h.cval, nullptr}, h.rrow);
    WK_LAUNCH_CHECK();
    return 0;
}

// row containing entry e (0 <= e < nnz): the last head at or before e
__device__ __forceinline__ int head_row_of(const HeadPlan& hp, int64_t e) {
    const int64_t w = e >> 8;
    const int pos = int(e & 255);
    int k = __ldg(hp.hoff + w);
    for (int q = 0; q < (pos >> 5); ++q) k += __popc(__ldg(hp.mask + w * 8 + q));
    k += __popc(__ldg(hp.mask + w * 8 + (pos >> 5)) & (0xffffffffu >> (31 - (pos & 31))));
    return __ldg(hp.hrow + k - 1);
}

__device__ __forceinline__ bool head_at(const HeadPlan& hp, int64_t e) {
    return (__ldg(hp.mask + (e >> 5)) >> (e & 31)) & 1u;
}

// warp range [wlo, whi): its boundary rows and the head plan of its 8 windows
// (mask words: lane l holds words l and l + 32 of the range; head offsets: lane < 8)
struct RangeCsr {
    unsigned pm0, pm1;
    int phoff;
};

__device__ __forceinline__ RangeCsr seg8_range_csr(int lane, int64_t wlo, int64_t whi, int64_t nnz, const HeadPlan& hp,
                                                   int& first_row, int& last_row) {
    const int64_t g = wlo / kS8PerWarp;  // ranges start at multiples of kS8PerWarp
    first_row = __ldg(hp.rrow + g);
    last_row = __ldg(hp.rrow + g + 1);  // row of entry whi (-1 past nnz)
    const int64_t w0 = wlo >> 8, nwin = (nnz + kS8Win - 1) / kS8Win;
    RangeCsr rc;
    rc.pm0 = (w0 + (lane >> 3) < nwin) ? __ldg(hp.mask + w0 * 8 + lane) : 0u;
    rc.pm1 = (w0 + 4 + (lane >> 3) < nwin) ? __ldg(hp.mask + w0 * 8 + 32 + lane) : 0u;
    rc.phoff = (lane < 8 && w0 + lane < nwin) ? __ldg(hp.hoff + w0 + lane) : 0;
    return rc;
}

// CSR row ids of window iw of the range: this lane's 8 mask bits, the heads of
// the lanes before (warp exclusive scan), consecutive hrow entries
__device__ __forceinline__ void seg8_csr_rows(int lane, int iw, const RangeCsr& rc, int nv, const HeadPlan& hp,
                                              int (&rw)[8]) {
    const unsigned FULL = 0xffffffffu;
    const unsigned mw = __shfl_sync(FULL, iw < 4 ? rc.pm0 : rc.pm1, (iw * 8 + (lane >> 2)) & 31);
    const unsigned bits = (mw >> ((lane & 3) * 8)) & 0xffu;
    const int cnt = __popc(bits);
    int incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int o = __shfl_up_sync(FULL, incl, d);
        if (lane >= d) incl += o;
    }
    int idx = __shfl_sync(FULL, rc.phoff, iw) + incl - cnt;
    int rcur = (idx > 0 && !(bits & 1u)) ? __ldg(hp.hrow + idx - 1) : 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        if ((bits >> u) & 1u) {
            rcur = __ldg(hp.hrow + idx);
            ++idx;
        }
        rw[u] = u < nv ? rcur : -1;
    }
}

// One window: per-lane sequential fold of the lane's 8 entries (a row ends
// when the next entry's row differs), one warp segmented scan, emission of the
// closed rows, and the carry of the row left open at lane 31 into the next
// window of the same range (closed at the range's last window).
template <class Emit>
__device__ __forceinline__ void seg8_fold(int lane, int nv, bool last_window, const double (&pv)[8],
                                          const int (&rw)[8], int& carry_row, double& carry, Emit emit) {
    const unsigned FULL = 0xffffffffu;
    const int first_r = nv > 0 ? rw[0] : -1;
    const int nxt = __shfl_down_sync(FULL, first_r, 1);
    double acc = 0.0, first_val = 0.0;
    int first_emit = -1;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        if (u < nv) {
            acc = __dadd_rn(acc, pv[u]);
            int rn;
            if (u + 1 < nv) {
                rn = rw[u + 1];
            } else if (lane < 31 && nxt >= 0) {
                rn = nxt;
            } else {
                rn = (lane == 31 && !last_window) ? INT_MIN : -1;  // INT_MIN: open, -1: range end
            }
            if (rn != rw[u] && rn != INT_MIN) {
                if (first_emit < 0) {
                    first_emit = rw[u];
                    first_val = acc;
                } else {
                    emit(rw[u], acc);
                }
                acc = 0.0;
            }
        }
    }
    // warp segmented scan of (closed a row, partial since the last close)
    int f = first_emit >= 0;
    double sv = acc;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double ov = __shfl_up_sync(FULL, sv, d);
        const int of = __shfl_up_sync(FULL, f, d);
        if (lane >= d) {
            if (!f) sv = __dadd_rn(ov, sv);
            f |= of;
        }
    }
    double ex = __shfl_up_sync(FULL, sv, 1);
    int exf = __shfl_up_sync(FULL, f, 1);
    if (lane == 0) {
        ex = 0.0;
        exf = 0;
    }
    // the window's carry-in continues the row of its first entry, or is complete
    const int w_first = __shfl_sync(FULL, first_r, 0);
    double cin = 0.0;
    if (carry_row >= 0) {
        if (carry_row == w_first)
            cin = carry;
        else if (lane == 0)
            emit(carry_row, carry);
    }
    if (!exf) ex = __dadd_rn(cin, ex);
    if (first_emit >= 0) emit(first_emit, __dadd_rn(ex, first_val));
    const double t31 = __shfl_sync(FULL, sv, 31);
    const int f31 = __shfl_sync(FULL, f, 31);
    const int r31 = __shfl_sync(FULL, nv > 0 ? rw[nv - 1] : -1, 31);
    if (!last_window) {
        carry_row = r31;
        carry = f31 ? t31 : __dadd_rn(cin, t31);
    } else {
        carry_row = -1;
    }
}


// One warp range [wlo, whi) of seg8.
template <bool kCsr>
__device__ __forceinline__ void seg8_range(int lane, int64_t g, int64_t nnz, int accumulate, bool vec,
                                           const int* __restrict__ rows, const int* __restrict__ col,
                                           const double* __restrict__ val, const double* __restrict__ x,
                                           double* __restrict__ y, const HeadPlan& hp) {
    const int64_t wlo = g * kS8PerWarp;
    const int64_t whi = (wlo + kS8PerWarp < nnz) ? wlo + kS8PerWarp : nnz;
    int first_row, last_row;
    RangeCsr rc{0u, 0u, 0};
    if (kCsr) {
        rc = seg8_range_csr(lane, wlo, whi, nnz, hp, first_row, last_row);
    } else {
        first_row = __ldg(rows + wlo);
        last_row = __ldg(rows + whi - 1);
    }
    // CSR: deterministic. Every row is stored by the range that closes it; a
    // row continuing past the range end leaves its part in the range's carry
    // slot, added in range order by seg8_fixup_kernel (no atomics). COO
    // (kernels.py:229-253 semantics): atomics for the two rows a range can
    // share with its neighbours.
    const bool carries = kCsr && whi < nnz && !head_at(hp, whi);
    if (kCsr && lane == 0) hp.crow[g] = carries ? last_row : -1;
    auto emit = [&](int r, double v) {
        if (kCsr) {
            if (carries && r == last_row)
                hp.cval[g] = v;
            else
                y[r] = v;
        } else if (r == first_row || r == last_row) {
            atomicAdd(y + r, v);
        } else {
            y[r] = accumulate ? __dadd_rn(y[r], v) : v;
        }
    };
    int carry_row = -1;
    double carry = 0.0;
    for (int64_t E = wlo; E < whi; E += kS8Win) {
        const int64_t kb = E + 8 * lane;
        const int nv = kb >= whi ? 0 : (whi - kb >= 8 ? 8 : int(whi - kb));
        double pv[8];
        int rw[8];
        // CSR row ids first: their hrow loads overlap the matrix stream and
        // the gathers instead of waiting behind the products
        if (kCsr) seg8_csr_rows(lane, int((E - wlo) >> 8), rc, nv, hp, rw);
        {
            int c[8];
            double v[8];
            if (vec && nv == 8) {
                const int4 c0 = ld_stream(reinterpret_cast<const int4*>(col + kb));
                const int4 c1 = ld_stream(reinterpret_cast<const int4*>(col + kb + 4));
                c[0] = c0.x, c[1] = c0.y, c[2] = c0.z, c[3] = c0.w, c[4] = c1.x, c[5] = c1.y, c[6] = c1.z, c[7] = c1.w;
#pragma unroll
                for (int u = 0; u < 8; u += 2) {
                    const double2 t = ld_stream(reinterpret_cast<const double2*>(val + kb + u));
                    v[u] = t.x;
                    v[u + 1] = t.y;
                }
                if (!kCsr) {
                    const int4 r0 = ld_stream(reinterpret_cast<const int4*>(rows + kb));
                    const int4 r1 = ld_stream(reinterpret_cast<const int4*>(rows + kb + 4));
                    rw[0] = r0.x, rw[1] = r0.y, rw[2] = r0.z, rw[3] = r0.w;
                    rw[4] = r1.x, rw[5] = r1.y, rw[6] = r1.z, rw[7] = r1.w;
                }
            } else {
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    c[u] = u < nv ? ld_stream(col + kb + u) : 0;
                    v[u] = u < nv ? ld_stream(val + kb + u) : 0.0;
                    if (!kCsr) rw[u] = u < nv ? ld_stream(rows + kb + u) : -1;
                }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) pv[u] = u < nv ? __dmul_rn(v[u], ld_x(x, c[u])) : 0.0;
        }
        seg8_fold(lane, nv, E + kS8Win >= whi, pv, rw, carry_row, carry, emit);
    }
}

// one warp range per warp
template <bool kCsr>
__global__ void __launch_bounds__(kS8Warps * 32, kCsr ? 3 : 4)
seg8_kernel(int64_t nnz, int accumulate, int vec, const int* __restrict__ rows, const int* __restrict__ col,
            const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y,
            const int* __restrict__ skip, HeadPlan hp) {
    if (skip != nullptr && *skip) return;
    const int lane = threadIdx.x & 31;
    const int64_t warp = int64_t(blockIdx.x) * kS8Warps + (threadIdx.x >> 5);
    if (warp * kS8PerWarp >= nnz) return;
    seg8_range<kCsr>(lane, warp, nnz, accumulate, vec != 0, rows, col, val, x, y, hp);
}

// rows cut by warp-range boundaries (CSR): the first range of each run of
// equal carry rows adds the run's parts, in range order, in front of the part
// stored by the range that closed the row
__global__ void seg8_fixup_kernel(int64_t nranges, const int* __restrict__ crow, const double* __restrict__ cval,
                                  double* __restrict__ y, const int* __restrict__ skip) {
    if (skip != nullptr && *skip) return;
    const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= nranges) return;
    const int r = crow[g];
    if (r < 0 || (g > 0 && crow[g - 1] == r)) return;
    double s = cval[g];
    for (int64_t u = g + 1; u < nranges && crow[u] == r; ++u) s = __dadd_rn(s, cval[u]);
    y[r] = __dadd_rn(s, y[r]);
}


// rows: COO row indices (csr = false) or unused (csr = true, row ids from hp).
inline int launch_seg8(bool csr, int64_t nnz, int accumulate, const int* rows, const int* col, const double* val,
                       const double* x, double* y, const int* skip, cudaStream_t st,
                       HeadPlan hp = HeadPlan{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr}) {
    if (nnz == 0) return 0;
    auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    const int vec = al(col) && al(val) && (csr || al(rows));  // 16/32-byte vector loads
    const unsigned blocks = (unsigned)ceil_div(seg8_warps(nnz), kS8Warps);
    if (csr)
        seg8_kernel<true><<<blocks, kS8Warps * 32, 0, st>>>(nnz, accumulate, vec, rows, col, val, x, y, skip, hp);
    else
        seg8_kernel<false><<<blocks, kS8Warps * 32, 0, st>>>(nnz, accumulate, vec, rows, col, val, x, y, skip, hp);
    WK_LAUNCH_CHECK();
    if (!csr) return 0;
    const int64_t nranges = seg8_warps(nnz);
    if (nranges > 1) {
        seg8_fixup_kernel<<<(unsigned)ceil_div(nranges, 256), 256, 0, st>>>(nranges, hp.crow, hp.cval, y, skip);
        WK_LAUNCH_CHECK();
    }
    return 0;
}

}  // namespace wk
