// Warp-range segmented-sum SpMV for COO and for load-balanced CSR
// (kernels.py:209-257 semantics: entries in row-major order, per-row segment
// sums by a warp segmented scan, atomics only at the run heads shared between
// work units).
//
// Each warp owns kSwPerWarp consecutive entries and walks them in groups of
// kSwU batches of 32 (one entry per lane). The next group's columns, values
// (and, for COO, row ids) are loaded while the current group is folded
// (software pipelining: 2*kSwU independent loads per lane in flight). Per
// batch an inclusive segmented scan keyed by row gives every row's sum at its
// last lane; the running tail of lane 31 carries into the next batch. Rows
// that begin and end inside the warp range are stored directly, the two rows a
// range can share with its neighbours (its first and last) go through
// atomicAdd on a zero-filled y (or on y itself when accumulating, Hybrid).
//
// CSR variant ("balanced"): equal nonzeros per warp whatever the row-length
// skew, reading 12 B per entry instead of COO's 16. Row ids are expanded on
// the fly from row_ptrs: per batch window [e, e+32) the lanes load 32 row
// starts from the next unpassed row (one coalesced load), a ballot marks the
// non-empty rows starting inside the window, and entry q's row is the last
// such row starting at or before q (popc + fns) — no per-entry index array.
// The row containing each warp range's first entry comes from a plan built
// once per matrix (binary search).
#pragma once

#include <climits>

#include "common.cuh"

namespace wk {

constexpr int kSwPerWarp = 1024;  // entries per warp range
constexpr int kSwU = 4;           // batches of 32 entries per group

inline int64_t seg_warps(int64_t nnz) { return ceil_div(nnz, kSwPerWarp); }

// CSR plan: wrow[w] = row containing entry w*kSwPerWarp (w < nwarps), -1 for w = nwarps
inline int64_t csr_balanced_plan_bytes(int64_t nnz) { return ceil_div((seg_warps(nnz) + 1) * 4, 16) * 16; }

__global__ void csr_balanced_plan_kernel(int64_t nrows, int64_t nnz, int64_t nwarps, const int* __restrict__ ptrs,
                                         int* __restrict__ wrow) {
    const int64_t w = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (w > nwarps) return;
    const int64_t e = w * kSwPerWarp;
    if (e >= nnz) {
        wrow[w] = -1;
        return;
    }
    // largest r in [0, nrows) with ptrs[r] <= e
    int64_t lo = 0, hi = nrows;  // invariant: ptrs[lo] <= e, answer in [lo, hi)
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (int64_t(ptrs[mid]) <= e)
            lo = mid;
        else
            hi = mid;
    }
    wrow[w] = int(lo);
}

template <bool kCsr>
__global__ void __launch_bounds__(256)
seg_warp_kernel(int64_t nnz, int64_t nrows, int accumulate, const int* __restrict__ rows,
                const int* __restrict__ wrow, const int* __restrict__ col, const double* __restrict__ val,
                const double* __restrict__ x, double* __restrict__ y, const int* __restrict__ skip) {
    if (skip != nullptr && *skip) return;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t wlo = warp * kSwPerWarp;
    if (wlo >= nnz) return;
    const int64_t whi = (wlo + kSwPerWarp < nnz) ? wlo + kSwPerWarp : nnz;
    // rows this range can share with its neighbours
    int first_row, last_row;
    if (kCsr) {
        first_row = __ldg(wrow + warp);
        last_row = __ldg(wrow + warp + 1);  // row containing entry whi (-1 past the end)
    } else {
        first_row = __ldg(rows + wlo);
        last_row = __ldg(rows + whi - 1);
    }
    // CSR row expansion state: the row of the last expanded entry, and the
    // first row whose start has not been passed
    int cur = first_row;
    int64_t rnext = int64_t(first_row) + 1;

    auto emit = [&](int r, double v) {
        if (r == first_row || r == last_row)
            atomicAdd(y + r, v);
        else
            y[r] = accumulate ? __dadd_rn(y[r], v) : v;
    };

    int gc[kSwU], gr[kSwU];
    double gv[kSwU];
    auto load_group = [&](int64_t b0) {
#pragma unroll
        for (int u = 0; u < kSwU; ++u) {
            const int64_t k = b0 + u * 32 + lane;
            gc[u] = 0;
            gv[u] = 0.0;
            gr[u] = -1;
            if (k < whi) {
                gc[u] = ld_stream(col + k);
                gv[u] = ld_stream(val + k);
                if (!kCsr) gr[u] = ld_stream(rows + k);
            }
        }
    };
    load_group(wlo);
    int carry_row = -1;
    double carry = 0.0;
    for (int64_t b0 = wlo; b0 < whi; b0 += kSwU * 32) {
        int c[kSwU], r[kSwU];
        double v[kSwU];
#pragma unroll
        for (int u = 0; u < kSwU; ++u) {
            c[u] = gc[u];
            v[u] = gv[u];
            r[u] = gr[u];
        }
        if (b0 + kSwU * 32 < whi) load_group(b0 + kSwU * 32);  // next group in flight
        double p[kSwU];
#pragma unroll
        for (int u = 0; u < kSwU; ++u) p[u] = (b0 + u * 32 + lane < whi) ? __dmul_rn(v[u], ld_x(x, c[u])) : 0.0;
        if (kCsr) {
#pragma unroll
            for (int u = 0; u < kSwU; ++u) {
                const int64_t e = b0 + u * 32;
                if (e >= whi) break;
                int rq = cur;
                for (;;) {
                    const int64_t rr = rnext + lane;
                    int s0 = INT_MAX;
                    if (rr < nrows) s0 = __ldg(rows + rr);
                    int s1 = __shfl_down_sync(FULL, s0, 1);
                    if (lane == 31) s1 = (rr < nrows) ? __ldg(rows + rr + 1) : INT_MAX;
                    const bool in = int64_t(s0) < e + 32;
                    const unsigned inwin = __ballot_sync(FULL, in);
                    const bool head = in && s1 > s0;
                    const unsigned heads = __ballot_sync(FULL, head);
                    const unsigned pm = __reduce_or_sync(FULL, head ? (1u << int(int64_t(s0) - e)) : 0u);
                    const int cnt = __popc(pm & (FULL >> (31 - lane)));
                    if (cnt > 0) rq = int(rnext) + int(__fns(heads, 0, cnt));
                    const int m = __popc(inwin);
                    rnext += m;
                    if (m < 32) break;
                }
                r[u] = (e + lane < whi) ? rq : -1;
                cur = __shfl_sync(FULL, rq, 31);
            }
        }
#pragma unroll
        for (int u = 0; u < kSwU; ++u) {
            if (b0 + u * 32 >= whi) break;
            int rr = r[u];
            double s = p[u];
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const double pv = __shfl_up_sync(FULL, s, d);
                const int pr = __shfl_up_sync(FULL, rr, d);
                if (lane >= d && pr == rr) s += pv;
            }
            const int nr = __shfl_down_sync(FULL, rr, 1);
            const bool valid = rr >= 0;
            const bool tail = valid && (lane == 31 || nr != rr);
            const int r0 = __shfl_sync(FULL, rr, 0);
            if (carry_row >= 0) {
                if (carry_row == r0) {
                    if (tail && rr == r0) s += carry;
                } else if (lane == 0) {
                    emit(carry_row, carry);
                }
            }
            const int r31 = __shfl_sync(FULL, rr, 31);
            const double s31 = __shfl_sync(FULL, s, 31);
            if (tail && lane != 31) emit(rr, s);
            if (r31 >= 0) {
                carry_row = r31;
                carry = s31;
            } else {
                carry_row = -1;
            }
        }
    }
    if (carry_row >= 0 && lane == 0) emit(carry_row, carry);
}

inline int launch_seg_warp(bool csr, int64_t nnz, int64_t nrows, int accumulate, const int* rows, const int* wrow,
                           const int* col, const double* val, const double* x, double* y, const int* skip,
                           cudaStream_t st) {
    const int64_t warps = seg_warps(nnz);
    const unsigned blocks = (unsigned)ceil_div(warps * 32, 256);
    if (csr)
        seg_warp_kernel<true><<<blocks, 256, 0, st>>>(nnz, nrows, accumulate, rows, wrow, col, val, x, y, skip);
    else
        seg_warp_kernel<false><<<blocks, 256, 0, st>>>(nnz, nrows, accumulate, rows, wrow, col, val, x, y, skip);
    WK_LAUNCH_CHECK();
    return 0;
}

}  // namespace wk

namespace wk {

// ---------------------------------------------------------------------------
// seg8: the same warp-range semantics with 8 consecutive entries per lane
// (windows of 256 entries). Each lane folds its entries sequentially
// (separately rounded, column order: rows inside one lane's 8 entries are the
// reference fold bit for bit) and ONE warp segmented scan per window joins the
// lanes — about an eighth of the shuffle work of seg_warp_kernel, whose
// per-32-entry scans made it issue-bound. Loads are 16/32-byte vectors per
// lane (each warp instruction covers 512 B / 1 KB contiguous). CSR row ids
// come from the row starts falling inside the window, recorded in a per-warp
// shared table (row of each head position + a 256-bit head mask).
// ---------------------------------------------------------------------------
constexpr int kS8Win = 256;                  // entries per window (8 per lane)
constexpr int kS8PerWarp = 8 * kS8Win;       // entries per warp range
constexpr int kS8Warps = 8;                  // warps per block
#ifndef WK_S8_MIN_BLOCKS
#define WK_S8_MIN_BLOCKS 1
#endif
constexpr int kS8MinBlocks = WK_S8_MIN_BLOCKS;  // resident blocks per SM the register budget targets

inline int64_t seg8_warps(int64_t nnz) { return ceil_div(nnz, kS8PerWarp); }
inline int64_t seg8_plan_bytes(int64_t nnz) { return ceil_div((seg8_warps(nnz) + 1) * 4, 16) * 16; }

__global__ void seg8_plan_kernel(int64_t nrows, int64_t nnz, int64_t nwarps, const int* __restrict__ ptrs,
                                 int* __restrict__ wrow) {
    const int64_t w = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (w > nwarps) return;
    const int64_t e = w * kS8PerWarp;
    if (e >= nnz) {
        wrow[w] = -1;
        return;
    }
    int64_t lo = 0, hi = nrows;
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (int64_t(ptrs[mid]) <= e)
            lo = mid;
        else
            hi = mid;
    }
    wrow[w] = int(lo);
}

template <bool kCsr>
__global__ void __launch_bounds__(kS8Warps * 32, kS8MinBlocks)
seg8_kernel(int64_t nnz, int64_t nrows, int accumulate, const int* __restrict__ rows, const int* __restrict__ wrow,
            const int* __restrict__ col, const double* __restrict__ val, const double* __restrict__ x,
            double* __restrict__ y, const int* __restrict__ skip) {
    if (skip != nullptr && *skip) return;
    const unsigned FULL = 0xffffffffu;
    __shared__ int s_row[kS8Warps][kS8Win];
    __shared__ unsigned s_mask[kS8Warps][kS8Win / 32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t warp = int64_t(blockIdx.x) * kS8Warps + wib;
    const int64_t wlo = warp * kS8PerWarp;
    if (wlo >= nnz) return;
    const int64_t whi = (wlo + kS8PerWarp < nnz) ? wlo + kS8PerWarp : nnz;
    int first_row, last_row;
    if (kCsr) {
        first_row = __ldg(wrow + warp);
        last_row = __ldg(wrow + warp + 1);
    } else {
        first_row = __ldg(rows + wlo);
        last_row = __ldg(rows + whi - 1);
    }
    auto emit = [&](int r, double v) {
        if (r == first_row || r == last_row)
            atomicAdd(y + r, v);
        else
            y[r] = accumulate ? __dadd_rn(y[r], v) : v;
    };
    int64_t rnext = int64_t(first_row) + 1;  // CSR: first row whose start is not passed
    int carry_row = -1;                      // open row entering the window, its partial
    double carry = 0.0;
    int prev_last = first_row;               // row of the last entry of the previous window
    for (int64_t E = wlo; E < whi; E += kS8Win) {
        const int64_t kb = E + 8 * lane;
        const int nv = kb >= whi ? 0 : (whi - kb >= 8 ? 8 : int(whi - kb));
        double pv[8];
        int rw[8];
        {
            int c[8];
            double v[8];
            if (nv == 8) {
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
        if (kCsr) {
            // heads: non-empty rows starting inside [E, E + 256)
            if (lane < kS8Win / 32) s_mask[wib][lane] = 0u;
            __syncwarp();
            // row starts of the next kSuper*32 rows in one batch of independent
            // loads (the expansion is a serial chain per warp: one latency per
            // batch instead of one per 32 rows — windows in sparse regions span
            // hundreds of mostly empty rows)
            constexpr int kSuper = 4;
            for (;;) {
                int s0[kSuper + 1];
#pragma unroll
                for (int k = 0; k < kSuper; ++k) {
                    const int64_t rr = rnext + 32 * k + lane;
                    s0[k] = rr < nrows ? __ldg(rows + rr) : INT_MAX;
                }
                {
                    const int64_t rr = rnext + 32 * kSuper;  // one past the batch, for lane 31's s1
                    s0[kSuper] = rr <= nrows ? __ldg(rows + rr) : INT_MAX;
                }
                int m = 0;
#pragma unroll
                for (int k = 0; k < kSuper; ++k) {
                    const int64_t rr = rnext + 32 * k + lane;
                    int s1 = __shfl_down_sync(FULL, s0[k], 1);
                    const int nxt0 = __shfl_sync(FULL, s0[k + 1], 0);
                    if (lane == 31) s1 = (k + 1 < kSuper) ? nxt0 : s0[kSuper];
                    if (rr == nrows - 1) s1 = __ldg(rows + nrows);  // the last row ends at nnz
                    const bool in = int64_t(s0[k]) < E + kS8Win;
                    if (in && s1 > s0[k]) {
                        const int p = int(int64_t(s0[k]) - E);
                        s_row[wib][p] = int(rr);
                        atomicOr(&s_mask[wib][p >> 5], 1u << (p & 31));
                    }
                    const int mk = __popc(__ballot_sync(FULL, in));
                    m += mk;
                    if (mk < 32) break;
                }
                rnext += m;
                if (m < 32 * kSuper) break;
            }
            __syncwarp();
            const unsigned bits = (s_mask[wib][lane >> 2] >> ((lane & 3) * 8)) & 0xffu;
            // row open at this lane's first entry: the last head of the lanes
            // before (inclusive max-scan of each lane's last head row)
            int lastr = bits ? s_row[wib][8 * lane + 31 - __clz(bits)] : -1;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int o = __shfl_up_sync(FULL, lastr, d);
                if (lane >= d && o > lastr) lastr = o;
            }
            int open = __shfl_up_sync(FULL, lastr, 1);
            if (lane == 0 || open < 0) open = prev_last;
            int rcur = open;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if ((bits >> u) & 1u) rcur = s_row[wib][8 * lane + u];
                rw[u] = u < nv ? rcur : -1;
            }
            __syncwarp();
        }
        // row of the entry before / after this lane's range
        const int first_r = nv > 0 ? rw[0] : -1;
        const int nxt = __shfl_down_sync(FULL, first_r, 1);
        const bool last_window = E + kS8Win >= whi;
        // fold: a row ends after entry u when the next entry's row differs;
        // lane 31's last row stays open (carried) unless this is the last window
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
        // carry-out: lane 31's open partial (rows of the last window all closed)
        const double t31 = __shfl_sync(FULL, sv, 31);
        const int f31 = __shfl_sync(FULL, f, 31);
        const int r31 = __shfl_sync(FULL, nv > 0 ? rw[nv - 1] : -1, 31);
        if (!last_window) {
            carry_row = r31;
            carry = f31 ? t31 : __dadd_rn(cin, t31);
            prev_last = r31;
        } else {
            carry_row = -1;
        }
    }
}

inline int launch_seg8(bool csr, int64_t nnz, int64_t nrows, int accumulate, const int* rows, const int* wrow,
                       const int* col, const double* val, const double* x, double* y, const int* skip,
                       cudaStream_t st) {
    const unsigned blocks = (unsigned)ceil_div(seg8_warps(nnz), kS8Warps);
    if (csr)
        seg8_kernel<true><<<blocks, kS8Warps * 32, 0, st>>>(nnz, nrows, accumulate, rows, wrow, col, val, x, y, skip);
    else
        seg8_kernel<false><<<blocks, kS8Warps * 32, 0, st>>>(nnz, nrows, accumulate, rows, wrow, col, val, x, y, skip);
    WK_LAUNCH_CHECK();
    return 0;
}

}  // namespace wk
