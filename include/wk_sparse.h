/*
 * wk_sparse.h — C ABI of the B200-native sparse fp64 hot path
 * (libwk_sparse.so, built for sm_100a).
 *
 * Drop-in boundary. The reference (`warpkit`, arXiv 2006.14290 workbench)
 * exposes this path as Python operations behind its registry
 * (`warpkit/dispatch.py:79-125`): `spmv_coo/csr/sellp(m, x, exec)`
 * (`kernels.py:409-418`), `cg_solve(m, b, tol, max_iters, exec)`
 * (`kernels.py:283`), plus the format conversions `coo_to_csr` /
 * `coo_to_sellp` (`sparse.py:212-242`). Its uncompiled CUDA fixtures give the
 * C shapes a native binding would take: `csr_spmv(nrows, row_ptrs, col_idx,
 * vals, x, y)` (tests/golden/src/cuda/matrix/csr_kernels.cu:30-31),
 * `coo_spmv(nnz, ...)` (coo_kernels.cu:34-35), `sellp_spmv(nrows, nslices,
 * slice_sets, col_idx, ...)` (sellp_kernels.cu:28-30), `cg_update(n, alpha,
 * beta, ..., stream)` (solver/cg_kernels.cu:35-36), `exec_settings{stream,
 * device_id}` (base/types.cuh:11-14). Each entry point below cites the
 * interface it replaces.
 *
 * Conventions
 *   - All array arguments are DEVICE pointers (current CUDA device) unless the
 *     name starts with `h_`. The library never frees caller memory.
 *   - Values are IEEE binary64; column/row indices are int32; offsets that
 *     index stored entries (slice_sets) are int64. The reference stores int64
 *     indices (sparse.py:21-25); int32 halves index traffic and covers every
 *     configuration (nnz < 2^31).
 *   - `stream` is a cudaStream_t passed as void*. Every call is asynchronous
 *     on that stream; only functions documented as "synchronises" block.
 *   - Return value: 0 on success, a cudaError_t value for CUDA failures, or a
 *     WK_ERR_* code; `wk_last_error()` gives a message (thread-local).
 */
#ifndef WK_SPARSE_H
#define WK_SPARSE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* wk_stream_t;

enum {
    WK_OK = 0,
    WK_ERR_INVALID = 1001,   /* bad argument (ValueError in the reference)             */
    WK_ERR_DIMENSION = 1002, /* errors.py:47-48 DimensionMismatch                      */
    WK_ERR_BREAKDOWN = 1003, /* errors.py:55-56 BreakdownError (p.Ap <= 0, rho == 0 …) */
    WK_ERR_SLICE = 1004,     /* errors.py:51-52 InvalidSliceSize                        */
    WK_ERR_PARSE = 1005,     /* errors.py:69-70 ParseError (MatrixMarket)               */
    WK_ERR_UNSUPPORTED = 1006 /* errors.py:73-74 UnsupportedFormat (MatrixMarket)       */
};

enum { WK_FMT_CSR = 0, WK_FMT_COO = 1, WK_FMT_ELL = 2, WK_FMT_SELLP = 3, WK_FMT_HYBRID = 4 };

/* CSR SpMV strategies: STREAM = nnz-chunked, TMA-staged, load-balanced for
 * any row-length distribution (bitwise for rows <= 256 entries); SUBWARP = one
 * power-of-two tile of lanes per row (kernels.py:163-196); ROWBLOCK = blocks
 * of 32k consecutive rows, TMA-staged, one lane folds one row (bitwise for
 * rows <= 64 entries; the fastest for regular matrices); MERGE = merge-path
 * tiles of 2048 (row end | nonzero) items per CTA, equal work whatever the
 * row-length skew (rows inside one thread's 8 items fold bitwise, others are
 * joined by deterministic segmented scans); LOAD_BALANCE = Ginkgo's
 * load_balance: 2048 nonzeros per warp, warp segmented scans with row ids
 * from a head plan (wk_csr_load_balance_plan_*), the partial sum of a row
 * continuing past a warp's range kept as that range's carry and added in
 * range order by a fix-up kernel (the fastest for skewed matrices;
 * deterministic, no atomics). */
enum { WK_CSR_STREAM = 0, WK_CSR_SUBWARP = 1, WK_CSR_ROWBLOCK = 2, WK_CSR_MERGE = 3, WK_CSR_LOAD_BALANCE = 4 };

const char* wk_last_error(void);
int wk_version(void);
/* number of SMs of the current device */
int wk_device_sm_count(void);

/* ---- SpMV: y = A x ------------------------------------------------------ */

/* replaces spmv_sellp (kernels.py:417-418 -> 116-157); sellp_spmv fixture
 * (sellp_kernels.cu:28-30). Bitwise equal to dense_spmv_reference.
 * row_lengths is only read when x[0] is not finite. */
int wk_spmv_sellp_f64(int64_t nrows, int64_t ncols, int64_t slice_size, const int64_t* slice_sets,
                      const int32_t* col_idx, const double* values, const int32_t* row_lengths,
                      const double* x, double* y, wk_stream_t stream);

/* ELL = SELL-P with one slice of stride `stride` >= nrows (no reference). */
int wk_spmv_ell_f64(int64_t nrows, int64_t ncols, int64_t width, int64_t stride, const int32_t* col_idx,
                    const double* values, const int32_t* row_lengths, const double* x, double* y,
                    wk_stream_t stream);

/* replaces spmv_csr (kernels.py:413-414 -> 163-203); csr_spmv fixture
 * (csr_kernels.cu:30-31). `plan` is required for WK_CSR_STREAM
 * (wk_csr_plan_bytes / wk_csr_plan_build) and for WK_CSR_MERGE
 * (wk_csr_merge_plan_bytes / wk_csr_merge_plan_build; also holds the
 * per-tile carries, so one SpMV at a time per plan) and for
 * WK_CSR_LOAD_BALANCE (wk_csr_load_balance_plan_*); subwarp_size <= 0 picks
 * the largest power of two <= nnz/nrows, clamped to [1, 32]. */
int wk_spmv_csr_f64(int64_t nrows, int64_t ncols, int64_t nnz, const int32_t* row_ptrs, const int32_t* col_idx,
                    const double* values, const double* x, double* y, int32_t strategy, int32_t subwarp_size,
                    void* plan, wk_stream_t stream);
int64_t wk_csr_plan_chunks(int64_t nnz);
int64_t wk_csr_plan_bytes(int64_t nnz);
int wk_csr_plan_build(int64_t nrows, int64_t nnz, const int32_t* row_ptrs, void* plan, wk_stream_t stream);
int64_t wk_csr_merge_plan_bytes(int64_t nrows, int64_t nnz);
int wk_csr_merge_plan_build(int64_t nrows, int64_t nnz, const int32_t* row_ptrs, void* plan, wk_stream_t stream);
int64_t wk_csr_load_balance_plan_bytes(int64_t nrows, int64_t nnz);
int wk_csr_load_balance_plan_build(int64_t nrows, int64_t nnz, const int32_t* row_ptrs, void* plan,
                                   wk_stream_t stream);


/* replaces spmv_coo (kernels.py:409-410 -> 209-264); coo_spmv fixture
 * (coo_kernels.cu:34-35). Entries sorted row-major. accumulate = 0 zero-fills y. */
int wk_spmv_coo_f64(int64_t nrows, int64_t ncols, int64_t nnz, const int32_t* row_idx, const int32_t* col_idx,
                    const double* values, const double* x, double* y, int32_t accumulate, wk_stream_t stream);

/* Hybrid = ELL(width) + sorted COO remainder (no reference; Ginkgo hybrid). */
int wk_spmv_hybrid_f64(int64_t nrows, int64_t ncols, int64_t ell_width, int64_t ell_stride,
                       const int32_t* ell_col, const double* ell_val, const int32_t* ell_row_lengths,
                       int64_t coo_nnz, const int32_t* coo_row, const int32_t* coo_col, const double* coo_val,
                       const double* x, double* y, wk_stream_t stream);

/* Format-generic operand used by wk_spmv and the solvers. Fields not used by
 * `format` are ignored. HYBRID uses the ELL fields plus coo_*. */
typedef struct wk_matrix {
    int32_t format;
    int32_t csr_strategy;   /* CSR: WK_CSR_* */
    int32_t subwarp_size;   /* CSR subwarp: tile size (<= 0: auto) */
    int32_t reserved;
    int64_t nrows, ncols, nnz;
    const int32_t* row_ptrs;  /* CSR */
    const int32_t* row_idx;   /* COO */
    const int32_t* col_idx;   /* CSR, COO, ELL, SELLP, HYBRID(ell part) */
    const double* values;
    int64_t slice_size;       /* SELLP */
    const int64_t* slice_sets;
    int64_t width, stride;    /* ELL, HYBRID */
    const int32_t* row_lengths; /* ELL, SELLP, HYBRID */
    int64_t coo_nnz;          /* HYBRID */
    const int32_t* coo_row;
    const int32_t* coo_col;
    const double* coo_val;
    void* plan;               /* CSR stream / merge / load_balance plan */
} wk_matrix;

int wk_spmv(const wk_matrix* A, const double* x, double* y, wk_stream_t stream);
/* same, but the launch is a no-op while *skip != 0 (device flag) */
int wk_spmv_masked(const wk_matrix* A, const double* x, double* y, const int32_t* skip, wk_stream_t stream);

/* ---- BLAS-1 (replaces numpy `@`, `+`, `*` in cg_solve, kernels.py:301-329;
 *      host_dot/cublasDdot fixture cg_kernels.cu:26-33; residual_norm
 *      residual_check.cu:17-32; axpy/scale_add cg_kernels.cu:7-21) ------- */

/* bytes of reduction workspace (partials + ticket); zero it once before first use */
int64_t wk_reduce_workspace_bytes(void);
/* *result (device) = x . y, deterministic two-level reduction */
int wk_dot_f64(int64_t n, const double* x, const double* y, double* result, void* workspace, wk_stream_t stream);
/* *result (device) = ||x||_2 */
int wk_norm2_f64(int64_t n, const double* x, double* result, void* workspace, wk_stream_t stream);
/* y = y + alpha * x (separately rounded, like numpy) */
int wk_axpy_f64(int64_t n, double alpha, const double* x, double* y, wk_stream_t stream);
/* y = x + beta * y  (p = r + beta p) */
int wk_xpby_f64(int64_t n, const double* x, double beta, double* y, wk_stream_t stream);
/* x = alpha * x */
int wk_scal_f64(int64_t n, double alpha, double* x, wk_stream_t stream);
/* batched dots: result[i] = V_i . w for i < k, V row-major k x ld (CGS) */
int wk_multidot_f64(int64_t n, int64_t k, const double* V, int64_t ld, const double* w, double* result,
                    void* workspace, wk_stream_t stream);
/* dst[i] = src[idx[i]] (halo pack) */
int wk_gather_f64(int64_t n, const int32_t* idx, const double* src, double* dst, wk_stream_t stream);

/* ---- conversions (replace coo_to_csr / coo_to_sellp, sparse.py:212-242;
 *      CSR->ELL / Hybrid have no reference). Bit-exact copies. ----------- */

/* row_lengths[r] = row_ptrs[r+1]-row_ptrs[r] */
int wk_csr_row_lengths(int64_t nrows, const int32_t* row_ptrs, int32_t* row_lengths, wk_stream_t stream);
/* *result (device, int64) = max row length */
int wk_csr_max_row_length(int64_t nrows, const int32_t* row_ptrs, int64_t* result, wk_stream_t stream);
/* hist[min(len, nbins-1)] += 1 ; hist zeroed by the call */
int wk_csr_row_length_histogram(int64_t nrows, const int32_t* row_ptrs, int64_t nbins, int64_t* hist,
                                wk_stream_t stream);
/* SELL-P pass 1: slice_sets[0..nslices] (cumulative widths, sparse.py:225-229) and
 * int32 row_lengths. scan_ws: wk_scan_workspace_bytes(nslices) bytes. */
int wk_csr_to_sellp_sets(int64_t nrows, int64_t slice_size, const int32_t* row_ptrs, int64_t* slice_sets,
                         int32_t* row_lengths, void* scan_ws, wk_stream_t stream);
/* SELL-P pass 2: scatter (sparse.py:230-241) incl. zero padding. */
int wk_csr_to_sellp_fill(int64_t nrows, int64_t slice_size, const int32_t* row_ptrs, const int32_t* col_idx,
                         const double* values, const int64_t* slice_sets, int32_t* s_col, double* s_val,
                         wk_stream_t stream);
/* ELL(width, stride) from CSR: each row's first min(len, width) entries,
 * padding (0, 0.0); e_row_lengths = min(len, width). Also the ELL part of Hybrid. */
int wk_csr_to_ell_fill(int64_t nrows, int64_t width, int64_t stride, const int32_t* row_ptrs,
                       const int32_t* col_idx, const double* values, int32_t* e_col, double* e_val,
                       int32_t* e_row_lengths, wk_stream_t stream);
/* Stable LSD radix sort of (key, value) pairs on the low key_bits bits of the
 * keys (8 bits per pass; from_entries' row-major lexsort, sparse.py:63-80).
 * Sorts in place; keys_alt / values_alt are n-element scratch buffers; work:
 * wk_sort_pairs_workspace(n) bytes. */
int64_t wk_sort_pairs_workspace(int64_t n);
int wk_sort_pairs_u64_f64(int64_t n, int32_t key_bits, uint64_t* keys, double* values, uint64_t* keys_alt,
                          double* values_alt, void* work, int64_t work_bytes, wk_stream_t stream);
/* Hybrid COO part, pass 1: offsets[0..nrows] = exclusive scan of max(len-width, 0) */
int wk_hybrid_coo_offsets(int64_t nrows, int64_t width, const int32_t* row_ptrs, int64_t* offsets, void* scan_ws,
                          wk_stream_t stream);
/* Hybrid COO part, pass 2: short rows in 32-row flattened runs, rows with
 * more than 256 overflow entries as 4096-entry segments spread over the grid.
 * work: 16-byte aligned device scratch of wk_hybrid_coo_fill_workspace(rem)
 * bytes, rem = offsets[nrows]. */
int64_t wk_hybrid_coo_fill_workspace(int64_t rem);
int wk_hybrid_coo_fill(int64_t nrows, int64_t width, const int32_t* row_ptrs, const int32_t* col_idx,
                       const double* values, const int64_t* offsets, int32_t* c_row, int32_t* c_col,
                       double* c_val, void* work, int64_t work_bytes, wk_stream_t stream);
/* Host-uploaded SELL-P / ELL: rewrite every slot past row_lengths[r] (and
 * the rows past nrows of the last slice / of the stride) as the reference
 * padding (col 0, val 0.0; sparse.py:230-232), in place. */
int wk_sellp_zero_padding(int64_t nrows, int64_t slice_size, const int64_t* slice_sets, const int32_t* row_lengths,
                          int32_t* col_idx, double* values, wk_stream_t stream);
int wk_ell_zero_padding(int64_t nrows, int64_t width, int64_t stride, const int32_t* row_lengths, int32_t* col_idx,
                        double* values, wk_stream_t stream);
/* sorted COO -> CSR row_ptrs (sparse.py:212-216) */
int wk_coo_to_csr_ptrs(int64_t nrows, int64_t nnz, const int32_t* row_idx, int32_t* row_ptrs, wk_stream_t stream);
/* CSR -> COO row indices */
int wk_csr_to_coo_rows(int64_t nrows, const int32_t* row_ptrs, int32_t* row_idx, wk_stream_t stream);

/* ---- scans (device-wide, decoupled three-pass) -------------------------- */
int64_t wk_scan_workspace_bytes(int64_t n);
/* out[0] = 0, out[i+1] = out[i] + in[i]  (n+1 outputs) */
int wk_exclusive_scan_i64(int64_t n, const int64_t* in, int64_t* out, void* ws, wk_stream_t stream);

/* ---- synthetic matrices (device generators) ----------------------------- */

/* Constant-coefficient stencil on an nx*ny*nz grid (row r = (k*ny+j)*nx+i),
 * points given on the host; columns ascend. Call with col_idx == NULL to get
 * row_ptrs (n+1, int32) only; then again with storage for row_ptrs[n]
 * entries. Restates corpus.py:33-50 for 3-D. scan_ws: wk_scan_workspace_bytes(n). */
int wk_gen_stencil_csr(int64_t nx, int64_t ny, int64_t nz, int32_t npoints, const int32_t* h_dx,
                       const int32_t* h_dy, const int32_t* h_dz, const double* h_values, int32_t* row_ptrs,
                       int32_t* col_idx, double* values, void* scan_ws, wk_stream_t stream);
/* R-MAT edges [edge_lo, edge_lo+count): key = row * 2^scale + col, value U[0,1)
 * (oracle/corpus_ref.py rmat_edges restates the same hash) */
int wk_gen_rmat_edges(int32_t scale, int32_t edge_factor, double a, double b, double c, uint64_t seed,
                      int64_t edge_lo, int64_t count, int64_t* keys, double* values, wk_stream_t stream);
/* from_entries duplicate fold (sparse.py:73-79) over keys sorted by
 * wk_sort_pairs_u64_f64: pass 1 counts the unique keys per 2048-key tile and
 * scans them (work: wk_coo_dedup_workspace(n) bytes; the unique count lands
 * at ((int64_t*)work)[wk_coo_dedup_tiles(n)]); pass 2 writes row = key / ncols,
 * col = key % ncols and value = 0.0 + v1 + v2 + ... in input order. keys
 * must be 16-byte aligned. */
int64_t wk_coo_dedup_tiles(int64_t n);
int64_t wk_coo_dedup_workspace(int64_t n);
int wk_coo_dedup_count(int64_t n, const int64_t* keys, void* work, wk_stream_t stream);
int wk_coo_dedup_scatter(int64_t n, int64_t ncols, const int64_t* keys, const double* values, const void* work,
                         int32_t* row, int32_t* col, double* out_values, wk_stream_t stream);

/* ---- Krylov solvers (replace cg_solve, kernels.py:283-331; BiCGSTAB and
 *      GMRES(m) have no reference). x, hist are device arrays; hist holds
 *      max_iters + 1 entries; *iterations (host) receives the count.
 *      Synchronises. Returns WK_ERR_BREAKDOWN on breakdown. ------------- */

int64_t wk_cg_workspace_bytes(int64_t n);
int wk_cg_solve(const wk_matrix* A, const double* b, double tol, int64_t max_iters, double* x, double* hist,
                int64_t* iterations, void* workspace, wk_stream_t stream);
int64_t wk_bicgstab_workspace_bytes(int64_t n);
int wk_bicgstab_solve(const wk_matrix* A, const double* b, double tol, int64_t max_iters, double* x,
                      double* hist, int64_t* iterations, void* workspace, wk_stream_t stream);
/* Jacobi-preconditioned CG (z = r / diag, the apply_jacobi fixture,
 * preconditioner.cu:9-17, inside the reference CG loop kernels.py:283-331;
 * no reference PCG: order of oracle/krylov_ref.py pcg_jacobi_solve).
 * diag from wk_extract_diagonal (missing entries -> 0.0). */
int wk_extract_diagonal(const wk_matrix* A, double* diag, wk_stream_t stream);
int64_t wk_pcg_workspace_bytes(int64_t n);
int wk_pcg_jacobi_solve(const wk_matrix* A, const double* diag, const double* b, double tol, int64_t max_iters,
                        double* x, double* hist, int64_t* iterations, void* workspace, wk_stream_t stream);
/* reduce_microbench (kernels.py:341-364; reduce_driver.cu:5-23): one warp,
 * tiles of `size` lanes reduce (rank + 1) `inner_loops` times with the
 * coop-group butterfly (shared_memory = 0) or the shared-memory tree
 * (residual_check.cu:17-32 style, shared_memory = 1); out[32] per-lane
 * results, *cycles = clock64 cycles of the loop (device pointers). */
int wk_reduce_microbench(int32_t size, int32_t inner_loops, int32_t shared_memory, double* out, long long* cycles,
                         wk_stream_t stream);
int64_t wk_gmres_workspace_bytes(int64_t n, int32_t restart);
int wk_gmres_solve(const wk_matrix* A, const double* b, double tol, int64_t max_iters, int32_t restart,
                   double* x, double* hist, int64_t* iterations, void* workspace, wk_stream_t stream);

/* ---- CG building blocks for the row-block distributed solver. The caller
 *      all-reduces the local dot results between steps (NCCL). State layout:
 *      wk_cg_state (device). ------------------------------------------- */
typedef struct wk_cg_state {
    double rho;        /* r.r of the current residual                        */
    double pq;         /* p.Ap (local, then all-reduced by the caller)        */
    double rr;         /* r.r after the update (local, then all-reduced)      */
    double threshold;  /* tol * ||b||                                          */
    double alpha, beta;
    int64_t iteration;
    int64_t max_iters;
    int32_t done;      /* converged / max_iters reached / breakdown          */
    int32_t breakdown;
    int32_t xpend;     /* wk_cg_solve: x += alpha p of the last r update pending */
    int32_t xdefer;    /* wk_cg_solve: x += alpha_prev p_prev deferred to the next x pass */
    double alpha_prev; /* wk_cg_solve: alpha of the deferred x update         */
} wk_cg_state;

/* rho := b.b (local), x = 0, r = p = b */
int wk_cg_init_local(int64_t n, const double* b, double* x, double* r, double* p, wk_cg_state* state,
                     void* workspace, wk_stream_t stream);
/* after all-reduce of rho: threshold, hist[0], done */
int wk_cg_init_finish(wk_cg_state* state, double tol, int64_t max_iters, double* hist, wk_stream_t stream);
/* state->pq = p.q (local) ; skipped when done */
int wk_cg_dot_pq(int64_t n, const double* p, const double* q, wk_cg_state* state, void* workspace,
                 wk_stream_t stream);
/* q = A p (masked by state->done) and state->pq = p.q (local) in one pass
 * (fused into the SELL-P(64) TMA kernel; SpMV + reduction otherwise). p is
 * the extended vector [owned | halo]; the dot covers the owned rows. */
int wk_cg_spmv_dot(const wk_matrix* A, const double* p, double* q, wk_cg_state* state, void* workspace,
                   wk_stream_t stream);
/* after all-reduce of pq: breakdown check, alpha, iteration += 1 */
int wk_cg_step_alpha(wk_cg_state* state, wk_stream_t stream);
/* x += alpha p ; unless replacement (iteration % 50 == 0): r -= alpha q and
 * state->rr = r.r (local) */
int wk_cg_update_xr(int64_t n, const double* p, const double* q, double* x, double* r, wk_cg_state* state,
                    void* workspace, wk_stream_t stream);
/* replacement iteration only: r = b - q (q = A x) ; state->rr = r.r (local) */
int wk_cg_replace_r(int64_t n, const double* b, const double* q, double* r, wk_cg_state* state, void* workspace,
                    wk_stream_t stream);
/* fused variants (one launch each instead of two): the alpha step evaluated
 * from the all-reduced p.Ap inside the x/r update, and the beta step from the
 * all-reduced r.r inside the p update */
/* two vector passes per iteration: x += alpha p is applied by
 * wk_cg_update_p_beta (which reads p anyway), except on residual-replacement
 * iterations, where the x/r update applies it (the replacement needs x) */
int wk_cg_update_xr_alpha(int64_t n, const double* p, const double* q, double* x, double* r, wk_cg_state* state,
                          void* workspace, wk_stream_t stream);
int wk_cg_update_p_beta(int64_t n, const double* r, double* p, double* x, wk_cg_state* state, double* hist,
                        void* workspace, wk_stream_t stream);
/* after all-reduce of rr: hist, beta, rho := rr, done */
int wk_cg_step_beta(wk_cg_state* state, double* hist, wk_stream_t stream);
/* p = r + beta p ; skipped when done */
int wk_cg_update_p(int64_t n, const double* r, double* p, const wk_cg_state* state, wk_stream_t stream);

/* ---- BiCGSTAB building blocks (oracle/krylov_ref.py bicgstab_solve order).
 *      Vector steps reduce into the local slots of wk_bicg_state; the caller
 *      all-reduces the named slot (distributed) and then runs the scalar step.
 *      Every step is a no-op once `done` is set. ----------------------------- */
typedef struct wk_bicg_state {
    double rho, rho_new, alpha, omega, beta, threshold;
    double rv, ss, tt, ts, rr; /* local partials: all-reduce rho_new, rv, ss, {tt,ts}, rr */
    double rho_next;           /* wk_bicgstab_solve: rh.r of the new r, fused into the x/r step */
    int64_t iteration, max_iters;
    int32_t done, breakdown, apply_half, pad;
} wk_bicg_state;

/* x = 0, r = rh = b, p = v = 0 ; rr = b.b (local) */
int wk_bicg_init(int64_t n, const double* b, double* x, double* r, double* rh, double* p, double* v,
                 wk_bicg_state* st, void* workspace, wk_stream_t stream);
/* after all-reduce of rr: hist[0] = ||b||, threshold, rho = alpha = omega = 1 */
int wk_bicg_init_finish(wk_bicg_state* st, double tol, int64_t max_iters, double* hist, wk_stream_t stream);
/* rho_new = rh.r (local) */
int wk_bicg_rho(int64_t n, const double* rh, const double* r, wk_bicg_state* st, void* workspace, wk_stream_t stream);
/* after all-reduce of rho_new: breakdown if 0, beta = (rho_new/rho)(alpha/omega) */
int wk_bicg_step_beta(wk_bicg_state* st, wk_stream_t stream);
/* p = r + beta (p - omega v) */
int wk_bicg_update_p(int64_t n, const double* r, const double* v, double* p, wk_bicg_state* st, wk_stream_t stream);
/* rv = rh.v (local) */
int wk_bicg_rv(int64_t n, const double* rh, const double* v, wk_bicg_state* st, void* workspace, wk_stream_t stream);
/* after all-reduce of rv: breakdown if 0, alpha = rho_new / rv */
int wk_bicg_step_alpha(wk_bicg_state* st, wk_stream_t stream);
/* s = r - alpha v ; ss = s.s (local) */
int wk_bicg_update_s(int64_t n, const double* r, const double* v, double* s, wk_bicg_state* st, void* workspace,
                     wk_stream_t stream);
/* after all-reduce of ss: iteration += 1; half-step convergence test */
int wk_bicg_step_s(wk_bicg_state* st, double* hist, wk_stream_t stream);
/* on half-step convergence: x = x + alpha p (then clears the flag) */
int wk_bicg_half_x(int64_t n, const double* p, double* x, wk_bicg_state* st, void* workspace, wk_stream_t stream);
/* tt = t.t, ts = t.s (local) */
int wk_bicg_tt_ts(int64_t n, const double* t, const double* s, wk_bicg_state* st, void* workspace,
                  wk_stream_t stream);
/* after all-reduce of {tt, ts}: breakdown if tt == 0, omega = ts / tt */
int wk_bicg_step_omega(wk_bicg_state* st, wk_stream_t stream);
/* x = x + alpha p + omega s ; r = s - omega t ; rr = r.r (local) */
int wk_bicg_update_xr(int64_t n, const double* p, const double* s, const double* t, double* x, double* r,
                      wk_bicg_state* st, void* workspace, wk_stream_t stream);
/* after all-reduce of rr: hist, rho = rho_new, convergence */
int wk_bicg_step_r(wk_bicg_state* st, double* hist, wk_stream_t stream);
/* fused steps (what wk_bicgstab_solve runs): v = A p with rv = r-hat.v
 * (mode 1, w = r-hat) or t = A s with tt, ts (mode 2, x = s extended, its
 * own rows read) in one SpMV when A is aligned SELL-P(64), else SpMV + dot;
 * rho_first: rho_next = r-hat.r; take_rho: rho_new = rho_next; update_xr_rho:
 * the x/r update with rr and rho_next = r-hat.r (new r) summed together */
int wk_bicg_spmv_dots(const wk_matrix* A, const double* x, double* y, wk_bicg_state* st, const double* w, int32_t mode,
                      void* workspace, wk_stream_t stream);
int wk_bicg_rho_first(int64_t n, const double* rh, const double* r, wk_bicg_state* st, void* workspace,
                      wk_stream_t stream);
int wk_bicg_take_rho(wk_bicg_state* st, wk_stream_t stream);
int wk_bicg_update_xr_rho(int64_t n, const double* p, const double* sv, const double* t, const double* rh, double* x,
                          double* r, wk_bicg_state* st, void* workspace, wk_stream_t stream);

/* ---- GMRES(m) building blocks (classical Gram-Schmidt; oracle order).
 *      H is (m+1) x m column-major; cs, sn: m; g: m+1; y: m. --------------- */
typedef struct wk_gmres_state {
    double beta, threshold, sq, hn; /* sq: local squared norm, all-reduced by the caller */
    int64_t iteration, max_iters;
    int32_t done, cycle_done, j_done, restart;
} wk_gmres_state;

/* x = 0, r = b ; sq = b.b (local) */
int wk_gmres_init(int64_t n, const double* b, double* x, double* r, wk_gmres_state* st, void* workspace,
                  wk_stream_t stream);
/* after all-reduce of sq */
int wk_gmres_init_finish(wk_gmres_state* st, double tol, int64_t max_iters, int32_t restart, double* hist,
                         wk_stream_t stream);
/* V0 = r / beta ; g = beta e1 ; opens a cycle */
int wk_gmres_cycle_start(int64_t n, const double* r, double* V0, double* g, wk_gmres_state* st, wk_stream_t stream);
/* Hj[i] = V_i . w for i <= j (local) */
int wk_gmres_multidot(int64_t n, int32_t j, const double* V, int64_t ld, const double* w, double* Hj,
                      wk_gmres_state* st, void* workspace, wk_stream_t stream);
/* w = w - sum_i Hj[i] V_i (i order) ; sq = w.w (local) */
int wk_gmres_orth(int64_t n, int32_t j, const double* V, int64_t ld, double* w, const double* Hj, wk_gmres_state* st,
                  void* workspace, wk_stream_t stream);
/* after all-reduce of sq: Givens rotations of column j, residual estimate,
 * cycle termination test */
int wk_gmres_givens(int32_t j, double* H, double* cs, double* sn, double* g, wk_gmres_state* st, double* hist,
                    wk_stream_t stream);
/* V_{j+1} = w / hn while the cycle continues */
int wk_gmres_next_basis(int64_t n, const double* w, double* Vn, wk_gmres_state* st, wk_stream_t stream);
/* y = H^-1 g (back substitution) ; x = x + sum y_i V_i */
int wk_gmres_update_x(int64_t n, const double* V, int64_t ld, const double* H, const double* g, double* y,
                      double* x, wk_gmres_state* st, wk_stream_t stream);
/* r = b - w (w = A x) ; sq = r.r (local) */
/* Deferred normalisation (what wk_gmres_solve runs): basis slot i holds u_i
 * with v_i = sig[i] u_i (sig[0] = 1, so cycle_start is unchanged). The SpMV
 * writes z = A u_j into slot j+1 and wk_gmres_multidot leaves u_i . z in Hj
 * (all-reduce it when distributed); wk_gmres_orth_scaled turns Hj into
 * h_i = sig_i sig_j (u_i . z) and slot j+1 into w = sig_j z - sum h_i sig_i u_i,
 * local ||w||^2 in sq; wk_gmres_givens_scaled also sets sig[j+1] = 1 / ||w||;
 * wk_gmres_update_x_scaled adds sum (y_i sig_i) u_i. No next_basis pass. */
int wk_gmres_orth_scaled(int64_t n, int32_t j, const double* V, int64_t ld, double* w, double* Hj, const double* sig,
                         wk_gmres_state* st, void* workspace, wk_stream_t stream);
int wk_gmres_givens_scaled(int32_t j, double* H, double* cs, double* sn, double* g, double* sig, wk_gmres_state* st,
                           double* hist, wk_stream_t stream);
int wk_gmres_update_x_scaled(int64_t n, const double* V, int64_t ld, const double* H, const double* g, double* y,
                             double* x, const double* sig, wk_gmres_state* st, wk_stream_t stream);
int wk_gmres_residual(int64_t n, const double* b, const double* w, double* r, wk_gmres_state* st, void* workspace,
                      wk_stream_t stream);
/* after all-reduce of sq: beta, true residual replaces the last history entry, convergence */
int wk_gmres_restart(wk_gmres_state* st, double* hist, wk_stream_t stream);

/* ---- MatrixMarket coordinate I/O on the host (replaces read_matrix_market /
 *      write_matrix_market, sparse.py:269-354; multi-threaded parse). ----- */
enum { WK_MM_REAL = 0, WK_MM_INTEGER = 1, WK_MM_PATTERN = 2 };
typedef struct wk_mm_header {
    int64_t nrows, ncols, nnz; /* declared sizes (nnz = entry lines)                  */
    int32_t field;             /* WK_MM_*                                             */
    int32_t symmetric;         /* 1: entries are mirrored (output <= 2 nnz)           */
    int64_t body_offset;       /* byte offset of the first entry line                 */
    int64_t body_line;         /* line number of the size line                        */
} wk_mm_header;
/* banner + size line; WK_ERR_PARSE / WK_ERR_UNSUPPORTED with a message */
int wk_mm_read_header(const char* data, int64_t len, wk_mm_header* header);
/* 0-based (row, col, value) triplets in file order (symmetric: entry, then
 * its mirror); duplicates are left for from_entries to sum. nthreads <= 0:
 * all hardware threads. */
int wk_mm_parse_entries(const char* data, int64_t len, const wk_mm_header* header, int32_t nthreads,
                        int64_t* rows, int64_t* cols, double* vals, int64_t capacity, int64_t* count);
/* 'coordinate real general', %.17g values; out == NULL: *written = bytes needed */
int wk_mm_write(int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* rows, const int64_t* cols,
                const double* vals, char* out, int64_t capacity, int64_t* written);

/* CG steps of the peer-memory distributed path with the two scalar
 * all-reduces fused into the kernels (peer: device copy of a wk_peer_ctx):
 * the producers' reduction epilogues store their local p.Ap / r.r into every
 * rank's arena, the consumers' prologues wait for all P partials and sum them
 * in rank order. Iteration: spmv_dot_peer -> update_xr_alpha_peer
 * [-> replace_r_peer every 50th] -> update_p_beta_peer. With `halo`
 * (device wk_peer_halo, may be NULL) update_p_beta_peer also stores the new
 * p's boundary rows into the neighbours' copies of p and releases their halo
 * flags, and spmv_dot_peer waits for the incoming halo before its gathers: no
 * exchange kernel either. */
typedef struct wk_peer_halo {
    int32_t n;                  /* sends (<= 8)                                     */
    int32_t peer[8];
    int64_t lo[8], hi[8];       /* owned rows [lo, hi) go to peer ...               */
    int64_t dst_off[8];         /* ... at this byte offset of its arena             */
    int32_t nrecv;
    int32_t recv_peer[8];
    int64_t int_lo, int_hi;     /* slices [int_lo, int_hi) of the local SELL-P matrix
                                   gather no halo column: the fused SpMV folds them
                                   before waiting for the halo (empty range: wait first) */
} wk_peer_halo;
int wk_cg_spmv_dot_peer(const wk_matrix* A, const double* p, double* q, wk_cg_state* state, void* workspace,
                        void* peer, const void* halo, wk_stream_t stream);
int wk_cg_update_xr_alpha_peer(int64_t n, const double* p, const double* q, double* x, double* r,
                               wk_cg_state* state, void* workspace, void* peer, wk_stream_t stream);
int wk_cg_replace_r_peer(int64_t n, const double* b, const double* q, double* r, wk_cg_state* state,
                         void* workspace, void* peer, wk_stream_t stream);
int wk_cg_update_p_beta_peer(int64_t n, const double* r, double* p, double* x, wk_cg_state* state, double* hist,
                             void* workspace, void* peer, const void* halo, wk_stream_t stream);

/* ---- peer-memory communication for the row-block distributed solvers
 *      (replaces the NCCL all-reduce / send-recv of distributed.py on GPUs
 *      with peer access; csrc/peer.cu). Arenas are cudaMalloc'd, exported
 *      with CUDA IPC and opened by every other rank. ---------------------- */
#define WK_PEER_MAX 64
typedef struct wk_peer_ctx {
    int32_t rank, world;
    void* arena[WK_PEER_MAX]; /* every rank's arena in this process's address space */
    int64_t* seq;             /* device int64[2]: all-reduce / halo sequence numbers (zeroed) */
    int32_t* error;           /* device int32: 1 / 2 after an all-reduce / halo wait timed out */
} wk_peer_ctx;
int wk_sym_alloc(int64_t bytes, void** ptr, void* ipc_handle /* 64 bytes out */);
int wk_sym_open(const void* ipc_handle, void** ptr);
int wk_sym_close(void* ptr);
int wk_sym_free(void* ptr);
/* bytes of the arena header (flags + all-reduce slots); vectors start after it */
int64_t wk_peer_arena_header_bytes(void);
/* dst[0..count) = sum over ranks of src[0..count) (count <= 32), summed in
 * rank order: bit-identical on every rank. One kernel (stream-ordered). */
int wk_peer_allreduce(const wk_peer_ctx* ctx, const double* src, double* dst, int32_t count, wk_stream_t stream);
/* halo exchange of vector x (in this rank's arena): for each send j,
 * peer_arena[send_peer[j]] + send_dst_offset[j] bytes receives
 * x[send_idx[j][0..send_count[j])]; returns after the halos of every
 * recv_peer arrived in this rank's copy (ticket: device u32, zeroed). */
int wk_peer_exchange(const wk_peer_ctx* ctx, const double* x, int32_t nsend, const int32_t* send_peer,
                     const int32_t* const* send_idx, const int64_t* send_count, const int64_t* send_dst_offset,
                     int32_t nrecv, const int32_t* recv_peer, void* ticket, wk_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* WK_SPARSE_H */
