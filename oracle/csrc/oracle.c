/*
 * CPU oracle, C restatement — TEST INFRASTRUCTURE / CPU BASELINE ONLY.
 *
 * Restates the reference's sequential SpMV fold (warpkit/sparse.py:367-417:
 * per row `acc = 0.0; acc += v * x[c]` in stored order) and its CG loop
 * (warpkit/kernels.py:283-331) in C so the CPU baseline can use every host
 * core. Built with -ffp-contract=off: each product and each sum is rounded
 * separately, so every row result is bitwise identical to the reference no
 * matter how rows are split across OpenMP threads. Dot products sum
 * per-thread blocks in thread order (the order depends on the thread count,
 * as the reference's OpenBLAS ddot does, see SURVEY.md §7 "Solver parity",
 * but not on thread timing).
 *
 * Index layout follows the device formats: int32 column indices, int64
 * row pointers / slice sets.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static void set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

int or_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* sparse.py:384-396 */
void or_spmv_csr(int64_t nrows, const int64_t* ptrs, const int32_t* col, const double* val,
                 const double* x, double* y, int nthreads) {
    set_threads(nthreads);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < nrows; ++r) {
        double acc = 0.0;
        for (int64_t k = ptrs[r]; k < ptrs[r + 1]; ++k) acc += val[k] * x[col[k]];
        y[r] = acc;
    }
}

/* sparse.py:397-417: walk row_lengths[r] entries at stride slice_size */
void or_spmv_sellp(int64_t nrows, int64_t ss, const int64_t* sets, const int32_t* col,
                   const double* val, const int64_t* lengths, const double* x, double* y,
                   int nthreads) {
    set_threads(nthreads);
    int64_t nslices = (nrows + ss - 1) / ss;
#pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < nslices; ++s) {
        int64_t hi = (s + 1) * ss < nrows ? (s + 1) * ss : nrows;
        for (int64_t r = s * ss; r < hi; ++r) {
            int64_t k = sets[s] * ss + (r - s * ss);
            double acc = 0.0;
            for (int64_t j = 0; j < lengths[r]; ++j, k += ss) acc += val[k] * x[col[k]];
            y[r] = acc;
        }
    }
}

/* ELL = single slice of stride `stride` */
void or_spmv_ell(int64_t nrows, int64_t stride, const int32_t* col, const double* val,
                 const int64_t* lengths, const double* x, double* y, int nthreads) {
    set_threads(nthreads);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < nrows; ++r) {
        double acc = 0.0;
        int64_t k = r;
        for (int64_t j = 0; j < lengths[r]; ++j, k += stride) acc += val[k] * x[col[k]];
        y[r] = acc;
    }
}

/* sparse.py:374-383: y[row] += v * x[col] in sorted order. Threads take
 * contiguous nnz ranges snapped to row starts, so every row is still folded
 * by one thread in order. */
void or_spmv_coo(int64_t nrows, int64_t nnz, const int32_t* row, const int32_t* col,
                 const double* val, const double* x, double* y, int nthreads) {
    set_threads(nthreads);
    memset(y, 0, sizeof(double) * (size_t)nrows);
#pragma omp parallel
    {
        int nt = 1, t = 0;
#ifdef _OPENMP
        nt = omp_get_num_threads();
        t = omp_get_thread_num();
#endif
        int64_t lo = nnz * t / nt, hi = nnz * (t + 1) / nt;
        while (lo > 0 && lo < nnz && row[lo] == row[lo - 1]) ++lo;
        while (hi > 0 && hi < nnz && row[hi] == row[hi - 1]) ++hi;
        for (int64_t k = lo; k < hi; ++k) y[row[k]] += val[k] * x[col[k]];
    }
}

/* Deterministic for a given thread count: thread t sums the contiguous block
 * [n t / T, n (t + 1) / T) in index order and the T partials are added in
 * thread order (an OpenMP `reduction(+)` combines them in arrival order, so
 * repeated runs of a chaotic solver -- BiCGSTAB on a nonsymmetric operator --
 * could take different iteration counts). */
#define OR_MAX_THREADS 1024
double or_dot(int64_t n, const double* a, const double* b, int nthreads) {
    set_threads(nthreads);
    double part[OR_MAX_THREADS];
    int used = 1;
#pragma omp parallel
    {
        int nt = 1, t = 0;
#ifdef _OPENMP
        nt = omp_get_num_threads();
        t = omp_get_thread_num();
#endif
        if (nt > OR_MAX_THREADS) nt = OR_MAX_THREADS;
        if (t < nt) {
            const int64_t lo = n * t / nt, hi = n * (t + 1) / nt;
            double s = 0.0;
            for (int64_t i = lo; i < hi; ++i) s += a[i] * b[i];
            part[t] = s;
        }
        if (t == 0) used = nt;
    }
    double s = 0.0;
    for (int t = 0; t < used; ++t) s += part[t];
    return s;
}

/*
 * kernels.py:283-331 on a SELL-P matrix. Returns the iteration count, -1 on
 * breakdown (p.Ap <= 0). `hist` must hold max_iters + 1 doubles.
 */
int64_t or_cg_sellp(int64_t n, int64_t ss, const int64_t* sets, const int32_t* col,
                    const double* val, const int64_t* lengths, const double* b, double tol,
                    int64_t max_iters, double* x, double* hist, int nthreads) {
    double* r = (double*)malloc(sizeof(double) * (size_t)n);
    double* p = (double*)malloc(sizeof(double) * (size_t)n);
    double* q = (double*)malloc(sizeof(double) * (size_t)n);
    set_threads(nthreads);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        x[i] = 0.0;
        r[i] = b[i];
        p[i] = b[i];
    }
    double rho = or_dot(n, b, b, nthreads);
    double b_norm = sqrt(rho);
    hist[0] = b_norm;
    int64_t it = 0;
    if (b_norm != 0.0) {
        double thr = tol * b_norm, last = b_norm;
        while (it < max_iters && last > thr) {
            or_spmv_sellp(n, ss, sets, col, val, lengths, p, q, nthreads);
            double pq = or_dot(n, p, q, nthreads);
            if (pq <= 0.0) { it = -1; break; }
            double alpha = rho / pq;
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < n; ++i) x[i] = x[i] + alpha * p[i];
            ++it;
            if (it % 50 == 0) {
                or_spmv_sellp(n, ss, sets, col, val, lengths, x, q, nthreads);
#pragma omp parallel for schedule(static)
                for (int64_t i = 0; i < n; ++i) r[i] = b[i] - q[i];
            } else {
#pragma omp parallel for schedule(static)
                for (int64_t i = 0; i < n; ++i) r[i] = r[i] - alpha * q[i];
            }
            double rho_next = or_dot(n, r, r, nthreads);
            last = sqrt(rho_next);
            hist[it] = last;
            double beta = rho_next / rho;
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < n; ++i) p[i] = r[i] + beta * p[i];
            rho = rho_next;
        }
    }
    free(r);
    free(p);
    free(q);
    return it;
}

/* ---- Krylov restatements beyond the reference (parity unpinned by it) ----
 * oracle/krylov_ref.py fixes the update order the B200 solvers follow; these
 * are the same statements in C + OpenMP so the BASELINE configs' full-size
 * systems (2M-134M rows) are checked against a CPU solve in seconds. They
 * are cross-checked against krylov_ref.py (bitwise SpMV, dots within
 * rounding) and against scipy.sparse.linalg.{bicgstab,gmres}
 * (tests/test_oracle_solvers.py). The operator is CSR (the SELL-P fold of
 * the same matrix is bitwise identical, sparse.py:384-417). */

static void vlin(int64_t n, double* out, const double* a, double alpha, const double* b) {
    /* out = a + alpha * b, separately rounded (numpy `a + alpha * b`) */
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = a[i] + alpha * b[i];
}

/* krylov_ref.bicgstab_solve. Returns iterations, -1 rho == 0, -2 r^.v == 0,
 * -3 t.t == 0. hist must hold max_iters + 1 doubles. */
int64_t or_bicgstab_csr(int64_t n, const int64_t* ptrs, const int32_t* col, const double* val,
                        const double* b, double tol, int64_t max_iters, double* x, double* hist,
                        int nthreads) {
    set_threads(nthreads);
    size_t bytes = sizeof(double) * (size_t)n;
    double *r = malloc(bytes), *rhat = malloc(bytes), *p = malloc(bytes), *v = malloc(bytes);
    double *s = malloc(bytes), *t = malloc(bytes);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        x[i] = 0.0;
        r[i] = b[i];
        rhat[i] = b[i];
        p[i] = 0.0;
        v[i] = 0.0;
    }
    double rho = 1.0, alpha = 1.0, omega = 1.0;
    double b_norm = sqrt(or_dot(n, b, b, nthreads));
    hist[0] = b_norm;
    int64_t it = 0;
    if (b_norm != 0.0) {
        double thr = tol * b_norm, last = b_norm;
        while (it < max_iters && last > thr) {
            double rho_new = or_dot(n, rhat, r, nthreads);
            if (rho_new == 0.0) { it = -1; break; }
            double beta = (rho_new / rho) * (alpha / omega);
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < n; ++i) p[i] = r[i] + beta * (p[i] - omega * v[i]);
            or_spmv_csr(n, ptrs, col, val, p, v, nthreads);
            double rv = or_dot(n, rhat, v, nthreads);
            if (rv == 0.0) { it = -2; break; }
            alpha = rho_new / rv;
            vlin(n, s, r, -alpha, v);
            ++it;
            double s_norm = sqrt(or_dot(n, s, s, nthreads));
            if (s_norm <= thr) {
                vlin(n, x, x, alpha, p);
                hist[it] = s_norm;
                break;
            }
            or_spmv_csr(n, ptrs, col, val, s, t, nthreads);
            double tt = or_dot(n, t, t, nthreads);
            if (tt == 0.0) { it = -3; break; }
            omega = or_dot(n, t, s, nthreads) / tt;
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < n; ++i) {
                x[i] = x[i] + alpha * p[i] + omega * s[i];
                r[i] = s[i] - omega * t[i];
            }
            last = sqrt(or_dot(n, r, r, nthreads));
            hist[it] = last;
            rho = rho_new;
        }
    }
    free(r); free(rhat); free(p); free(v); free(s); free(t);
    return it;
}

/* krylov_ref.givens */
static void or_givens(double a, double b, double* c, double* s) {
    if (b == 0.0) { *c = 1.0; *s = 0.0; return; }
    double h = hypot(a, b);
    *c = a / h;
    *s = b / h;
}

/* krylov_ref.gmres_solve: restarted GMRES(m), classical Gram-Schmidt with
 * batched dots, Givens rotations, true residual at every restart (replacing
 * the cycle's last history entry). Returns iterations, or -4 when the basis
 * cannot be allocated. hist must hold max_iters + 1 doubles. */
int64_t or_gmres_csr(int64_t n, const int64_t* ptrs, const int32_t* col, const double* val,
                     const double* b, double tol, int64_t max_iters, int64_t restart, double* x,
                     double* hist, int nthreads) {
    set_threads(nthreads);
    int64_t m = restart;
    size_t bytes = sizeof(double) * (size_t)n;
    double* V = malloc(bytes * (size_t)(m + 1));
    double *w = malloc(bytes), *r = malloc(bytes);
    double* H = calloc((size_t)((m + 1) * m), sizeof(double)); /* H[i*m + j] */
    double *cs = calloc((size_t)m, sizeof(double)), *sn = calloc((size_t)m, sizeof(double));
    double *g = calloc((size_t)(m + 1), sizeof(double)), *h = calloc((size_t)(m + 1), sizeof(double));
    double* y = calloc((size_t)m, sizeof(double));
    if (!V || !w || !r) {
        free(V); free(w); free(r); free(H); free(cs); free(sn); free(g); free(h); free(y);
        return -4;
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        x[i] = 0.0;
        r[i] = b[i];
    }
    double b_norm = sqrt(or_dot(n, b, b, nthreads));
    hist[0] = b_norm;
    int64_t it = 0;
    double beta = b_norm, thr = tol * b_norm;
    while (b_norm != 0.0 && it < max_iters && beta > thr) {
        memset(H, 0, sizeof(double) * (size_t)((m + 1) * m));
        memset(g, 0, sizeof(double) * (size_t)(m + 1));
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i) V[i] = r[i] / beta;
        g[0] = beta;
        int64_t j_done = 0;
        for (int64_t j = 0; j < m; ++j) {
            const double* vj = V + (size_t)j * (size_t)n;
            or_spmv_csr(n, ptrs, col, val, vj, w, nthreads);
            for (int64_t i = 0; i <= j; ++i) h[i] = or_dot(n, V + (size_t)i * (size_t)n, w, nthreads);
#pragma omp parallel for schedule(static)
            for (int64_t k = 0; k < n; ++k) {
                double acc = w[k];
                for (int64_t i = 0; i <= j; ++i) acc = acc - h[i] * V[(size_t)i * (size_t)n + k];
                w[k] = acc;
            }
            double hn = sqrt(or_dot(n, w, w, nthreads));
            if (hn != 0.0) {
                double* vn = V + (size_t)(j + 1) * (size_t)n;
#pragma omp parallel for schedule(static)
                for (int64_t k = 0; k < n; ++k) vn[k] = w[k] / hn;
            }
            for (int64_t i = 0; i <= j; ++i) H[i * m + j] = h[i];
            H[(j + 1) * m + j] = hn;
            for (int64_t i = 0; i < j; ++i) {
                double a = H[i * m + j], c = H[(i + 1) * m + j];
                H[i * m + j] = cs[i] * a + sn[i] * c;
                H[(i + 1) * m + j] = -sn[i] * a + cs[i] * c;
            }
            or_givens(H[j * m + j], H[(j + 1) * m + j], &cs[j], &sn[j]);
            H[j * m + j] = cs[j] * H[j * m + j] + sn[j] * H[(j + 1) * m + j];
            H[(j + 1) * m + j] = 0.0;
            g[j + 1] = -sn[j] * g[j];
            g[j] = cs[j] * g[j];
            ++it;
            j_done = j + 1;
            hist[it] = fabs(g[j + 1]);
            if (fabs(g[j + 1]) <= thr || it >= max_iters || hn == 0.0) break;
        }
        for (int64_t i = j_done - 1; i >= 0; --i) {
            double acc = g[i];
            for (int64_t k = i + 1; k < j_done; ++k) acc = acc - H[i * m + k] * y[k];
            y[i] = acc / H[i * m + i];
        }
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < n; ++k) {
            double acc = x[k];
            for (int64_t i = 0; i < j_done; ++i) acc = acc + y[i] * V[(size_t)i * (size_t)n + k];
            x[k] = acc;
        }
        or_spmv_csr(n, ptrs, col, val, x, w, nthreads);
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < n; ++k) r[k] = b[k] - w[k];
        beta = sqrt(or_dot(n, r, r, nthreads));
        hist[it] = beta;
    }
    free(V); free(w); free(r); free(H); free(cs); free(sn); free(g); free(h); free(y);
    return it;
}

/* ---- matrix construction for the full-size CPU baseline ----------------------------------
 * corpus_ref.stencil (rows of a constant-coefficient stencil on an
 * nx*ny*nz grid, points already sorted by linear offset so columns ascend)
 * and sparse_ref.csr_to_sellp (sparse.py:219-242) in C, so the reference arm
 * builds BASELINE config 2 (214M entries) in seconds. Checked against the
 * numpy restatements by tests/test_oracle_golden.py. */

/* pass 1: row lengths of rows [row_lo, row_hi) into ptrs[1..], ptrs[0] = 0;
 * returns nnz (ptrs becomes the prefix sum). */
int64_t or_stencil_ptrs(int64_t nx, int64_t ny, int64_t nz, int npts, const int32_t* pts, int64_t row_lo,
                        int64_t row_hi, int64_t* ptrs, int nthreads) {
    set_threads(nthreads);
    int64_t n = row_hi - row_lo;
    ptrs[0] = 0;
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < n; ++q) {
        int64_t r = row_lo + q, i = r % nx, j = (r / nx) % ny, k = r / (nx * ny), c = 0;
        for (int p = 0; p < npts; ++p) {
            int64_t a = i + pts[3 * p], b = j + pts[3 * p + 1], d = k + pts[3 * p + 2];
            c += (a >= 0 && a < nx && b >= 0 && b < ny && d >= 0 && d < nz);
        }
        ptrs[q + 1] = c;
    }
    for (int64_t q = 0; q < n; ++q) ptrs[q + 1] += ptrs[q];
    return ptrs[n];
}

void or_stencil_fill(int64_t nx, int64_t ny, int64_t nz, int npts, const int32_t* pts, const double* vals,
                     int64_t row_lo, int64_t row_hi, const int64_t* ptrs, int32_t* col, double* val,
                     int nthreads) {
    set_threads(nthreads);
    int64_t n = row_hi - row_lo;
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < n; ++q) {
        int64_t r = row_lo + q, i = r % nx, j = (r / nx) % ny, k = r / (nx * ny), e = ptrs[q];
        for (int p = 0; p < npts; ++p) {
            int64_t a = i + pts[3 * p], b = j + pts[3 * p + 1], d = k + pts[3 * p + 2];
            if (a >= 0 && a < nx && b >= 0 && b < ny && d >= 0 && d < nz) {
                col[e] = (int32_t)(r + (int64_t)pts[3 * p + 2] * nx * ny + (int64_t)pts[3 * p + 1] * nx + pts[3 * p]);
                val[e] = vals[p];
                ++e;
            }
        }
    }
}

/* slice_sets (nslices + 1) and row lengths; returns the stored slot count */
int64_t or_sellp_sets(int64_t nrows, int64_t ss, const int64_t* ptrs, int64_t* sets, int64_t* lengths,
                      int nthreads) {
    set_threads(nthreads);
    int64_t nslices = (nrows + ss - 1) / ss;
    sets[0] = 0;
#pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < nslices; ++s) {
        int64_t w = 0, hi = (s + 1) * ss < nrows ? (s + 1) * ss : nrows;
        for (int64_t r = s * ss; r < hi; ++r) {
            lengths[r] = ptrs[r + 1] - ptrs[r];
            if (lengths[r] > w) w = lengths[r];
        }
        sets[s + 1] = w;
    }
    for (int64_t s = 0; s < nslices; ++s) sets[s + 1] += sets[s];
    return sets[nslices] * ss;
}

/* zero-filled storage, entry j of row r at sets[s]*ss + j*ss + (r - s*ss) */
void or_sellp_fill(int64_t nrows, int64_t ss, const int64_t* ptrs, const int32_t* ccol, const double* cval,
                   const int64_t* sets, int32_t* col, double* val, int nthreads) {
    set_threads(nthreads);
    int64_t nslices = (nrows + ss - 1) / ss;
#pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < nslices; ++s) {
        int64_t base = sets[s] * ss, w = sets[s + 1] - sets[s];
        memset(col + base, 0, sizeof(int32_t) * (size_t)(w * ss));
        memset(val + base, 0, sizeof(double) * (size_t)(w * ss));
        int64_t hi = (s + 1) * ss < nrows ? (s + 1) * ss : nrows;
        for (int64_t r = s * ss; r < hi; ++r)
            for (int64_t e = ptrs[r], j = 0; e < ptrs[r + 1]; ++e, ++j) {
                col[base + j * ss + (r - s * ss)] = ccol[e];
                val[base + j * ss + (r - s * ss)] = cval[e];
            }
    }
}

/* ---- R-MAT ingestion (BASELINE config 3) ------------------------------------
 * corpus_ref.splitmix64 / uniform / rmat_edges / coo_from_entries restated so
 * the whole scale-24 pipeline (268M raw edges -> sorted, duplicate-summed COO)
 * can be checked entry for entry against the device generator, the device
 * radix sort and the device dedup at full size. */

static inline uint64_t or_splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static inline double or_uniform(uint64_t seed, uint64_t ctr) {
    return (double)(or_splitmix64(seed * 0xD1B54A32D192ED03ull + ctr) >> 11) * (1.0 / 9007199254740992.0);
}

/* corpus_ref.rmat_edges for edges [edge_lo, edge_hi): key = row * 2^scale + col */
void or_rmat_keys(int scale, double a, double b, double c, uint64_t seed, int64_t edge_lo, int64_t edge_hi,
                  int64_t* keys, double* vals, int nthreads) {
    set_threads(nthreads);
    const double ab = a + b, abc = a + b + c;
    const uint64_t L = (uint64_t)scale + 1;
#pragma omp parallel for schedule(static)
    for (int64_t e = edge_lo; e < edge_hi; ++e) {
        int64_t row = 0, col = 0;
        for (int l = 0; l < scale; ++l) {
            double u = or_uniform(seed, (uint64_t)e * L + (uint64_t)l);
            int64_t bit = (int64_t)1 << (scale - 1 - l);
            if (u >= ab) row |= bit;
            if ((u >= a && u < ab) || u >= abc) col |= bit;
        }
        keys[e - edge_lo] = (row << scale) | col;
        vals[e - edge_lo] = or_uniform(seed, (uint64_t)e * L + (uint64_t)scale);
    }
}

/* Stable LSD radix sort of (key, value) pairs on the low `key_bits` bits,
 * 8-bit digits. Thread t owns the contiguous block [n t / T, n (t+1) / T);
 * bucket offsets are laid out digit-major, thread-minor, so equal keys keep
 * their input order (np.lexsort is stable). The result ends in keys/vals. */
void or_sort_pairs(int64_t n, int key_bits, int64_t* keys, double* vals, int64_t* keys_alt,
                   double* vals_alt, int nthreads) {
    set_threads(nthreads);
    int64_t* cnt = (int64_t*)malloc(sizeof(int64_t) * 256 * OR_MAX_THREADS);
    int64_t *ks = keys, *kd = keys_alt;
    double *vs = vals, *vd = vals_alt;
    for (int shift = 0; shift < key_bits; shift += 8) {
#pragma omp parallel
        {
            int nt = 1, t = 0;
#ifdef _OPENMP
            nt = omp_get_num_threads();
            t = omp_get_thread_num();
#endif
            if (nt > OR_MAX_THREADS) nt = OR_MAX_THREADS;
            const int64_t lo = n * t / nt, hi = n * (t + 1) / nt;
            int64_t* mine = cnt + 256 * (int64_t)t;
            if (t < nt) {
                memset(mine, 0, sizeof(int64_t) * 256);
                for (int64_t i = lo; i < hi; ++i) ++mine[((uint64_t)ks[i] >> shift) & 255];
            }
#pragma omp barrier
#pragma omp single
            {
                int64_t run = 0;
                for (int d = 0; d < 256; ++d)
                    for (int u = 0; u < nt; ++u) {
                        int64_t v = cnt[256 * (int64_t)u + d];
                        cnt[256 * (int64_t)u + d] = run;
                        run += v;
                    }
            }
            if (t < nt)
                for (int64_t i = lo; i < hi; ++i) {
                    int64_t p = mine[((uint64_t)ks[i] >> shift) & 255]++;
                    kd[p] = ks[i];
                    vd[p] = vs[i];
                }
        }
        int64_t* tk = ks; ks = kd; kd = tk;
        double* tv = vs; vs = vd; vd = tv;
    }
    if (ks != keys) {
        memcpy(keys, ks, sizeof(int64_t) * (size_t)n);
        memcpy(vals, vs, sizeof(double) * (size_t)n);
    }
    free(cnt);
}

/* sparse_ref.coo_from_entries' duplicate sum over sorted keys: each run of
 * equal keys folds 0.0 + v0 + v1 + ... in input order (np.add.at into zeros).
 * Writes int32 row/col and the sums; returns the unique count. */
int64_t or_coo_dedup(int64_t n, int64_t ncols, const int64_t* keys, const double* vals, int32_t* row,
                     int32_t* col, double* out) {
    int64_t u = -1;
    for (int64_t i = 0; i < n; ++i) {
        if (i == 0 || keys[i] != keys[i - 1]) {
            ++u;
            row[u] = (int32_t)(keys[i] / ncols);
            col[u] = (int32_t)(keys[i] % ncols);
            out[u] = 0.0;
        }
        out[u] += vals[i];
    }
    return u + 1;
}
