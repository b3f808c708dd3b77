/*
 * CPU oracle, C restatement — TEST INFRASTRUCTURE / CPU BASELINE ONLY.
 *
 * Restates the reference's sequential SpMV fold (warpkit/sparse.py:367-417:
 * per row `acc = 0.0; acc += v * x[c]` in stored order) and its CG loop
 * (warpkit/kernels.py:283-331) in C so the CPU baseline can use every host
 * core. Built with -ffp-contract=off: each product and each sum is rounded
 * separately, so every row result is bitwise identical to the reference no
 * matter how rows are split across OpenMP threads. Dot products use an
 * OpenMP reduction (summation order depends on the thread count, exactly as
 * the reference's OpenBLAS ddot does, see SURVEY.md §7 "Solver parity").
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

double or_dot(int64_t n, const double* a, const double* b, int nthreads) {
    set_threads(nthreads);
    double s = 0.0;
#pragma omp parallel for reduction(+ : s) schedule(static)
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
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
