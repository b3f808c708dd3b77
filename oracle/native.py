"""ctypes binding of oracle/csrc/oracle.c — TEST INFRASTRUCTURE / CPU
BASELINE ONLY (never imported by the product package)."""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.or_max_threads.restype = ctypes.c_int
        L.or_spmv_csr.argtypes = [_I64, _P, _P, _P, _P, _P, ctypes.c_int]
        L.or_spmv_sellp.argtypes = [_I64, _I64, _P, _P, _P, _P, _P, _P, ctypes.c_int]
        L.or_spmv_ell.argtypes = [_I64, _I64, _P, _P, _P, _P, _P, ctypes.c_int]
        L.or_spmv_coo.argtypes = [_I64, _I64, _P, _P, _P, _P, _P, ctypes.c_int]
        L.or_dot.argtypes = [_I64, _P, _P, ctypes.c_int]
        L.or_dot.restype = ctypes.c_double
        L.or_cg_sellp.argtypes = [_I64, _I64, _P, _P, _P, _P, _P, ctypes.c_double, _I64, _P, _P,
                                  ctypes.c_int]
        L.or_cg_sellp.restype = _I64
        L.or_bicgstab_csr.argtypes = [_I64, _P, _P, _P, _P, ctypes.c_double, _I64, _P, _P, ctypes.c_int]
        L.or_bicgstab_csr.restype = _I64
        L.or_gmres_csr.argtypes = [_I64, _P, _P, _P, _P, ctypes.c_double, _I64, _I64, _P, _P,
                                   ctypes.c_int]
        L.or_gmres_csr.restype = _I64
        L.or_stencil_ptrs.argtypes = [_I64, _I64, _I64, ctypes.c_int, _P, _I64, _I64, _P, ctypes.c_int]
        L.or_stencil_ptrs.restype = _I64
        L.or_stencil_fill.argtypes = [_I64, _I64, _I64, ctypes.c_int, _P, _P, _I64, _I64, _P, _P, _P, ctypes.c_int]
        L.or_sellp_sets.argtypes = [_I64, _I64, _P, _P, _P, ctypes.c_int]
        L.or_sellp_sets.restype = _I64
        L.or_sellp_fill.argtypes = [_I64, _I64, _P, _P, _P, _P, _P, _P, ctypes.c_int]
        L.or_rmat_keys.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                   ctypes.c_uint64, _I64, _I64, _P, _P, ctypes.c_int]
        L.or_sort_pairs.argtypes = [_I64, ctypes.c_int, _P, _P, _P, _P, ctypes.c_int]
        L.or_coo_dedup.argtypes = [_I64, _I64, _P, _P, _P, _P, _P]
        L.or_coo_dedup.restype = _I64
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def max_threads():
    return lib().or_max_threads()


class Prepared:
    """Host arrays of one matrix in the C oracle's layout (int32 columns,
    int64 offsets), converted once so timed calls only run the fold."""

    def __init__(self, m):
        self.nrows, self.ncols = int(m.nrows), int(m.ncols)
        self.col = np.ascontiguousarray(np.asarray(m.col_idx), dtype=np.int32)
        self.val = np.ascontiguousarray(np.asarray(m.values), dtype=np.float64)
        if hasattr(m, "slice_sets"):
            self.kind = "sellp"
            self.ss = int(m.slice_size)
            self.sets = np.ascontiguousarray(np.asarray(m.slice_sets), dtype=np.int64)
            self.lengths = np.ascontiguousarray(np.asarray(m.row_lengths), dtype=np.int64)
        elif hasattr(m, "stride"):
            self.kind = "ell"
            self.stride = int(m.stride)
            self.lengths = np.ascontiguousarray(np.asarray(m.row_lengths), dtype=np.int64)
        elif hasattr(m, "row_ptrs"):
            self.kind = "csr"
            self.ptrs = np.ascontiguousarray(np.asarray(m.row_ptrs), dtype=np.int64)
        else:
            self.kind = "coo"
            self.row = np.ascontiguousarray(np.asarray(m.row_idx), dtype=np.int32)

    def spmv(self, x, y=None, nthreads=0):
        x = np.ascontiguousarray(x, dtype=np.float64)
        if y is None:
            y = np.empty(self.nrows, dtype=np.float64)
        L = lib()
        if self.kind == "csr":
            L.or_spmv_csr(self.nrows, _p(self.ptrs), _p(self.col), _p(self.val), _p(x), _p(y), nthreads)
        elif self.kind == "sellp":
            L.or_spmv_sellp(self.nrows, self.ss, _p(self.sets), _p(self.col), _p(self.val),
                            _p(self.lengths), _p(x), _p(y), nthreads)
        elif self.kind == "ell":
            L.or_spmv_ell(self.nrows, self.stride, _p(self.col), _p(self.val), _p(self.lengths),
                          _p(x), _p(y), nthreads)
        else:
            L.or_spmv_coo(self.nrows, len(self.val), _p(self.row), _p(self.col), _p(self.val),
                          _p(x), _p(y), nthreads)
        return y

    def cg(self, b, tol, max_iters, nthreads=0):
        assert self.kind == "sellp"
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty(self.nrows, dtype=np.float64)
        hist = np.empty(max_iters + 1, dtype=np.float64)
        it = lib().or_cg_sellp(self.nrows, self.ss, _p(self.sets), _p(self.col), _p(self.val),
                               _p(self.lengths), _p(b), tol, max_iters, _p(x), _p(hist), nthreads)
        if it < 0:
            raise RuntimeError("CG breakdown")
        return x, hist[: it + 1]


    def bicgstab(self, b, tol, max_iters, nthreads=0):
        """krylov_ref.bicgstab_solve in C (CSR operator)."""
        assert self.kind == "csr"
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty(self.nrows, dtype=np.float64)
        hist = np.empty(max_iters + 1, dtype=np.float64)
        it = lib().or_bicgstab_csr(self.nrows, _p(self.ptrs), _p(self.col), _p(self.val), _p(b), tol,
                                   max_iters, _p(x), _p(hist), nthreads)
        if it < 0:
            raise RuntimeError(f"BiCGSTAB breakdown ({it})")
        return x, hist[: it + 1]

    def gmres(self, b, tol, max_iters, restart=30, nthreads=0):
        """krylov_ref.gmres_solve in C (CSR operator)."""
        assert self.kind == "csr"
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty(self.nrows, dtype=np.float64)
        hist = np.empty(max_iters + 1, dtype=np.float64)
        it = lib().or_gmres_csr(self.nrows, _p(self.ptrs), _p(self.col), _p(self.val), _p(b), tol,
                                max_iters, restart, _p(x), _p(hist), nthreads)
        if it < 0:
            raise MemoryError("GMRES basis allocation failed")
        return x, hist[: it + 1]


def dot(a, b, nthreads=0):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return lib().or_dot(len(a), _p(a), _p(b), nthreads)


def stencil_csr(nx, ny, nz, points, row_lo=0, row_hi=None, nthreads=0):
    """corpus_ref.stencil in C (int32 columns, int64 row pointers)."""
    from types import SimpleNamespace

    from .corpus_ref import _sorted_points

    pts = _sorted_points(points, nx, ny)
    off = np.ascontiguousarray([[p[0], p[1], p[2]] for p in pts], dtype=np.int32)
    vals = np.ascontiguousarray([p[3] for p in pts], dtype=np.float64)
    row_hi = nx * ny * nz if row_hi is None else row_hi
    n = row_hi - row_lo
    ptrs = np.empty(n + 1, dtype=np.int64)
    L = lib()
    nnz = L.or_stencil_ptrs(nx, ny, nz, len(pts), _p(off), row_lo, row_hi, _p(ptrs), nthreads)
    col = np.empty(nnz, dtype=np.int32)
    val = np.empty(nnz, dtype=np.float64)
    L.or_stencil_fill(nx, ny, nz, len(pts), _p(off), _p(vals), row_lo, row_hi, _p(ptrs), _p(col), _p(val), nthreads)
    return SimpleNamespace(nrows=n, ncols=nx * ny * nz, row_ptrs=ptrs, col_idx=col, values=val)


def csr_to_sellp(m, slice_size=64, nthreads=0):
    """sparse_ref.csr_to_sellp in C (sparse.py:219-242)."""
    from types import SimpleNamespace

    n, ss = int(m.nrows), int(slice_size)
    ptrs = np.ascontiguousarray(m.row_ptrs, dtype=np.int64)
    ccol = np.ascontiguousarray(m.col_idx, dtype=np.int32)
    cval = np.ascontiguousarray(m.values, dtype=np.float64)
    nslices = (n + ss - 1) // ss
    sets = np.empty(nslices + 1, dtype=np.int64)
    lengths = np.empty(n, dtype=np.int64)
    L = lib()
    total = L.or_sellp_sets(n, ss, _p(ptrs), _p(sets), _p(lengths), nthreads)
    col = np.empty(total, dtype=np.int32)
    val = np.empty(total, dtype=np.float64)
    L.or_sellp_fill(n, ss, _p(ptrs), _p(ccol), _p(cval), _p(sets), _p(col), _p(val), nthreads)
    return SimpleNamespace(nrows=n, ncols=m.ncols, slice_size=ss, slice_sets=sets, col_idx=col, values=val,
                           row_lengths=lengths)


def rmat_keys(scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=42, nthreads=0):
    """corpus_ref.rmat_edges in C as (row * 2**scale + col int64 keys, values)."""
    n = (1 << scale) * edge_factor
    keys = np.empty(n, dtype=np.int64)
    vals = np.empty(n, dtype=np.float64)
    lib().or_rmat_keys(scale, a, b, c, seed, 0, n, _p(keys), _p(vals), nthreads)
    return keys, vals


def sort_pairs(keys, vals, key_bits=64, nthreads=0):
    """Stable LSD radix sort of (int64 key, f64 value) pairs, in place."""
    assert keys.dtype == np.int64 and vals.dtype == np.float64 and len(keys) == len(vals)
    assert keys.flags.c_contiguous and vals.flags.c_contiguous
    ka, va = np.empty_like(keys), np.empty_like(vals)
    lib().or_sort_pairs(len(keys), key_bits, _p(keys), _p(vals), _p(ka), _p(va), nthreads)
    return keys, vals


def coo_from_keys(nrows, ncols, keys, vals, key_bits=64, nthreads=0):
    """sparse_ref.coo_from_entries (sum_duplicates) on packed keys, in C:
    stable sort, then each duplicate run folded 0.0 + v0 + v1 + ... in input
    order. int32 row/column indices. Sorts keys/vals in place."""
    from types import SimpleNamespace

    sort_pairs(keys, vals, key_bits, nthreads)
    n = len(keys)
    row = np.empty(n, dtype=np.int32)
    col = np.empty(n, dtype=np.int32)
    out = np.empty(n, dtype=np.float64)
    u = lib().or_coo_dedup(n, ncols, _p(keys), _p(vals), _p(row), _p(col), _p(out))
    return SimpleNamespace(nrows=nrows, ncols=ncols, row_idx=row[:u], col_idx=col[:u], values=out[:u])


def rmat_coo(scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=42, nthreads=0):
    """corpus_ref.rmat (sorted, duplicate-summed R-MAT COO) in C."""
    n = 1 << scale
    keys, vals = rmat_keys(scale, edge_factor, a, b, c, seed, nthreads)
    return coo_from_keys(n, n, keys, vals, 2 * scale, nthreads)
