"""MatrixMarket coordinate I/O — the on-disk format feeding the SpMV path.

Drop-in for `warpkit.sparse.read_matrix_market` / `write_matrix_market`
(`sparse.py:269-354`): same accepted sources (file-like objects, bytes, a
path, or the text itself), same subset (coordinate; real / integer / pattern;
general / symmetric), same exceptions (`ParseError`, `UnsupportedFormat`),
same result (a `CooMatrix` with duplicates summed by `from_entries`).

The text is parsed by the native multi-threaded parser in libwk_sparse
(`csrc/mmio.cpp`, `wk_mm_read_header` / `wk_mm_parse_entries`); the
duplicate sort + fold runs on the GPU (`CooMatrix.from_entries`), so the
parse -> CSR/SELL-P pipeline never goes through per-entry Python.
"""

import ctypes
import os

import numpy as np

from . import _lib


def _open_stream(source) -> bytes:
    """Byte content of `source` (sparse.py:250-266 rules)."""
    if hasattr(source, "read"):
        data = source.read()
        if isinstance(data, bytes):
            return data
        return data.encode("ascii")
    if isinstance(source, bytes):
        return source
    if isinstance(source, str) and "\n" not in source and os.path.exists(source):
        with open(source, "rb") as fh:
            return fh.read()
    if isinstance(source, os.PathLike):
        with open(source, "rb") as fh:
            return fh.read()
    if isinstance(source, str):
        return source.encode("ascii")
    raise TypeError(f"cannot read MatrixMarket data from {type(source)!r}")


def read_matrix_market_entries(source, nthreads: int = 0):
    """Parse without summing duplicates: (nrows, ncols, rows, cols, values)
    in file order (symmetric: each off-diagonal entry followed by its mirror),
    0-based int64 indices, float64 values."""
    data = _open_stream(source)
    lib = _lib.load()
    buf = ctypes.create_string_buffer(data, len(data))
    hdr = _lib.WkMmHeader()
    _lib.check(lib.wk_mm_read_header(buf, len(data), ctypes.byref(hdr)), "read_matrix_market")
    cap = int(hdr.nnz) * (2 if hdr.symmetric else 1)
    rows = np.empty(cap, dtype=np.int64)
    cols = np.empty(cap, dtype=np.int64)
    vals = np.empty(cap, dtype=np.float64)
    count = ctypes.c_int64(0)
    _lib.check(lib.wk_mm_parse_entries(buf, len(data), ctypes.byref(hdr), int(nthreads), rows.ctypes.data,
                                       cols.ctypes.data, vals.ctypes.data, cap, ctypes.byref(count)),
               "read_matrix_market")
    k = count.value
    return int(hdr.nrows), int(hdr.ncols), rows[:k], cols[:k], vals[:k]


def read_matrix_market(source, *, device=None, nthreads: int = 0):
    """Parse a MatrixMarket coordinate stream into a `CooMatrix`
    (sparse.py:269-335): 1-based -> 0-based, symmetric expanded, pattern
    values 1.0, duplicates summed (`from_entries`, on the GPU). With
    `device=` the result stays on the device (`DeviceCoo`)."""
    nrows, ncols, rows, cols, vals = read_matrix_market_entries(source, nthreads)
    if device is not None:
        from .device import coo_from_entries_device

        return coo_from_entries_device(nrows, ncols, rows, cols, vals, device=device)
    from .sparse import CooMatrix

    return CooMatrix.from_entries(nrows, ncols, rows, cols, vals)


def write_matrix_market(m, target=None) -> str:
    """Serialise as 'coordinate real general' with %.17g values
    (sparse.py:338-353); writes to `target` (path or file-like) if given and
    returns the text."""
    rows = np.ascontiguousarray(np.asarray(m.row_idx, dtype=np.int64))
    cols = np.ascontiguousarray(np.asarray(m.col_idx, dtype=np.int64))
    vals = np.ascontiguousarray(np.asarray(m.values, dtype=np.float64))
    nnz = len(vals)
    lib = _lib.load()
    need = ctypes.c_int64(0)
    _lib.check(lib.wk_mm_write(m.nrows, m.ncols, nnz, rows.ctypes.data, cols.ctypes.data, vals.ctypes.data, None, 0,
                               ctypes.byref(need)), "write_matrix_market")
    out = ctypes.create_string_buffer(need.value)
    _lib.check(lib.wk_mm_write(m.nrows, m.ncols, nnz, rows.ctypes.data, cols.ctypes.data, vals.ctypes.data, out,
                               need.value, ctypes.byref(need)), "write_matrix_market")
    text = out.raw[: need.value].decode("ascii")
    if target is not None:
        if hasattr(target, "write"):
            target.write(text)
        else:
            with open(target, "w") as fh:
                fh.write(text)
    return text
