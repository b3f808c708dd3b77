"""CPU oracle (TEST INFRASTRUCTURE ONLY): sparse formats, conversions and the
sequential SpMV fold of the reference `warpkit.sparse`.

Everything here restates `/root/reference/pkg/src/warpkit/sparse.py` with
vectorised numpy so that config-scale inputs finish in seconds. Bit-exactness
with the reference holds by construction and is pinned by
`tests/test_oracle_golden.py` against fixtures that the reference itself
produced (`tests/golden/make_golden.py`):

* the SpMV fold is `acc = 0.0; acc = acc + (v * x[c])` per row, entries in
  stored order, one rounding for the product and one for the sum — exactly
  `dense_spmv_reference` (sparse.py:367-430). Numpy's elementwise `a * b`
  and `a + b` are separately rounded (no FMA contraction), so folding
  "position j of every row" as one vector step reproduces the scalar loop
  bit for bit;
* conversions are integer bookkeeping plus copies and must match
  `coo_to_csr` (sparse.py:212-216) and `coo_to_sellp` (sparse.py:219-242)
  array for array.

Objects are duck-typed on the reference's field names (`row_ptrs`,
`slice_sets`, `row_idx`, ...), so warpkit matrices, the product package's
host matrices and the plain `SimpleNamespace`s built here all work.
"""

from types import SimpleNamespace

import numpy as np


def _i64(a):
    return np.asarray(a, dtype=np.int64)


def _f64(a):
    return np.asarray(a, dtype=np.float64)


def is_power_of_two(n):
    return n > 0 and (n & (n - 1)) == 0


# -- COO ----------------------------------------------------------------------


def coo_from_entries(nrows, ncols, rows, cols, values, sum_duplicates=True):
    """Sort triplets row-major and sum duplicates (sparse.py:63-80).

    Duplicate groups are summed with `np.add.at` in lexsorted order, the same
    unbuffered left-to-right accumulation the reference uses.
    """
    rows, cols, values = _i64(rows), _i64(cols), _f64(values)
    if len(rows) == 0:
        return SimpleNamespace(nrows=nrows, ncols=ncols, row_idx=rows, col_idx=cols, values=values)
    order = np.lexsort((cols, rows))
    rows, cols, values = rows[order], cols[order], values[order]
    if sum_duplicates:
        keys = rows * max(ncols, 1) + cols
        unique_mask = np.concatenate(([True], np.diff(keys) != 0))
        group_ids = np.cumsum(unique_mask) - 1
        summed = np.zeros(group_ids[-1] + 1, dtype=np.float64)
        np.add.at(summed, group_ids, values)
        rows, cols, values = rows[unique_mask], cols[unique_mask], summed
    return SimpleNamespace(nrows=nrows, ncols=ncols, row_idx=rows, col_idx=cols, values=values)


def coo_row_nnz(nrows, row_idx):
    return np.bincount(_i64(row_idx), minlength=nrows).astype(np.int64)


# -- conversions ----------------------------------------------------------------


def coo_to_csr(m):
    """row counts -> cumsum -> row_ptrs; col/val copied (sparse.py:212-216)."""
    counts = np.zeros(m.nrows + 1, dtype=np.int64)
    counts[1:] = coo_row_nnz(m.nrows, m.row_idx)
    return SimpleNamespace(nrows=m.nrows, ncols=m.ncols, row_ptrs=np.cumsum(counts),
                           col_idx=_i64(m.col_idx).copy(), values=_f64(m.values).copy())


def csr_to_coo(m):
    ptrs = _i64(m.row_ptrs)
    rows = np.repeat(np.arange(m.nrows, dtype=np.int64), np.diff(ptrs))
    return SimpleNamespace(nrows=m.nrows, ncols=m.ncols, row_idx=rows,
                           col_idx=_i64(m.col_idx).copy(), values=_f64(m.values).copy())


def _row_positions(ptrs):
    """For every stored CSR entry: (row, position-within-row)."""
    lengths = np.diff(ptrs)
    rows = np.repeat(np.arange(len(lengths), dtype=np.int64), lengths)
    pos = np.arange(int(ptrs[-1]), dtype=np.int64) - ptrs[rows]
    return rows, pos, lengths


def csr_to_sellp(m, slice_size=64):
    """Vectorised restatement of `coo_to_sellp` (sparse.py:219-242).

    widths[s] = max row length in slice s (0 for an empty slice chunk),
    slice_sets = [0, cumsum(widths)], zero-filled storage with padding
    (col 0, val 0.0), entry j of row r at slice_sets[s]*ss + j*ss + local.
    """
    if not is_power_of_two(slice_size):
        raise ValueError(f"slice_size must be a positive power of two, got {slice_size}")
    ss = int(slice_size)
    ptrs = _i64(m.row_ptrs)
    n = m.nrows
    rows, pos, lengths = _row_positions(ptrs)
    nslices = (n + ss - 1) // ss
    padded = np.zeros(nslices * ss, dtype=np.int64)
    padded[:n] = lengths
    widths = padded.reshape(nslices, ss).max(axis=1) if nslices else np.zeros(0, np.int64)
    slice_sets = np.concatenate(([0], np.cumsum(widths))).astype(np.int64)
    total = int(slice_sets[-1]) * ss if nslices else 0
    col_idx = np.zeros(total, dtype=np.int64)
    values = np.zeros(total, dtype=np.float64)
    k = slice_sets[rows // ss] * ss + pos * ss + rows % ss
    col_idx[k] = _i64(m.col_idx)
    values[k] = _f64(m.values)
    return SimpleNamespace(nrows=n, ncols=m.ncols, slice_size=ss, slice_sets=slice_sets,
                           col_idx=col_idx, values=values, row_lengths=lengths.astype(np.int64))


def csr_to_ell(m, width=None, stride=None):
    """ELL = SELL-P with a single slice of stride `stride` (>= nrows).

    Restated from the SELL-P layout rule (sparse.py:233-241) with one slice:
    entry j of row r at j*stride + r, padding (col 0, val 0.0). `width`
    defaults to the longest row; rows longer than `width` are rejected (that
    is what Hybrid is for).
    """
    ptrs = _i64(m.row_ptrs)
    n = m.nrows
    rows, pos, lengths = _row_positions(ptrs)
    maxlen = int(lengths.max()) if n else 0
    width = maxlen if width is None else int(width)
    if maxlen > width:
        raise ValueError(f"row of length {maxlen} does not fit ELL width {width}")
    stride = n if stride is None else int(stride)
    if stride < n:
        raise ValueError("stride must be >= nrows")
    col_idx = np.zeros(width * stride, dtype=np.int64)
    values = np.zeros(width * stride, dtype=np.float64)
    k = pos * stride + rows
    col_idx[k] = _i64(m.col_idx)
    values[k] = _f64(m.values)
    return SimpleNamespace(nrows=n, ncols=m.ncols, width=width, stride=stride,
                           col_idx=col_idx, values=values, row_lengths=lengths.astype(np.int64))


def hybrid_ell_width(row_lengths, strategy="minimal_storage", percent=0.8):
    """ELL width k for the Hybrid split (no reference; Ginkgo strategies).

    * "imbalance_limit": k = the `percent` quantile of the sorted row lengths
      (Ginkgo `hybrid::imbalance_limit`: sorted[int(n * percent)] clamped).
    * "minimal_storage": k minimising stored bytes 12*k*n + 16*rem(k), where
      rem(k) = sum(max(len - k, 0)). rem decreases by #rows{len > k} per unit
      of k, so the optimum is the smallest k with #rows{len > k} * 16 <= 12*n.
    """
    lengths = np.sort(_i64(row_lengths))
    n = len(lengths)
    if n == 0:
        return 0
    if strategy == "imbalance_limit":
        idx = min(int(n * percent), n - 1)
        return int(lengths[idx])
    if strategy == "minimal_storage":
        # rows_longer(k) = n - searchsorted(lengths, k, 'right')
        k = 0
        maxlen = int(lengths[-1])
        while k < maxlen:
            longer = n - int(np.searchsorted(lengths, k, side="right"))
            if longer * 16 <= 12 * n:
                break
            k += 1
        return k
    raise ValueError(f"unknown hybrid strategy {strategy!r}")


def csr_to_hybrid(m, width, stride=None):
    """Hybrid = ELL(width) holding each row's first min(len, width) entries
    plus a row-major COO remainder with the rest, in column order."""
    ptrs = _i64(m.row_ptrs)
    n = m.nrows
    rows, pos, lengths = _row_positions(ptrs)
    width = int(width)
    stride = n if stride is None else int(stride)
    in_ell = pos < width
    col = _i64(m.col_idx)
    val = _f64(m.values)
    ell_col = np.zeros(width * stride, dtype=np.int64)
    ell_val = np.zeros(width * stride, dtype=np.float64)
    k = pos[in_ell] * stride + rows[in_ell]
    ell_col[k] = col[in_ell]
    ell_val[k] = val[in_ell]
    ell = SimpleNamespace(nrows=n, ncols=m.ncols, width=width, stride=stride, col_idx=ell_col,
                          values=ell_val, row_lengths=np.minimum(lengths, width).astype(np.int64))
    rem = ~in_ell
    coo = SimpleNamespace(nrows=n, ncols=m.ncols, row_idx=rows[rem], col_idx=col[rem], values=val[rem])
    return SimpleNamespace(nrows=n, ncols=m.ncols, ell=ell, coo=coo)


# -- the sequential fold ------------------------------------------------------------


def _fold(starts, step, lengths, cols, vals, x, acc=None):
    """acc[r] = acc[r] + vals[k] * x[cols[k]] for k = starts[r] + j*step,
    j = 0..lengths[r]-1, in that order — vectorised over rows at fixed j.

    Rows are visited longest-first so the active set at step j is a prefix,
    which keeps the total work O(nnz) even for power-law row lengths.
    """
    n = len(lengths)
    if acc is None:
        acc = np.zeros(n, dtype=np.float64)
    if n == 0:
        return acc
    order = np.argsort(-lengths, kind="stable")
    sl = lengths[order]
    st = starts[order]
    a = acc[order].copy()
    maxlen = int(sl[0]) if n else 0
    # active[j] = number of rows with length > j
    active = np.searchsorted(-sl, -np.arange(maxlen), side="left")
    for j in range(maxlen):
        cnt = int(active[j])
        k = st[:cnt] + j * step
        a[:cnt] = a[:cnt] + vals[k] * x[cols[k]]
    out = np.empty_like(acc)
    out[order] = a
    return out


def _check_x(m, x):
    x = _f64(x)
    if x.ndim != 1 or len(x) != m.ncols:
        raise ValueError(f"matrix is {m.nrows}x{m.ncols}, x has length {len(x)}")
    return x


def spmv(m, x):
    """y = A x with the reference's per-row sequential fold (sparse.py:367-417).

    COO folds into y[row] in sorted order (sparse.py:374-383), which equals
    the CSR fold; SELL-P walks only `row_lengths[r]` entries at stride
    `slice_size` (sparse.py:397-417); ELL is the single-slice case; Hybrid
    folds its ELL entries and then continues the same accumulator over the
    row's COO remainder, which again equals the CSR fold.
    """
    if hasattr(m, "ell") and hasattr(m, "coo"):
        x = _check_x(m, x)
        acc = _spmv_ell(m.ell, x)
        c = m.coo
        ptrs = coo_to_csr(c).row_ptrs
        return _fold(ptrs[:-1], 1, np.diff(ptrs), _i64(c.col_idx), _f64(c.values), x, acc)
    x = _check_x(m, x)
    if hasattr(m, "slice_sets"):
        ss = int(m.slice_size)
        rows = np.arange(m.nrows, dtype=np.int64)
        starts = _i64(m.slice_sets)[rows // ss] * ss + rows % ss
        return _fold(starts, ss, _i64(m.row_lengths), _i64(m.col_idx), _f64(m.values), x)
    if hasattr(m, "stride"):
        return _spmv_ell(m, x)
    if hasattr(m, "row_ptrs"):
        ptrs = _i64(m.row_ptrs)
        return _fold(ptrs[:-1], 1, np.diff(ptrs), _i64(m.col_idx), _f64(m.values), x)
    if hasattr(m, "row_idx"):
        ptrs = coo_to_csr(m).row_ptrs
        return _fold(ptrs[:-1], 1, np.diff(ptrs), _i64(m.col_idx), _f64(m.values), x)
    raise TypeError(f"unsupported matrix type {type(m)!r}")


def _spmv_ell(m, x):
    return _fold(np.arange(m.nrows, dtype=np.int64), int(m.stride), _i64(m.row_lengths),
                 _i64(m.col_idx), _f64(m.values), x)


def spmv_loop(m, x):
    """Pure-Python scalar loop over CSR-like storage (small inputs only):
    literal restatement of dense_spmv_reference's CSR branch
    (sparse.py:384-396), used to cross-check `spmv` itself."""
    if not hasattr(m, "row_ptrs"):
        m = coo_to_csr(m)
    xs = _f64(x).tolist()
    ptrs = _i64(m.row_ptrs).tolist()
    cols = _i64(m.col_idx).tolist()
    vals = _f64(m.values).tolist()
    y = [0.0] * m.nrows
    for r in range(m.nrows):
        acc = 0.0
        for k in range(ptrs[r], ptrs[r + 1]):
            acc += vals[k] * xs[cols[k]]
        y[r] = acc
    return np.asarray(y, dtype=np.float64)


def row_nnz(m):
    if hasattr(m, "row_ptrs"):
        return np.diff(_i64(m.row_ptrs))
    if hasattr(m, "row_lengths"):
        return _i64(m.row_lengths)
    if hasattr(m, "ell"):
        return _i64(m.ell.row_lengths) + coo_row_nnz(m.nrows, m.coo.row_idx)
    return coo_row_nnz(m.nrows, m.row_idx)


def max_scaled_rel_err(y, reference, row_nnz):
    """Parity metric of the reference harness (bench.py:43-53):
    max_i |y_i - ref_i| / (max(nnz_i, 1) * max(|ref_i|, 1))."""
    y = _f64(y)
    reference = _f64(reference)
    if y.shape != reference.shape:
        raise ValueError(f"shape mismatch: {y.shape} vs {reference.shape}")
    if len(y) == 0:
        return 0.0
    scale = np.maximum(_f64(row_nnz), 1.0) * np.maximum(np.abs(reference), 1.0)
    return float(np.max(np.abs(y - reference) / scale))


def to_dense(m):
    """Dense reconstruction of any format (cf. the to_dense methods,
    sparse.py:82-85, 135-140, 181-192)."""
    if hasattr(m, "ell") and hasattr(m, "coo"):
        return to_dense(m.ell) + to_dense(m.coo)
    d = np.zeros((m.nrows, m.ncols))
    if hasattr(m, "slice_sets"):
        ss = int(m.slice_size)
        rows = np.repeat(np.arange(m.nrows), _i64(m.row_lengths))
        pos = np.arange(len(rows)) - np.repeat(np.cumsum(_i64(m.row_lengths)) - _i64(m.row_lengths),
                                               _i64(m.row_lengths))
        k = _i64(m.slice_sets)[rows // ss] * ss + pos * ss + rows % ss
        np.add.at(d, (rows, _i64(m.col_idx)[k]), _f64(m.values)[k])
        return d
    if hasattr(m, "stride"):
        lens = _i64(m.row_lengths)
        rows = np.repeat(np.arange(m.nrows), lens)
        pos = np.arange(len(rows)) - np.repeat(np.cumsum(lens) - lens, lens)
        k = pos * int(m.stride) + rows
        np.add.at(d, (rows, _i64(m.col_idx)[k]), _f64(m.values)[k])
        return d
    if hasattr(m, "row_ptrs"):
        m = csr_to_coo(m)
    np.add.at(d, (_i64(m.row_idx), _i64(m.col_idx)), _f64(m.values))
    return d
