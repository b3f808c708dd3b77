"""Host-side matrix containers of the drop-in API.

Same classes, field names, dtypes (int64 indices, float64 values) and
validation rules as `warpkit/sparse.py` — `CooMatrix` (sparse.py:28-100),
`CsrMatrix` (103-144), `SellpMatrix` (147-209) — plus `EllMatrix` and
`HybridMatrix`, which the reference lacks. These objects only hold and
validate data; every computation on them (SpMV, conversions, solvers,
duplicate summation) runs on the B200 through `device.py`. The validation
loops of the reference (e.g. the per-row Python loop of CsrMatrix,
sparse.py:125-130) are vectorised; the accepted/rejected inputs are the same.
"""

from dataclasses import dataclass

import numpy as np

from .config import is_power_of_two
from .errors import InvalidSliceSize


def _as_index_array(values, name):
    arr = np.asarray(values, dtype=np.int64)
    if arr.ndim != 1:
        raise ValueError(f"{name} must be one-dimensional")
    return arr


def _row_of_entries(row_ptrs, nnz):
    return np.repeat(np.arange(len(row_ptrs) - 1, dtype=np.int64), np.diff(row_ptrs)) if nnz else np.zeros(0, np.int64)


@dataclass(frozen=True, eq=False)
class CooMatrix:
    """Coordinate storage, sorted row-major with unique (row, col) pairs."""

    nrows: int
    ncols: int
    row_idx: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "row_idx", _as_index_array(self.row_idx, "row_idx"))
        object.__setattr__(self, "col_idx", _as_index_array(self.col_idx, "col_idx"))
        object.__setattr__(self, "values", np.asarray(self.values, dtype=np.float64))
        if not (len(self.row_idx) == len(self.col_idx) == len(self.values)):
            raise ValueError("row_idx, col_idx, values must have equal length")
        if self.nrows < 0 or self.ncols < 0:
            raise ValueError("matrix dimensions must be nonnegative")
        if self.nnz:
            if self.row_idx.min() < 0 or self.row_idx.max() >= self.nrows:
                raise ValueError("row index out of bounds")
            if self.col_idx.min() < 0 or self.col_idx.max() >= self.ncols:
                raise ValueError("column index out of bounds")
            keys = self.row_idx * self.ncols + self.col_idx
            if not np.all(np.diff(keys) > 0):
                raise ValueError("entries must be sorted row-major with unique (row, col) pairs")

    @property
    def nnz(self) -> int:
        return len(self.values)

    @classmethod
    def from_entries(cls, nrows, ncols, rows, cols, values, *, sum_duplicates=True, device=None) -> "CooMatrix":
        """Build from unsorted triplets; duplicates are summed (sparse.py:63-80).

        Sorting and duplicate summation run on the GPU (stable key sort, then
        one thread per (row, col) group folding 0.0 + v1 + v2 + ... in input
        order — the `np.add.at` order of the reference).
        """
        from .device import coo_from_entries_device

        return coo_from_entries_device(nrows, ncols, rows, cols, values, sum_duplicates=sum_duplicates,
                                       device=device).to_host()

    def to_dense(self) -> np.ndarray:
        dense = np.zeros((self.nrows, self.ncols))
        dense[self.row_idx, self.col_idx] += self.values
        return dense

    def row_nnz(self) -> np.ndarray:
        return np.bincount(self.row_idx, minlength=self.nrows).astype(np.int64)

    def is_symmetric(self) -> bool:
        if self.nrows != self.ncols:
            return False
        order = np.lexsort((self.row_idx, self.col_idx))
        return (np.array_equal(self.col_idx[order], self.row_idx)
                and np.array_equal(self.row_idx[order], self.col_idx)
                and np.array_equal(self.values[order], self.values))


@dataclass(frozen=True, eq=False)
class CsrMatrix:
    """Compressed sparse row storage with strictly increasing columns per row."""

    nrows: int
    ncols: int
    row_ptrs: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "row_ptrs", _as_index_array(self.row_ptrs, "row_ptrs"))
        object.__setattr__(self, "col_idx", _as_index_array(self.col_idx, "col_idx"))
        object.__setattr__(self, "values", np.asarray(self.values, dtype=np.float64))
        if len(self.row_ptrs) != self.nrows + 1:
            raise ValueError("row_ptrs must have length nrows + 1")
        if self.row_ptrs[0] != 0 or self.row_ptrs[-1] != len(self.values):
            raise ValueError("row_ptrs must start at 0 and end at nnz")
        if np.any(np.diff(self.row_ptrs) < 0):
            raise ValueError("row_ptrs must be nondecreasing")
        if len(self.col_idx) != len(self.values):
            raise ValueError("col_idx and values must have equal length")
        if self.nnz:
            if self.col_idx.min() < 0 or self.col_idx.max() >= self.ncols:
                raise ValueError("column index out of bounds")
            rows = _row_of_entries(self.row_ptrs, self.nnz)
            same_row = rows[1:] == rows[:-1]
            bad = same_row & (np.diff(self.col_idx) <= 0)
            if np.any(bad):
                r = int(rows[1:][bad][0])
                raise ValueError(f"columns of row {r} must be strictly increasing")

    @property
    def nnz(self) -> int:
        return len(self.values)

    def to_dense(self) -> np.ndarray:
        dense = np.zeros((self.nrows, self.ncols))
        rows = _row_of_entries(self.row_ptrs, self.nnz)
        dense[rows, self.col_idx] += self.values
        return dense

    def row_nnz(self) -> np.ndarray:
        return np.diff(self.row_ptrs)


@dataclass(frozen=True, eq=False)
class SellpMatrix:
    """Sliced ELLPACK with padding (sparse.py:147-209).

    Slice s occupies storage [slice_sets[s]*ss, slice_sets[s+1]*ss), column
    major with stride ss; padding entries hold column 0 and value 0.
    """

    nrows: int
    ncols: int
    slice_size: int
    slice_sets: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    row_lengths: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "slice_sets", _as_index_array(self.slice_sets, "slice_sets"))
        object.__setattr__(self, "col_idx", _as_index_array(self.col_idx, "col_idx"))
        object.__setattr__(self, "values", np.asarray(self.values, dtype=np.float64))
        object.__setattr__(self, "row_lengths", _as_index_array(self.row_lengths, "row_lengths"))
        if not is_power_of_two(int(self.slice_size)):
            raise InvalidSliceSize(f"slice_size must be a positive power of two, got {self.slice_size}")
        nslices = (self.nrows + self.slice_size - 1) // self.slice_size
        if len(self.slice_sets) != nslices + 1 or (nslices and self.slice_sets[0] != 0):
            raise ValueError("slice_sets must hold cumulative widths for every slice")
        if len(self.slice_sets) and np.any(np.diff(self.slice_sets) < 0):
            raise ValueError("slice widths must be nonnegative")
        stored = (self.slice_sets[-1] if nslices else 0) * self.slice_size
        if len(self.values) != stored or len(self.col_idx) != stored:
            raise ValueError("storage size must equal slice_size times the total width")
        if len(self.row_lengths) != self.nrows:
            raise ValueError("row_lengths must have one entry per row")

    @property
    def nslices(self) -> int:
        return (self.nrows + self.slice_size - 1) // self.slice_size

    @property
    def nnz(self) -> int:
        return int(self.row_lengths.sum())

    def slice_width(self, s: int) -> int:
        return int(self.slice_sets[s + 1] - self.slice_sets[s])

    def _entry_index(self):
        lens = self.row_lengths
        rows = np.repeat(np.arange(self.nrows, dtype=np.int64), lens)
        pos = np.arange(len(rows), dtype=np.int64) - np.repeat(np.cumsum(lens) - lens, lens)
        ss = self.slice_size
        return rows, self.slice_sets[rows // ss] * ss + pos * ss + rows % ss

    def to_dense(self) -> np.ndarray:
        dense = np.zeros((self.nrows, self.ncols))
        rows, k = self._entry_index()
        np.add.at(dense, (rows, self.col_idx[k]), self.values[k])
        return dense

    def row_nnz(self) -> np.ndarray:
        return self.row_lengths.copy()


@dataclass(frozen=True, eq=False)
class EllMatrix:
    """ELLPACK: one slice of stride `stride` >= nrows, column major.

    Entry j of row r lives at j*stride + r; padding holds (0, 0.0), as in
    SELL-P. `row_lengths` keeps the true per-row counts (the kernels read it
    only when x[0] is not finite).
    """

    nrows: int
    ncols: int
    width: int
    stride: int
    col_idx: np.ndarray
    values: np.ndarray
    row_lengths: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "col_idx", _as_index_array(self.col_idx, "col_idx"))
        object.__setattr__(self, "values", np.asarray(self.values, dtype=np.float64))
        object.__setattr__(self, "row_lengths", _as_index_array(self.row_lengths, "row_lengths"))
        if self.width < 0 or self.stride < self.nrows:
            raise ValueError("ELL needs width >= 0 and stride >= nrows")
        if len(self.values) != self.width * self.stride or len(self.col_idx) != len(self.values):
            raise ValueError("storage size must equal width * stride")
        if len(self.row_lengths) != self.nrows:
            raise ValueError("row_lengths must have one entry per row")
        if self.nrows and (self.row_lengths.min() < 0 or self.row_lengths.max() > self.width):
            raise ValueError("row lengths must lie in [0, width]")

    @property
    def nnz(self) -> int:
        return int(self.row_lengths.sum())

    def to_dense(self) -> np.ndarray:
        dense = np.zeros((self.nrows, self.ncols))
        lens = self.row_lengths
        rows = np.repeat(np.arange(self.nrows, dtype=np.int64), lens)
        pos = np.arange(len(rows), dtype=np.int64) - np.repeat(np.cumsum(lens) - lens, lens)
        k = pos * self.stride + rows
        np.add.at(dense, (rows, self.col_idx[k]), self.values[k])
        return dense

    def row_nnz(self) -> np.ndarray:
        return self.row_lengths.copy()


@dataclass(frozen=True, eq=False)
class HybridMatrix:
    """ELL(width) holding each row's leading entries plus a sorted COO
    remainder (Ginkgo's hybrid format; no reference counterpart)."""

    nrows: int
    ncols: int
    ell: EllMatrix
    coo: CooMatrix

    def __post_init__(self):
        if (self.ell.nrows, self.ell.ncols) != (self.nrows, self.ncols) or \
                (self.coo.nrows, self.coo.ncols) != (self.nrows, self.ncols):
            raise ValueError("ELL and COO parts must have the matrix's shape")

    @property
    def nnz(self) -> int:
        return self.ell.nnz + self.coo.nnz

    def to_dense(self) -> np.ndarray:
        return self.ell.to_dense() + self.coo.to_dense()

    def row_nnz(self) -> np.ndarray:
        return self.ell.row_lengths + self.coo.row_nnz()
