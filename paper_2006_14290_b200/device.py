"""Device-resident matrices (HBM layout) and the on-device conversions.

Layout in HBM (see DESIGN.md §Data layout): values float64, column/row
indices int32, row pointers int32, SELL-P slice_sets int64, row_lengths
int32. PyTorch tensors own the buffers (plumbing only); every operation on
them is a libwk_sparse kernel called through the C ABI on the current torch
stream.

Host objects (`sparse.py`, or the reference's own warpkit dataclasses —
duck-typed on field names) are uploaded once and cached per object, like the
reference caches list views per matrix (`kernels.py:80-95`).
"""

import ctypes
import weakref

import numpy as np
import torch

from . import _lib
from ._lib import P, WkMatrix
from .errors import DimensionMismatch, InvalidSliceSize

INT32_MAX = 2**31 - 1


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None and t.numel() else ctypes.c_void_p(0)


def stream_handle(device=None):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _dev(device):
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    if isinstance(device, torch.device):
        return device if device.index is not None else torch.device("cuda", torch.cuda.current_device())
    return torch.device("cuda", int(device))


def _i32(a, device, name):
    a = np.asarray(a)
    if a.size and (a.max() > INT32_MAX or a.min() < -INT32_MAX - 1):
        raise ValueError(f"{name} does not fit the int32 device layout")
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(device)


def _f64(a, device):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(device)


def _i64(a, device):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64)).to(device)


def _np64(t):
    return t.to(torch.int64).cpu().numpy()


class _Workspace:
    """Per-(device, stream) scratch: reduction partials (zeroed once; tickets
    are self-cleaning) and a growable scan buffer. Keyed on the current
    stream too, so reductions enqueued on different streams never share the
    partials / ticket of one workspace."""

    _per_device = {}

    def __init__(self, device):
        self.device = device
        self.red = torch.zeros(int(_lib.load().wk_reduce_workspace_bytes()), dtype=torch.uint8, device=device)
        self.scan = torch.empty(0, dtype=torch.uint8, device=device)
        self.scalar = torch.zeros(64, dtype=torch.float64, device=device)

    @classmethod
    def get(cls, device):
        device = _dev(device)
        key = (device.index, torch.cuda.current_stream(device).cuda_stream)
        ws = cls._per_device.get(key)
        if ws is None:
            ws = cls(device)
            cls._per_device[key] = ws
        return ws

    def scan_ws(self, n):
        need = int(_lib.load().wk_scan_workspace_bytes(int(n)))
        if self.scan.numel() < need:
            self.scan = torch.empty(need, dtype=torch.uint8, device=self.device)
        return self.scan


def workspace(device=None):
    return _Workspace.get(device)


# ---- device matrices -------------------------------------------------------------


class DeviceMatrix:
    """Common interface of the device twins."""

    fmt = None

    def wk(self) -> WkMatrix:
        """The `wk_matrix` operand (kept alive by this object)."""
        if getattr(self, "_wk", None) is None:
            self._wk = self._make_wk()
        return self._wk

    def wk_ptr(self):
        return ctypes.byref(self.wk())

    @property
    def shape(self):
        return (self.nrows, self.ncols)


class DeviceCsr(DeviceMatrix):
    fmt = "csr"

    def __init__(self, nrows, ncols, row_ptrs, col_idx, values):
        self.nrows, self.ncols = int(nrows), int(ncols)
        self.row_ptrs, self.col_idx, self.values = row_ptrs, col_idx, values
        self.device = values.device
        self.nnz = int(values.numel())
        self._plan = None
        self._wk = None
        self.strategy = None  # "auto", resolved at the first launch (auto_strategy)
        self.subwarp = 0
        self._auto = None

    def plan(self):
        """nnz-chunk plan of the load-balanced stream kernel (built once)."""
        if self._plan is None:
            L = _lib.load()
            self._plan = torch.empty(int(L.wk_csr_plan_bytes(self.nnz)), dtype=torch.uint8, device=self.device)
            _lib.call("wk_csr_plan_build", self.nrows, self.nnz, _ptr(self.row_ptrs), _ptr(self._plan),
                      stream_handle(self.device))
        return self._plan

    def merge_plan(self):
        """merge-path tile coordinates + per-tile carry slots (built once)."""
        if getattr(self, "_merge_plan", None) is None:
            L = _lib.load()
            nb = int(L.wk_csr_merge_plan_bytes(self.nrows, self.nnz))
            self._merge_plan = torch.empty(nb, dtype=torch.uint8, device=self.device)
            _lib.call("wk_csr_merge_plan_build", self.nrows, self.nnz, _ptr(self.row_ptrs), _ptr(self._merge_plan),
                      stream_handle(self.device))
        return self._merge_plan

    def load_balance_plan(self):
        """head plan of the load-balance kernel (segwarp.cuh HeadPlan: per 256-entry
        window the row-start mask and head count, the row id of every head;
        built once)."""
        if getattr(self, "_lb_plan", None) is None:
            L = _lib.load()
            self._lb_plan = torch.empty(int(L.wk_csr_load_balance_plan_bytes(self.nrows, self.nnz)), dtype=torch.uint8,
                                        device=self.device)
            _lib.call("wk_csr_load_balance_plan_build", self.nrows, self.nnz, _ptr(self.row_ptrs),
                      _ptr(self._lb_plan), stream_handle(self.device))
        return self._lb_plan

    def auto_strategy(self):
        """rowblock when every row is short and the mean is moderate (one lane
        folds one row from a TMA-staged block; bitwise), load_balance
        otherwise (Ginkgo's choice for irregular matrices: equal nonzeros per
        warp whatever the row-length skew). Decided once per matrix (one D2H
        read); deterministic (range carries added in range order, no
        atomics). `merge` (deterministic) and `stream` (bitwise) are explicit
        choices."""
        if getattr(self, "_auto", None) is None:
            if self.nrows == 0:
                self._auto = "load_balance"
            else:
                maxlen = max_row_length(self)
                self._auto = "rowblock" if maxlen <= 64 and self.nnz <= 28 * self.nrows else "load_balance"
        return self._auto

    def with_strategy(self, strategy, subwarp=0):
        if strategy == "auto":
            strategy = self.auto_strategy()
        st = {"stream": _lib.WK_CSR_STREAM, "subwarp": _lib.WK_CSR_SUBWARP, "rowblock": _lib.WK_CSR_ROWBLOCK,
              "merge": _lib.WK_CSR_MERGE, "load_balance": _lib.WK_CSR_LOAD_BALANCE}[strategy]
        if st != self.strategy or subwarp != self.subwarp:
            self.strategy, self.subwarp = st, int(subwarp)
            self._wk = None
        return self

    def _make_wk(self):
        if self.strategy is None:
            self.with_strategy("auto")
        m = WkMatrix()
        m.format = _lib.WK_FMT_CSR
        m.csr_strategy = self.strategy
        m.subwarp_size = self.subwarp
        m.nrows, m.ncols, m.nnz = self.nrows, self.ncols, self.nnz
        m.row_ptrs, m.col_idx, m.values = _ptr(self.row_ptrs), _ptr(self.col_idx), _ptr(self.values)
        if self.strategy == _lib.WK_CSR_STREAM:
            m.plan = _ptr(self.plan())
        elif self.strategy == _lib.WK_CSR_MERGE:
            m.plan = _ptr(self.merge_plan())
        elif self.strategy == _lib.WK_CSR_LOAD_BALANCE:
            m.plan = _ptr(self.load_balance_plan())
        return m

    def row_lengths(self):
        out = torch.empty(self.nrows, dtype=torch.int32, device=self.device)
        _lib.call("wk_csr_row_lengths", self.nrows, _ptr(self.row_ptrs), _ptr(out), stream_handle(self.device))
        return out

    def algorithmic_bytes(self):
        """12 B per entry + 4(n+1) row_ptrs + 8 ncols (x) + 8 nrows (y)."""
        return 12 * self.nnz + 4 * (self.nrows + 1) + 8 * self.ncols + 8 * self.nrows

    def to_host(self):
        from .sparse import CsrMatrix

        return CsrMatrix(self.nrows, self.ncols, _np64(self.row_ptrs), _np64(self.col_idx), self.values.cpu().numpy())


class DeviceCoo(DeviceMatrix):
    fmt = "coo"

    def __init__(self, nrows, ncols, row_idx, col_idx, values):
        self.nrows, self.ncols = int(nrows), int(ncols)
        self.row_idx, self.col_idx, self.values = row_idx, col_idx, values
        self.device = values.device
        self.nnz = int(values.numel())
        self._wk = None

    def _make_wk(self):
        m = WkMatrix()
        m.format = _lib.WK_FMT_COO
        m.nrows, m.ncols, m.nnz = self.nrows, self.ncols, self.nnz
        m.row_idx, m.col_idx, m.values = _ptr(self.row_idx), _ptr(self.col_idx), _ptr(self.values)
        return m

    def algorithmic_bytes(self):
        """16 B per entry (row, col int32 + value) + x + y."""
        return 16 * self.nnz + 8 * self.ncols + 8 * self.nrows

    def to_host(self):
        from .sparse import CooMatrix

        return CooMatrix(self.nrows, self.ncols, _np64(self.row_idx), _np64(self.col_idx), self.values.cpu().numpy())


class DeviceSellp(DeviceMatrix):
    fmt = "sellp"

    def __init__(self, nrows, ncols, slice_size, slice_sets, col_idx, values, row_lengths):
        self.nrows, self.ncols, self.slice_size = int(nrows), int(ncols), int(slice_size)
        self.slice_sets, self.col_idx, self.values, self.row_lengths_t = slice_sets, col_idx, values, row_lengths
        self.device = values.device
        self.stored = int(values.numel())
        self._nnz = None
        self._wk = None

    @property
    def nslices(self):
        return (self.nrows + self.slice_size - 1) // self.slice_size

    @property
    def nnz(self):
        if self._nnz is None:
            self._nnz = int(self.row_lengths_t.sum().item()) if self.nrows else 0
        return self._nnz

    def _make_wk(self):
        m = WkMatrix()
        m.format = _lib.WK_FMT_SELLP
        m.nrows, m.ncols, m.nnz = self.nrows, self.ncols, self.stored
        m.col_idx, m.values = _ptr(self.col_idx), _ptr(self.values)
        m.slice_size, m.slice_sets, m.row_lengths = self.slice_size, _ptr(self.slice_sets), _ptr(self.row_lengths_t)
        return m

    def algorithmic_bytes(self):
        """12 B per stored slot (padding included) + 8(nslices+1) + x + y."""
        return 12 * self.stored + 8 * (self.nslices + 1) + 8 * self.ncols + 8 * self.nrows

    def to_host(self):
        from .sparse import SellpMatrix

        return SellpMatrix(self.nrows, self.ncols, self.slice_size, self.slice_sets.cpu().numpy(),
                           _np64(self.col_idx), self.values.cpu().numpy(), _np64(self.row_lengths_t))


class DeviceEll(DeviceMatrix):
    fmt = "ell"

    def __init__(self, nrows, ncols, width, stride, col_idx, values, row_lengths):
        self.nrows, self.ncols, self.width, self.stride = int(nrows), int(ncols), int(width), int(stride)
        self.col_idx, self.values, self.row_lengths_t = col_idx, values, row_lengths
        self.device = values.device
        self.stored = int(values.numel())
        self._nnz = None
        self._wk = None

    @property
    def nnz(self):
        if self._nnz is None:
            self._nnz = int(self.row_lengths_t.sum().item()) if self.nrows else 0
        return self._nnz

    def _fill_wk(self, m):
        m.nrows, m.ncols = self.nrows, self.ncols
        m.col_idx, m.values = _ptr(self.col_idx), _ptr(self.values)
        m.width, m.stride, m.row_lengths = self.width, self.stride, _ptr(self.row_lengths_t)

    def _make_wk(self):
        m = WkMatrix()
        m.format = _lib.WK_FMT_ELL
        self._fill_wk(m)
        m.nnz = self.stored
        return m

    def algorithmic_bytes(self):
        """12 B per stored slot (width * stride) + x + y."""
        return 12 * self.stored + 8 * self.ncols + 8 * self.nrows

    def to_host(self):
        from .sparse import EllMatrix

        return EllMatrix(self.nrows, self.ncols, self.width, self.stride, _np64(self.col_idx),
                         self.values.cpu().numpy(), _np64(self.row_lengths_t))


class DeviceHybrid(DeviceMatrix):
    fmt = "hybrid"

    def __init__(self, ell: DeviceEll, coo: DeviceCoo):
        self.ell, self.coo = ell, coo
        self.nrows, self.ncols = ell.nrows, ell.ncols
        self.device = ell.device
        self._wk = None

    @property
    def nnz(self):
        return self.ell.nnz + self.coo.nnz

    def _make_wk(self):
        m = WkMatrix()
        m.format = _lib.WK_FMT_HYBRID
        self.ell._fill_wk(m)
        m.nnz = self.ell.stored + self.coo.nnz
        m.coo_nnz = self.coo.nnz
        m.coo_row, m.coo_col, m.coo_val = _ptr(self.coo.row_idx), _ptr(self.coo.col_idx), _ptr(self.coo.values)
        return m

    def algorithmic_bytes(self):
        """ELL part 12 B/slot (padding included) + COO
        part 16 B/entry + x read once + y written once = 12kn + 16 rem + 16n."""
        return 12 * self.ell.stored + 16 * self.coo.nnz + 8 * self.ncols + 8 * self.nrows

    def to_host(self):
        from .sparse import HybridMatrix

        return HybridMatrix(self.nrows, self.ncols, self.ell.to_host(), self.coo.to_host())


# ---- upload / download ------------------------------------------------------------------

_CACHE = {}


def _format_of(m):
    if isinstance(m, DeviceMatrix):
        return m.fmt
    if hasattr(m, "ell") and hasattr(m, "coo"):
        return "hybrid"
    if hasattr(m, "slice_sets"):
        return "sellp"
    if hasattr(m, "stride") and hasattr(m, "width"):
        return "ell"
    if hasattr(m, "row_ptrs"):
        return "csr"
    if hasattr(m, "row_idx"):
        return "coo"
    raise TypeError(f"unsupported matrix type {type(m)!r}")


def upload(m, device=None) -> DeviceMatrix:
    """Copy a host matrix (this package's or warpkit's) into HBM. SELL-P and
    ELL padding slots are rewritten as (col 0, val 0.0) in the device copy
    (the reference only folds row_lengths entries, sparse.py:413; the device
    kernels fold whole slices, so other padding, e.g. Ginkgo's col -1, must
    not reach them)."""
    dev = _dev(device)
    fmt = _format_of(m)
    if fmt == "csr":
        return DeviceCsr(m.nrows, m.ncols, _i32(m.row_ptrs, dev, "row_ptrs"), _i32(m.col_idx, dev, "col_idx"),
                         _f64(m.values, dev))
    if fmt == "coo":
        return DeviceCoo(m.nrows, m.ncols, _i32(m.row_idx, dev, "row_idx"), _i32(m.col_idx, dev, "col_idx"),
                         _f64(m.values, dev))
    if fmt == "sellp":
        d = DeviceSellp(m.nrows, m.ncols, m.slice_size, _i64(m.slice_sets, dev), _i32(m.col_idx, dev, "col_idx"),
                        _f64(m.values, dev), _i32(m.row_lengths, dev, "row_lengths"))
        _lib.call("wk_sellp_zero_padding", d.nrows, d.slice_size, _ptr(d.slice_sets), _ptr(d.row_lengths_t),
                  _ptr(d.col_idx), _ptr(d.values), stream_handle(dev))
        return d
    if fmt == "ell":
        d = DeviceEll(m.nrows, m.ncols, m.width, m.stride, _i32(m.col_idx, dev, "col_idx"), _f64(m.values, dev),
                      _i32(m.row_lengths, dev, "row_lengths"))
        _lib.call("wk_ell_zero_padding", d.nrows, d.width, d.stride, _ptr(d.row_lengths_t), _ptr(d.col_idx),
                  _ptr(d.values), stream_handle(dev))
        return d
    return DeviceHybrid(upload(m.ell, dev), upload(m.coo, dev))


_ARRAY_FIELDS = {"csr": ("row_ptrs", "col_idx", "values"), "coo": ("row_idx", "col_idx", "values"),
                 "sellp": ("slice_sets", "col_idx", "values", "row_lengths"),
                 "ell": ("col_idx", "values", "row_lengths")}


def _host_arrays(m):
    fmt = _format_of(m)
    if fmt == "hybrid":
        return _host_arrays(m.ell) + _host_arrays(m.coo)
    return [getattr(m, k) for k in _ARRAY_FIELDS[fmt]]


def _fingerprint(arrs):
    """Identity of the host buffers: data pointer, shape, dtype and the
    writeable flag (cleared while the upload is cached)."""
    return tuple((a.__array_interface__["data"][0], a.shape, a.dtype.str, a.strides, bool(a.flags.writeable))
                 for a in arrs)


def as_device(m, device=None) -> DeviceMatrix:
    """Device twin of `m`: itself if already on the device, else an upload
    cached for as long as `m` lives.

    While cached, the host arrays are frozen (numpy writeable = False), so an
    in-place edit raises instead of silently running on the stale device
    copy; the cache entry is re-validated on every call (same buffers, still
    frozen) and re-uploaded otherwise (e.g. after `arr.flags.writeable =
    True`, or new arrays). `release(m)` drops the entry and unfreezes the
    arrays it froze. Matrices whose arrays are not numpy arrays are uploaded
    on every call."""
    if isinstance(m, DeviceMatrix):
        return m
    dev = _dev(device)
    key = (id(m), dev.index)
    hit = _CACHE.get(key)
    try:
        arrs = _host_arrays(m)
    except AttributeError:
        arrs = None
    cacheable = arrs is not None and all(isinstance(a, np.ndarray) for a in arrs)
    if hit is not None and hit[0]() is m and cacheable and hit[2] == _fingerprint(arrs):
        return hit[1]
    if hit is not None:
        release(m, dev)
    twin = upload(m, dev)
    if not cacheable:
        return twin
    frozen = []
    for a in arrs:
        if a.flags.writeable:
            try:
                a.flags.writeable = False
                frozen.append(a)
            except ValueError:
                pass
    try:
        ref = weakref.ref(m, lambda _r, k=key: _drop(k))
    except TypeError:
        for a in frozen:
            a.flags.writeable = True
        return twin
    _CACHE[key] = (ref, twin, _fingerprint(arrs), frozen)
    return twin


def _thaw(arrays):
    for a in arrays:
        try:
            a.flags.writeable = True
        except ValueError:
            pass


def _drop(key):
    ent = _CACHE.pop(key, None)
    if ent is not None:
        _thaw(ent[3])


def release(m, device=None):
    """Drop the cached device copy of host matrix `m` (all devices when
    `device` is None) and make the arrays `as_device` froze writeable again."""
    keys = [k for k in _CACHE if k[0] == id(m) and (device is None or k[1] == _dev(device).index)]
    for k in keys:
        ent = _CACHE.pop(k)
        if ent[0]() is m:
            _thaw(ent[3])


def check_vector(x, n, name="x"):
    """`_check_spmv_dims` (kernels.py:106-110) before any device work: x must
    be 1-D of length n, else DimensionMismatch."""
    shape = tuple(x.shape) if isinstance(x, torch.Tensor) else np.shape(x)
    if len(shape) != 1 or shape[0] != n:
        raise DimensionMismatch(f"matrix needs {name} of length {n}, got shape {shape}")


def as_device_vector(x, n, device=None, name="x"):
    """(tensor on device, came_from_host). Raises DimensionMismatch like
    `_check_spmv_dims` (kernels.py:106-110)."""
    dev = _dev(device)
    if isinstance(x, torch.Tensor):
        if x.dim() != 1 or x.numel() != n:
            raise DimensionMismatch(f"{name} has shape {tuple(x.shape)}, expected ({n},)")
        if x.device.type == "cpu":
            # host torch tensor (pinned -> asynchronous DMA); the result goes
            # back to the host as a torch tensor (see to_host_like)
            xt = x.to(dtype=torch.float64).contiguous().to(dev, non_blocking=x.is_pinned())
            return xt, "torch_pinned" if x.is_pinned() else "torch"
        if x.device != dev or x.dtype != torch.float64 or not x.is_contiguous():
            x = x.to(device=dev, dtype=torch.float64).contiguous()
        return x, False
    arr = np.asarray(x, dtype=np.float64)
    if arr.ndim != 1 or len(arr) != n:
        raise DimensionMismatch(f"matrix needs {name} of length {n}, got shape {arr.shape}")
    return torch.from_numpy(np.ascontiguousarray(arr)).to(dev), True


def to_host_like(y, host):
    """Return device result `y` in the caller's host representation."""
    if not host:
        return y
    if host == "torch_pinned":
        out = torch.empty(y.shape, dtype=y.dtype, pin_memory=True)
        out.copy_(y, non_blocking=True)
        torch.cuda.current_stream(y.device).synchronize()
        return out
    if host == "torch":
        return y.cpu()
    return y.cpu().numpy()


# ---- conversions (bit-exact; sparse.py:212-242 semantics) -------------------------------------


def coo_to_csr(m, device=None) -> DeviceCsr:
    """row_ptrs from the sorted row indices (sparse.py:212-216); columns and
    values are shared with the COO (device arrays are immutable here)."""
    d = as_device(m, device)
    ptrs = torch.empty(d.nrows + 1, dtype=torch.int32, device=d.device)
    _lib.call("wk_coo_to_csr_ptrs", d.nrows, d.nnz, _ptr(d.row_idx), _ptr(ptrs), stream_handle(d.device))
    return DeviceCsr(d.nrows, d.ncols, ptrs, d.col_idx, d.values)


def csr_to_coo(m, device=None) -> DeviceCoo:
    d = as_device(m, device)
    rows = torch.empty(d.nnz, dtype=torch.int32, device=d.device)
    _lib.call("wk_csr_to_coo_rows", d.nrows, _ptr(d.row_ptrs), _ptr(rows), stream_handle(d.device))
    return DeviceCoo(d.nrows, d.ncols, rows, d.col_idx, d.values)


def _check_slice(slice_size):
    if not (isinstance(slice_size, (int, np.integer)) and slice_size > 0 and (slice_size & (slice_size - 1)) == 0):
        raise InvalidSliceSize(f"slice_size must be a positive power of two, got {slice_size}")


def csr_to_sellp(m, slice_size=64, device=None) -> DeviceSellp:
    """sparse.py:219-242 on the device: per-slice max row length, cumulative
    widths, zero-filled column-major storage."""
    _check_slice(slice_size)
    d = as_device(m, device)
    st = stream_handle(d.device)
    ws = workspace(d.device)
    nslices = (d.nrows + slice_size - 1) // slice_size
    sets = torch.empty(nslices + 1, dtype=torch.int64, device=d.device)
    lengths = torch.empty(d.nrows, dtype=torch.int32, device=d.device)
    _lib.call("wk_csr_to_sellp_sets", d.nrows, slice_size, _ptr(d.row_ptrs), _ptr(sets), _ptr(lengths),
              _ptr(ws.scan_ws(nslices)), st)
    total = int(sets[-1].item()) * slice_size
    col = torch.empty(total, dtype=torch.int32, device=d.device)
    val = torch.empty(total, dtype=torch.float64, device=d.device)
    _lib.call("wk_csr_to_sellp_fill", d.nrows, slice_size, _ptr(d.row_ptrs), _ptr(d.col_idx), _ptr(d.values),
              _ptr(sets), _ptr(col), _ptr(val), st)
    out = DeviceSellp(d.nrows, d.ncols, slice_size, sets, col, val, lengths)
    out._nnz = d.nnz
    return out


def max_row_length(m, device=None) -> int:
    d = as_device(m, device)
    res = torch.empty(1, dtype=torch.int64, device=d.device)
    _lib.call("wk_csr_max_row_length", d.nrows, _ptr(d.row_ptrs), _ptr(res), stream_handle(d.device))
    return int(res.item())


def csr_to_ell(m, width=None, stride=None, device=None) -> DeviceEll:
    """ELL(width, stride): entry j of row r at j*stride + r, padding (0, 0.0).
    Rows longer than `width` are rejected (use Hybrid)."""
    d = as_device(m, device)
    maxlen = max_row_length(d)
    width = maxlen if width is None else int(width)
    if maxlen > width:
        raise ValueError(f"row of length {maxlen} does not fit ELL width {width}")
    stride = d.nrows if stride is None else int(stride)
    if stride < d.nrows:
        raise ValueError("stride must be >= nrows")
    return _ell_fill(d, width, stride)


def _ell_fill(d, width, stride):
    col = torch.empty(width * stride, dtype=torch.int32, device=d.device)
    val = torch.empty(width * stride, dtype=torch.float64, device=d.device)
    lengths = torch.empty(d.nrows, dtype=torch.int32, device=d.device)
    _lib.call("wk_csr_to_ell_fill", d.nrows, width, stride, _ptr(d.row_ptrs), _ptr(d.col_idx), _ptr(d.values),
              _ptr(col), _ptr(val), _ptr(lengths), stream_handle(d.device))
    return DeviceEll(d.nrows, d.ncols, width, stride, col, val, lengths)


def row_length_histogram(m, nbins=None, device=None) -> np.ndarray:
    d = as_device(m, device)
    if nbins is None:
        nbins = min(max_row_length(d) + 1, 1 << 16)
    hist = torch.empty(max(int(nbins), 1), dtype=torch.int64, device=d.device)
    _lib.call("wk_csr_row_length_histogram", d.nrows, _ptr(d.row_ptrs), hist.numel(), _ptr(hist),
              stream_handle(d.device))
    return hist.cpu().numpy()


def hybrid_width(m, strategy="minimal_storage", percent=0.8, device=None) -> int:
    """ELL width of the Hybrid split from the device row-length histogram
    (same rules as oracle.sparse_ref.hybrid_ell_width)."""
    d = as_device(m, device)
    if d.nrows == 0:
        return 0
    hist = row_length_histogram(d)
    n = d.nrows
    if strategy == "imbalance_limit":
        idx = min(int(n * percent), n - 1)
        cum = np.cumsum(hist)
        return int(np.searchsorted(cum, idx, side="right"))
    if strategy == "minimal_storage":
        # rows longer than k: n - cumsum(hist)[k]; smallest k with 16*longer <= 12*n
        longer = n - np.cumsum(hist)
        ok = np.nonzero(longer * 16 <= 12 * n)[0]
        return int(ok[0]) if len(ok) else len(hist) - 1
    raise ValueError(f"unknown hybrid strategy {strategy!r}")


def csr_to_hybrid(m, width=None, strategy="minimal_storage", percent=0.8, stride=None, device=None) -> DeviceHybrid:
    d = as_device(m, device)
    if width is None:
        width = hybrid_width(d, strategy, percent)
    width = int(width)
    stride = d.nrows if stride is None else int(stride)
    ell = _ell_fill(d, width, stride)
    st = stream_handle(d.device)
    ws = workspace(d.device)
    offsets = torch.empty(d.nrows + 1, dtype=torch.int64, device=d.device)
    _lib.call("wk_hybrid_coo_offsets", d.nrows, width, _ptr(d.row_ptrs), _ptr(offsets), _ptr(ws.scan_ws(d.nrows)), st)
    rem = int(offsets[-1].item())
    crow = torch.empty(rem, dtype=torch.int32, device=d.device)
    ccol = torch.empty(rem, dtype=torch.int32, device=d.device)
    cval = torch.empty(rem, dtype=torch.float64, device=d.device)
    if rem:
        nwork = int(_lib.load().wk_hybrid_coo_fill_workspace(rem))
        work = torch.empty((nwork + 15) // 16 * 2, dtype=torch.int64, device=d.device)
        _lib.call("wk_hybrid_coo_fill", d.nrows, width, _ptr(d.row_ptrs), _ptr(d.col_idx), _ptr(d.values),
                  _ptr(offsets), _ptr(crow), _ptr(ccol), _ptr(cval), _ptr(work), nwork, st)
    return DeviceHybrid(ell, DeviceCoo(d.nrows, d.ncols, crow, ccol, cval))


def coo_from_entries_device(nrows, ncols, rows, cols, values, sum_duplicates=True, device=None) -> DeviceCoo:
    """Sort triplets row-major and sum duplicates (sparse.py:63-80) on the GPU.

    The key sort is `wk_sort_pairs_u64_f64` (stable LSD radix sort over the
    bits of nrows * ncols, values moved with their keys); the duplicate fold
    is `wk_coo_dedup_count` + `wk_coo_dedup_scatter`: 0.0 + v1 + v2 + ... per
    key in input order, which is `np.add.at` on zeros in the reference.
    """
    dev = _dev(device)
    r = torch.as_tensor(np.asarray(rows, dtype=np.int64), device=dev) if not isinstance(rows, torch.Tensor) else rows.to(dev, torch.int64)
    c = torch.as_tensor(np.asarray(cols, dtype=np.int64), device=dev) if not isinstance(cols, torch.Tensor) else cols.to(dev, torch.int64)
    v = torch.as_tensor(np.asarray(values, dtype=np.float64), device=dev) if not isinstance(values, torch.Tensor) else values.to(dev, torch.float64)
    if not (r.numel() == c.numel() == v.numel()):
        raise ValueError("rows, cols, values must have equal length")
    n = r.numel()
    if n and (int(r.min()) < 0 or int(r.max()) >= nrows or int(c.min()) < 0 or int(c.max()) >= ncols):
        raise ValueError("index out of bounds")
    keys = r * max(int(ncols), 1) + c
    return coo_from_keys(nrows, ncols, keys, v, sum_duplicates=sum_duplicates)


def sort_pairs(keys, values, key_bits=64, inplace=False):
    """Stable sort of int64 keys (>= 0, < 2**key_bits) with their f64 values
    (csrc/sort.cu, 8-bit LSD passes over the low key_bits bits). Returns the
    sorted (keys, values); with inplace=True the given contiguous tensors are
    sorted and returned, otherwise copies."""
    n = keys.numel()
    if inplace:
        assert keys.is_contiguous() and values.is_contiguous() and values.dtype == torch.float64
        assert keys.data_ptr() % 16 == 0 and values.data_ptr() % 16 == 0, "sort_pairs needs 16-byte aligned tensors"
        k, v = keys, values
    else:
        k = keys.contiguous().clone()
        v = values.to(torch.float64).contiguous().clone()
    if n <= 1:
        return k, v
    ka = torch.empty_like(k)
    va = torch.empty_like(v)
    nwork = int(_lib.load().wk_sort_pairs_workspace(n))
    work = torch.empty((nwork + 15) // 16 * 2, dtype=torch.int64, device=k.device)
    _lib.call("wk_sort_pairs_u64_f64", n, int(key_bits), _ptr(k), _ptr(v), _ptr(ka), _ptr(va), _ptr(work), nwork,
              stream_handle(k.device))
    return k, v


def coo_from_keys(nrows, ncols, keys, values, sum_duplicates=True, owned=False) -> DeviceCoo:
    """COO from int64 keys row * ncols + col (any order, duplicates allowed)
    and values; owned=True lets the sort reorder `keys` / `values` in place."""
    dev = keys.device
    n = keys.numel()
    if n == 0:
        e32 = torch.empty(0, dtype=torch.int32, device=dev)
        return DeviceCoo(nrows, ncols, e32, e32.clone(), torch.empty(0, dtype=torch.float64, device=dev))
    sk, sv = sort_pairs(keys, values, key_bits=max(int(nrows) * max(int(ncols), 1) - 1, 0).bit_length(),
                        inplace=owned)
    if not sum_duplicates:
        if n > 1 and bool((sk[1:] == sk[:-1]).any()):
            raise ValueError("entries must be sorted row-major with unique (row, col) pairs")
        nc = max(int(ncols), 1)
        return DeviceCoo(nrows, ncols, (sk // nc).to(torch.int32), (sk % nc).to(torch.int32), sv.contiguous())
    st = stream_handle(dev)
    L = _lib.load()
    nt = int(L.wk_coo_dedup_tiles(n))
    work = torch.empty(nt + 1, dtype=torch.int64, device=dev)
    _lib.call("wk_coo_dedup_count", n, _ptr(sk), _ptr(work), st)
    nu = int(work[nt].item())
    row = torch.empty(nu, dtype=torch.int32, device=dev)
    col = torch.empty(nu, dtype=torch.int32, device=dev)
    val = torch.empty(nu, dtype=torch.float64, device=dev)
    _lib.call("wk_coo_dedup_scatter", n, int(ncols), _ptr(sk), _ptr(sv), _ptr(work), _ptr(row), _ptr(col), _ptr(val),
              st)
    return DeviceCoo(nrows, ncols, row, col, val)
