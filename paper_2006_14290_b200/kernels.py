"""Operations of the drop-in API, registered per backend.

Public wrappers keep the reference's signatures (`kernels.py:409-418`):
`spmv_coo/csr/sellp(m, x, exec)`, plus `spmv_ell`, `spmv_hybrid`, `spmv`
(format-generic), BLAS-1 `dot`, `norm2`, `axpy`, and the conversions.
Inputs may be host matrices (this package's, or warpkit's own dataclasses),
or device twins (`device.py`). Host x in -> host numpy y out (the reference's
contract: impls return new arrays, `kernels.py:150`); torch x on the device
-> torch y on the device, with no host round trip.
"""

import numpy as np
import torch

from . import _lib
from . import device as D
from .dispatch import EXEC_B200, Executor, dispatch, register

_FMT_OF_OP = {"spmv_coo": "coo", "spmv_csr": "csr", "spmv_sellp": "sellp", "spmv_ell": "ell", "spmv_hybrid": "hybrid"}


def _prepare(exec: Executor, m, fmt=None):
    d = D.as_device(m, exec.device)
    if fmt is not None and d.fmt != fmt:
        raise TypeError(f"expected a {fmt} matrix, got {d.fmt}")
    if d.fmt == "csr":
        t = exec.tuning
        d.with_strategy(t["csr_strategy"], t["csr_subwarp_size"])
    return d


def spmv_device(d, x, y=None, stream=None):
    """y = A x for a device matrix and device vectors (no checks, no sync)."""
    if y is None:
        y = torch.empty(d.nrows, dtype=torch.float64, device=d.device)
    st = stream if stream is not None else D.stream_handle(d.device)
    _lib.call("wk_spmv", d.wk_ptr(), D._ptr(x), D._ptr(y), st)
    return y


def _launches(d):
    """Kernels one SpMV enqueues: COO zero-fill + seg8, Hybrid ELL + COO
    part, CSR load_balance zero-fill + seg8 + range fix-up, merge tiles +
    fix-up; one otherwise."""
    if d.fmt == "csr":
        return {_lib.WK_CSR_LOAD_BALANCE: 3, _lib.WK_CSR_MERGE: 2}.get(d.strategy, 1)
    return {"coo": 2, "hybrid": 2}.get(d.fmt, 1)


def _spmv_b200(exec: Executor, m, x, fmt=None):
    D.check_vector(x, m.ncols)
    d = _prepare(exec, m, fmt)
    xt, host = D.as_device_vector(x, d.ncols, d.device)
    y = spmv_device(d, xt)
    exec.counters.lane_steps += int(d.nnz)
    exec.counters.launches += _launches(d)
    return D.to_host_like(y, host)


def _spmv_op(fmt):
    def impl(exec, m, x):
        return _spmv_b200(exec, m, x, fmt)

    impl.__name__ = f"_spmv_{fmt}_b200"
    return impl


def _spmv_any(exec, m, x):
    return _spmv_b200(exec, m, x, None)


# ---- BLAS-1 -----------------------------------------------------------------------


def _vec_pair(exec, x, y):
    dev = exec.torch_device()
    n = x.numel() if isinstance(x, torch.Tensor) else len(np.asarray(x))
    xt, hx = D.as_device_vector(x, n, dev, "x")
    yt, hy = D.as_device_vector(y, n, dev, "y")
    return xt, yt, hx or hy


def _dot_b200(exec, x, y):
    xt, yt, _ = _vec_pair(exec, x, y)
    ws = D.workspace(xt.device)
    res = torch.empty(1, dtype=torch.float64, device=xt.device)
    _lib.call("wk_dot_f64", xt.numel(), D._ptr(xt), D._ptr(yt), D._ptr(res), D._ptr(ws.red), D.stream_handle(xt.device))
    exec.counters.launches += 1
    exec.counters.lane_steps += xt.numel()
    return float(res.item())


def _norm2_b200(exec, x):
    dev = exec.torch_device()
    n = x.numel() if isinstance(x, torch.Tensor) else len(np.asarray(x))
    xt, _ = D.as_device_vector(x, n, dev, "x")
    ws = D.workspace(xt.device)
    res = torch.empty(1, dtype=torch.float64, device=xt.device)
    _lib.call("wk_norm2_f64", n, D._ptr(xt), D._ptr(res), D._ptr(ws.red), D.stream_handle(xt.device))
    exec.counters.launches += 1
    exec.counters.lane_steps += n
    return float(res.item())


def _axpy_b200(exec, alpha, x, y):
    """y + alpha * x; returns a new array for host inputs (reference style),
    updates y in place for device tensors."""
    if isinstance(y, torch.Tensor):
        xt, _ = D.as_device_vector(x, y.numel(), y.device, "x")
        _lib.call("wk_axpy_f64", y.numel(), float(alpha), D._ptr(xt), D._ptr(y), D.stream_handle(y.device))
        exec.counters.launches += 1
        return y
    xt, yt, _ = _vec_pair(exec, x, y)
    yt = yt.clone()
    _lib.call("wk_axpy_f64", yt.numel(), float(alpha), D._ptr(xt), D._ptr(yt), D.stream_handle(yt.device))
    exec.counters.launches += 1
    return yt.cpu().numpy()


# ---- conversions --------------------------------------------------------------------


def _convert(exec, fn, m, *args, **kwargs):
    d = D.as_device(m, exec.device)
    out = fn(d, *args, **kwargs)
    exec.counters.launches += 2
    return out if isinstance(m, D.DeviceMatrix) else out.to_host()


def _coo_to_csr_b200(exec, m):
    return _convert(exec, D.coo_to_csr, m)


def _coo_to_sellp_b200(exec, m, slice_size=64):
    D._check_slice(slice_size)
    d = D.coo_to_csr(D.as_device(m, exec.device))
    out = D.csr_to_sellp(d, slice_size)
    return out if isinstance(m, D.DeviceMatrix) else out.to_host()


def _csr_to_sellp_b200(exec, m, slice_size=64):
    return _convert(exec, D.csr_to_sellp, m, slice_size)


def _csr_to_ell_b200(exec, m, width=None, stride=None):
    return _convert(exec, D.csr_to_ell, m, width, stride)


def _csr_to_hybrid_b200(exec, m, width=None, strategy=None, percent=None):
    t = exec.tuning
    return _convert(exec, D.csr_to_hybrid, m, width, strategy or t["hybrid_strategy"],
                    t["hybrid_percent"] if percent is None else percent)


def _csr_to_coo_b200(exec, m):
    return _convert(exec, D.csr_to_coo, m)


for _name, _fmt in _FMT_OF_OP.items():
    register(_name, {EXEC_B200: _spmv_op(_fmt)})
register("spmv", {EXEC_B200: _spmv_any})
register("dot", {EXEC_B200: _dot_b200})
register("norm2", {EXEC_B200: _norm2_b200})
register("axpy", {EXEC_B200: _axpy_b200})
register("coo_to_csr", {EXEC_B200: _coo_to_csr_b200})
register("coo_to_sellp", {EXEC_B200: _coo_to_sellp_b200})
register("csr_to_sellp", {EXEC_B200: _csr_to_sellp_b200})
register("csr_to_ell", {EXEC_B200: _csr_to_ell_b200})
register("csr_to_hybrid", {EXEC_B200: _csr_to_hybrid_b200})
register("csr_to_coo", {EXEC_B200: _csr_to_coo_b200})


def _default_exec(exec):
    if exec is None:
        from .dispatch import make_executor

        return make_executor("b200")
    return exec


def spmv_coo(m, x, exec: Executor):
    return dispatch("spmv_coo", exec, m, x)


def spmv_csr(m, x, exec: Executor):
    return dispatch("spmv_csr", exec, m, x)


def spmv_sellp(m, x, exec: Executor):
    return dispatch("spmv_sellp", exec, m, x)


def spmv_ell(m, x, exec: Executor):
    return dispatch("spmv_ell", exec, m, x)


def spmv_hybrid(m, x, exec: Executor):
    return dispatch("spmv_hybrid", exec, m, x)


def spmv(m, x, exec: Executor = None):
    return dispatch("spmv", _default_exec(exec), m, x)


def dot(x, y, exec: Executor = None) -> float:
    return dispatch("dot", _default_exec(exec), x, y)


def norm2(x, exec: Executor = None) -> float:
    return dispatch("norm2", _default_exec(exec), x)


def axpy(alpha, x, y, exec: Executor = None):
    return dispatch("axpy", _default_exec(exec), alpha, x, y)


def coo_to_csr(m, exec: Executor = None):
    """sparse.py:212-216 on the device."""
    return dispatch("coo_to_csr", _default_exec(exec), m)


def coo_to_sellp(m, slice_size: int = 64, exec: Executor = None):
    """sparse.py:219-242 on the device."""
    return dispatch("coo_to_sellp", _default_exec(exec), m, slice_size)


def csr_to_sellp(m, slice_size: int = 64, exec: Executor = None):
    return dispatch("csr_to_sellp", _default_exec(exec), m, slice_size)


def csr_to_ell(m, width=None, stride=None, exec: Executor = None):
    return dispatch("csr_to_ell", _default_exec(exec), m, width, stride)


def csr_to_hybrid(m, width=None, strategy=None, exec: Executor = None):
    return dispatch("csr_to_hybrid", _default_exec(exec), m, width, strategy)


def csr_to_coo(m, exec: Executor = None):
    return dispatch("csr_to_coo", _default_exec(exec), m)
