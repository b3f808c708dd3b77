"""Krylov solvers on the B200: CG (the reference's `cg_solve`,
kernels.py:283-331), BiCGSTAB and GMRES(m) (no reference), each with the
reference's call shape `solver(m, b, tol, max_iters, exec)` and a
Ginkgo-style factory API: `Cg(criteria).generate(A).apply(b)` with stopping
criteria objects.

The whole iteration loop runs on the device (`wk_cg_solve`,
`wk_bicgstab_solve`, `wk_gmres_solve`): scalars never leave HBM, a CUDA
graph of 50 CG iterations (one residual-replacement period) is replayed until
the device-side convergence flag is set, and the host only reads the flag
between replays.
"""

import ctypes
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from . import device as D
from .dispatch import EXEC_B200, Executor, dispatch, make_executor, op_impl, register
from .errors import DimensionMismatch


def _check(m, b, tol):
    """Argument checks in the reference's order (kernels.py:292-298)."""
    if m.nrows != m.ncols:
        raise DimensionMismatch(f"CG needs a square matrix, got {m.nrows}x{m.ncols}")
    if isinstance(b, torch.Tensor):
        if b.dim() != 1 or b.numel() != m.nrows:
            raise DimensionMismatch(f"b has shape {tuple(b.shape)}, matrix is {m.nrows}x{m.ncols}")
    else:
        b = np.asarray(b, dtype=np.float64)
        if b.ndim != 1 or len(b) != m.nrows:
            raise DimensionMismatch(f"b has length {len(b)}, matrix is {m.nrows}x{m.ncols}")
    if tol <= 0:
        raise ValueError("tol must be positive")


def diagonal(m, exec: Executor = None):
    """Main diagonal of a matrix as a device vector (wk_extract_diagonal;
    missing entries are 0.0)."""
    from .kernels import _prepare

    d = _prepare(exec if exec is not None else make_executor("b200"), m)
    n = min(d.nrows, d.ncols)
    out = torch.empty(n, dtype=torch.float64, device=d.device)
    _lib.call("wk_extract_diagonal", d.wk_ptr(), D._ptr(out), D.stream_handle(d.device))
    return out


def _run(kind, exec: Executor, m, b, tol, max_iters, restart=30, diag=None):
    _check(m, b, tol)
    from .kernels import _prepare

    d = _prepare(exec, m)
    bt, host = D.as_device_vector(b, d.nrows, d.device, "b")
    n = d.nrows
    max_iters = int(max_iters)
    x = torch.empty(n, dtype=torch.float64, device=d.device)
    hist = torch.zeros(max(max_iters, 0) + 1, dtype=torch.float64, device=d.device)
    iters = ctypes.c_int64(0)
    L = _lib.load()
    st = D.stream_handle(d.device)
    if kind == "cg":
        ws = torch.empty(int(L.wk_cg_workspace_bytes(n)), dtype=torch.uint8, device=d.device)
        rc = L.wk_cg_solve(d.wk_ptr(), D._ptr(bt), float(tol), max_iters, D._ptr(x), D._ptr(hist),
                           ctypes.byref(iters), D._ptr(ws), st)
    elif kind == "pcg":
        dg = diag if diag is not None else diagonal(d, exec)
        dg, _ = D.as_device_vector(dg, n, d.device, "diag")
        ws = torch.empty(int(L.wk_pcg_workspace_bytes(n)), dtype=torch.uint8, device=d.device)
        rc = L.wk_pcg_jacobi_solve(d.wk_ptr(), D._ptr(dg), D._ptr(bt), float(tol), max_iters, D._ptr(x),
                                   D._ptr(hist), ctypes.byref(iters), D._ptr(ws), st)
    elif kind == "bicgstab":
        ws = torch.empty(int(L.wk_bicgstab_workspace_bytes(n)), dtype=torch.uint8, device=d.device)
        rc = L.wk_bicgstab_solve(d.wk_ptr(), D._ptr(bt), float(tol), max_iters, D._ptr(x), D._ptr(hist),
                                 ctypes.byref(iters), D._ptr(ws), st)
    else:
        ws = torch.empty(int(L.wk_gmres_workspace_bytes(n, int(restart))), dtype=torch.uint8, device=d.device)
        rc = L.wk_gmres_solve(d.wk_ptr(), D._ptr(bt), float(tol), max_iters, int(restart), D._ptr(x),
                              D._ptr(hist), ctypes.byref(iters), D._ptr(ws), st)
    _lib.check(rc, f"{kind}_solve")
    it = int(iters.value)
    hist = hist[: it + 1]
    exec.counters.lane_steps += int(d.nnz) * it
    return D.to_host_like(x, host), D.to_host_like(hist, host)


def _cg_b200(exec, m, b, tol, max_iters):
    return _run("cg", exec, m, b, tol, max_iters)


def _pcg_b200(exec, m, b, tol, max_iters, diag=None):
    return _run("pcg", exec, m, b, tol, max_iters, diag=diag)


def _bicgstab_b200(exec, m, b, tol, max_iters):
    return _run("bicgstab", exec, m, b, tol, max_iters)


def _gmres_b200(exec, m, b, tol, max_iters, restart=30):
    return _run("gmres", exec, m, b, tol, max_iters, restart)


register("cg", {EXEC_B200: _cg_b200})
register("pcg", {EXEC_B200: _pcg_b200})
register("bicgstab", {EXEC_B200: _bicgstab_b200})
register("gmres", {EXEC_B200: _gmres_b200})


def cg_solve(m, b, tol: float, max_iters: int, exec: Executor):
    """Unpreconditioned CG (kernels.py:283-331). Returns (x, residual_history)
    with len(history) == iterations + 1. Like the reference it does not reset
    the executor's counters (it bypasses dispatch, kernels.py:299)."""
    return op_impl("cg", exec)(exec, m, b, tol, max_iters)


def pcg_solve(m, b, tol: float, max_iters: int, exec: Executor, diag=None):
    """Jacobi-preconditioned CG: the reference CG loop (kernels.py:283-331)
    with z = r / diag (the apply_jacobi fixture, preconditioner.cu:9-17);
    `diag` defaults to the matrix's main diagonal. Returns (x, ||r|| history)."""
    return op_impl("pcg", exec)(exec, m, b, tol, max_iters, diag)


def bicgstab_solve(m, b, tol: float, max_iters: int, exec: Executor):
    return op_impl("bicgstab", exec)(exec, m, b, tol, max_iters)


def gmres_solve(m, b, tol: float, max_iters: int, exec: Executor, restart: int = 30):
    return op_impl("gmres", exec)(exec, m, b, tol, max_iters, restart)


# ---- Ginkgo-style factories with stopping criteria ------------------------------------


@dataclass(frozen=True)
class Iteration:
    """Stop after `max_iters` iterations (gko::stop::Iteration)."""

    max_iters: int


@dataclass(frozen=True)
class ResidualNorm:
    """Stop when ||r|| <= reduction_factor * baseline (gko::stop::ResidualNorm).

    baseline "rhs_norm" (the reference's criterion, kernels.py:313) and
    "initial_resnorm" coincide for the zero initial guess; "absolute" uses
    reduction_factor as the threshold itself.
    """

    reduction_factor: float
    baseline: str = "rhs_norm"

    def __post_init__(self):
        if self.baseline not in ("rhs_norm", "initial_resnorm", "absolute"):
            raise ValueError(f"unknown baseline {self.baseline!r}")
        if self.reduction_factor <= 0:
            raise ValueError("reduction_factor must be positive")


def _criteria_to_params(criteria: Sequence, b, exec):
    max_iters = None
    tol = None
    for c in criteria:
        if isinstance(c, Iteration):
            max_iters = c.max_iters if max_iters is None else min(max_iters, c.max_iters)
        elif isinstance(c, ResidualNorm):
            if c.baseline == "absolute":
                bn = dispatch("norm2", exec, b)
                t = c.reduction_factor / bn if bn > 0 else c.reduction_factor
            else:
                t = c.reduction_factor
            tol = t if tol is None else max(tol, t)
        else:
            raise TypeError(f"unsupported stopping criterion {c!r}")
    if max_iters is None and tol is None:
        raise ValueError("at least one stopping criterion is required")
    return (tol if tol is not None else 1e-300), (max_iters if max_iters is not None else 2**62)


@dataclass
class _Solver:
    kind: str
    A: object
    criteria: tuple
    exec: Executor
    restart: int = 30
    preconditioner: Optional[object] = None
    iterations: int = 0
    residual_history: Optional[object] = None
    _diag: Optional[object] = None

    def apply(self, b, x=None):
        """Solve A x = b from the zero initial guess; returns x (and fills
        `iterations`, `residual_history`)."""
        if x is not None:
            xz = x if isinstance(x, torch.Tensor) else np.asarray(x)
            if bool((xz != 0).any()):
                raise NotImplementedError("only the zero initial guess is supported (as in the reference)")
        tol, max_iters = _criteria_to_params(self.criteria, b, self.exec)
        if self.kind == "gmres":
            sol, hist = _gmres_b200(self.exec, self.A, b, tol, max_iters, self.restart)
        elif self.kind == "cg" and self.preconditioner is not None:
            if self._diag is None:
                self._diag = self.preconditioner.generate(self.A, self.exec)
            sol, hist = _run("pcg", self.exec, self.A, b, tol, max_iters, diag=self._diag)
        else:
            sol, hist = _run(self.kind, self.exec, self.A, b, tol, max_iters)
        self.iterations = len(hist) - 1
        self.residual_history = hist
        if x is not None:
            if isinstance(x, torch.Tensor):
                x.copy_(sol if isinstance(sol, torch.Tensor) else torch.from_numpy(sol))
            else:
                x[...] = sol if isinstance(sol, np.ndarray) else sol.cpu().numpy()
            return x
        return sol


@dataclass
class _Factory:
    kind: str
    criteria: tuple = field(default_factory=tuple)
    exec: Optional[Executor] = None
    restart: int = 30
    preconditioner: Optional[object] = None

    def generate(self, A) -> _Solver:
        ex = self.exec if self.exec is not None else make_executor("b200")
        from .kernels import _prepare

        d = _prepare(ex, A)  # upload once, at generate time (Ginkgo semantics)
        if d.nrows != d.ncols:
            raise DimensionMismatch(f"solver needs a square matrix, got {d.nrows}x{d.ncols}")
        return _Solver(self.kind, d, tuple(self.criteria), ex, self.restart, self.preconditioner)


@dataclass(frozen=True)
class Jacobi:
    """Scalar Jacobi preconditioner M = diag(A) (gko::preconditioner::Jacobi
    with block size 1; apply z = r / diag as the fixture's apply_jacobi)."""

    def generate(self, A, exec=None):
        return diagonal(A, exec)


def Cg(criteria=(), exec=None, preconditioner=None) -> _Factory:
    """CG factory; preconditioner=Jacobi() gives the preconditioned solver."""
    if preconditioner is not None and not isinstance(preconditioner, Jacobi):
        raise TypeError(f"unsupported preconditioner {preconditioner!r}")
    return _Factory("cg", tuple(criteria), exec, preconditioner=preconditioner)


def Bicgstab(criteria=(), exec=None) -> _Factory:
    return _Factory("bicgstab", tuple(criteria), exec)


def Gmres(criteria=(), exec=None, restart=30) -> _Factory:
    return _Factory("gmres", tuple(criteria), exec, restart)


def reduce_microbench(size: int, inner_loops: int, exec: Executor = None, shared_memory: bool = False):
    """The reference's reduction microbenchmark (kernels.py:341-364) on the
    GPU: one warp, tiles of `size` lanes butterfly-reduce (rank + 1)
    `inner_loops` times (coop groups, or the legacy shared-memory tree with
    shared_memory=True). Returns (per-lane results of the first tile
    (length size), device clock cycles of the loop)."""
    ex = exec if exec is not None else make_executor("b200")
    dev = ex.torch_device()
    out = torch.empty(32, dtype=torch.float64, device=dev)
    cyc = torch.zeros(1, dtype=torch.int64, device=dev)
    _lib.call("wk_reduce_microbench", int(size), int(inner_loops), int(bool(shared_memory)), D._ptr(out), D._ptr(cyc),
              D.stream_handle(dev))
    ex.counters.launches += 1
    return out[: int(size)].cpu().numpy(), int(cyc.item())
