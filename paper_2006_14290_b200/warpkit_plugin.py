"""Install the B200 backend INTO the reference package's own registry.

warpkit's registry is closed by design (`dispatch.py:7-8`, `SPEC.md:411`):
`EXEC_KINDS` is a module-level tuple (`dispatch.py:18-21`) checked by
`Executor.__post_init__` (`dispatch.py:43-44`) and `make_executor`
(`dispatch.py:66-67`), and each `Operation.impls` is a plain dict
(`dispatch.py:92`). `install(warpkit)` — the binding a warpkit maintainer
would add — therefore:

1. appends "b200" to `warpkit.dispatch.EXEC_KINDS` and to `CLI_EXEC_NAMES`
   (so `make_executor("b200")`, `BenchConfig(execs=("ref", "b200"))` and the
   `bench` CLI accept it);
2. adds a "b200" slot to the existing operations `spmv_coo`, `spmv_csr`,
   `spmv_sellp`, `cg` and `reduce_microbench`, each calling this package.

After that, the reference's own entry points run on the GPU unchanged:
`warpkit.kernels.spmv_sellp(m, x, warpkit.make_executor("b200"))`,
`warpkit.dispatch.dispatch("cg", ex, m, b, tol, max_iters)` and the harness
`warpkit.bench.run_benchmark(...)`, which validates every result against
warpkit's own sequential oracle (`bench.py:209-266`).
"""

import functools

import numpy as np

from .errors import WarpkitError

EXEC_B200 = "b200"


def _warpkit_errors(fn, we):
    """Re-raise this package's exceptions as the same-named warpkit.errors
    class, so `except warpkit.DimensionMismatch` / `BreakdownError` around
    warpkit's own entry points keeps working with the b200 slot installed.
    (ValueError and friends are builtins: shared already.)"""

    @functools.wraps(fn)
    def wrapped(*args, **kwargs):
        try:
            return fn(*args, **kwargs)
        except WarpkitError as exc:
            cls = getattr(we, type(exc).__name__, None)
            if not (isinstance(cls, type) and issubclass(cls, Exception)):
                raise
            if type(exc).__name__ == "NotImplementedForBackend":
                raise cls(exc.op_name, exc.exec_kind) from exc
            raise cls(str(exc)) from exc

    return wrapped


def install(warpkit_module=None, device=None):
    """Register the b200 backend in warpkit; returns the patched dispatch module."""
    if warpkit_module is None:
        import warpkit as warpkit_module  # noqa: F401
    import importlib

    wd = importlib.import_module("warpkit.dispatch")
    wkk = importlib.import_module("warpkit.kernels")
    we = importlib.import_module("warpkit.errors")

    from . import kernels as K
    from . import solvers as S
    from .dispatch import make_executor

    if EXEC_B200 not in wd.EXEC_KINDS:
        wd.EXEC_KINDS = tuple(wd.EXEC_KINDS) + (EXEC_B200,)
    wd.CLI_EXEC_NAMES[EXEC_B200] = EXEC_B200
    ours = make_executor("b200", device=device)

    def _count(exec, m):
        # lane_steps += true nonzeros, as warpkit's own backends (kernels.py:156, 202, 263)
        nnz = int(np.asarray(m.row_lengths).sum()) if hasattr(m, "row_lengths") else len(m.values)
        exec.counters.lane_steps += nnz

    def spmv_coo(exec, m, x):
        _count(exec, m)
        return K._spmv_b200(ours, m, x, "coo")

    def spmv_csr(exec, m, x):
        _count(exec, m)
        return K._spmv_b200(ours, m, x, "csr")

    def spmv_sellp(exec, m, x):
        _count(exec, m)
        return K._spmv_b200(ours, m, x, "sellp")

    def cg(exec, m, b, tol, max_iters):
        return S._run("cg", ours, m, b, tol, max_iters)

    def reduce_microbench(exec, size, inner_loops):
        # the butterfly of `size` lanes reduces ranks 1..size (kernels.py:351-364), on the GPU
        out, _cycles = S.reduce_microbench(size, inner_loops, ours)
        exec.counters.lane_steps += int(inner_loops) * int(size)
        return out

    for name, fn in (("spmv_coo", spmv_coo), ("spmv_csr", spmv_csr), ("spmv_sellp", spmv_sellp), ("cg", cg),
                     ("reduce_microbench", reduce_microbench)):
        try:
            op = wd.get_operation(name)
        except KeyError:
            continue
        op.impls[EXEC_B200] = _warpkit_errors(fn, we)
    assert wkk is not None
    return wd


def make_b200_executor():
    """A warpkit Executor of kind "b200" (config-free, like "reference")."""
    import importlib

    wd = importlib.import_module("warpkit.dispatch")
    if EXEC_B200 not in wd.EXEC_KINDS:
        raise RuntimeError("call install() first")
    return wd.Executor(kind=EXEC_B200)
