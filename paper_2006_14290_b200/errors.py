"""Exception contract of the drop-in boundary.

Mirrors `warpkit/errors.py:4-78` name for name so code written against the
reference catches the same types. C status codes from libwk_sparse
(`include/wk_sparse.h`) map onto them in `_lib.check`.
"""


class WarpkitError(Exception):
    """Base class (errors.py:4-5)."""


class DimensionMismatch(WarpkitError):
    """Operand shapes are incompatible (errors.py:47-48)."""


class InvalidSliceSize(WarpkitError):
    """SELL-P slice size must be a positive power of two (errors.py:51-52)."""


class BreakdownError(WarpkitError):
    """Krylov breakdown: CG p.Ap <= 0 (errors.py:55-56); BiCGSTAB rho == 0,
    r^.v == 0 or t.t == 0."""


class NotImplementedForBackend(WarpkitError):
    """The operation has no implementation registered for this executor
    (errors.py:59-66)."""

    def __init__(self, op_name, exec_kind):
        self.op_name = op_name
        self.exec_kind = exec_kind
        super().__init__(f"operation {op_name!r} is not implemented for backend {exec_kind!r}")


class ParseError(WarpkitError):
    """Malformed MatrixMarket header or entry (errors.py:69-70)."""


class UnsupportedFormat(WarpkitError):
    """MatrixMarket variant outside the supported subset (errors.py:73-74)."""


class DeviceError(WarpkitError):
    """A CUDA call inside libwk_sparse failed (no reference counterpart: the
    reference never touches a device)."""

    def __init__(self, code, message):
        self.code = code
        super().__init__(f"libwk_sparse error {code}: {message}")


class NativeLibraryMissing(WarpkitError):
    """libwk_sparse.so is not built or cannot be loaded. There is no CPU
    fallback: build it with `python -c 'import __graft_entry__ as g; g.build()'`."""
