"""B200-native sparse fp64 hot path (SpMV / BLAS-1 / Krylov / conversions).

Drop-in for the hot path of the reference package `warpkit`
(arXiv 2006.14290 workbench): the same matrix classes and operation
signatures (`spmv_coo/csr/sellp(m, x, exec)`, `cg_solve(m, b, tol,
max_iters, exec)`, `coo_to_csr`, `coo_to_sellp`, executor registry), backed by
hand-written sm_100a CUDA kernels in `_lib/libwk_sparse.so` (C ABI:
`include/wk_sparse.h`). Extended with ELL/Hybrid, load-balanced CSR, dot /
norm2 / axpy, BiCGSTAB, GMRES(m), stopping criteria and row-block
partitioned multi-GPU operators (`distributed`).
"""

from .config import B200Config
from .dispatch import (
    EXEC_B200,
    EXEC_REFERENCE,
    Executor,
    Instrumentation,
    Operation,
    dispatch,
    get_operation,
    instrumentation_report,
    make_executor,
    register,
    registered_operations,
)
from .errors import (
    BreakdownError,
    DeviceError,
    DimensionMismatch,
    InvalidSliceSize,
    NativeLibraryMissing,
    NotImplementedForBackend,
    ParseError,
    UnsupportedFormat,
    WarpkitError,
)
from .sparse import CooMatrix, CsrMatrix, EllMatrix, HybridMatrix, SellpMatrix
from .kernels import (
    axpy,
    coo_to_csr,
    coo_to_sellp,
    csr_to_coo,
    csr_to_ell,
    csr_to_hybrid,
    csr_to_sellp,
    dot,
    norm2,
    spmv,
    spmv_coo,
    spmv_csr,
    spmv_ell,
    spmv_hybrid,
    spmv_sellp,
)
from .pipeline import SpmvPipeline
from .device import release
from .mmio import read_matrix_market, read_matrix_market_entries, write_matrix_market
from .solvers import (Bicgstab, Cg, Gmres, Iteration, Jacobi, ResidualNorm, bicgstab_solve, cg_solve, diagonal,
                      gmres_solve, pcg_solve, reduce_microbench)

__version__ = "0.1.0"

__all__ = [
    "B200Config", "EXEC_B200", "EXEC_REFERENCE", "Executor", "Instrumentation", "Operation", "dispatch",
    "get_operation", "instrumentation_report", "make_executor", "register", "registered_operations",
    "BreakdownError", "DeviceError", "DimensionMismatch", "InvalidSliceSize", "NativeLibraryMissing",
    "NotImplementedForBackend", "ParseError", "UnsupportedFormat", "WarpkitError",
    "CooMatrix", "CsrMatrix", "EllMatrix", "HybridMatrix", "SellpMatrix",
    "axpy", "coo_to_csr", "coo_to_sellp", "csr_to_coo", "csr_to_ell", "csr_to_hybrid", "csr_to_sellp", "dot",
    "norm2", "spmv", "spmv_coo", "spmv_csr", "spmv_ell", "spmv_hybrid", "spmv_sellp",
    "read_matrix_market", "read_matrix_market_entries", "write_matrix_market", "SpmvPipeline",
    "Bicgstab", "Cg", "Gmres", "Iteration", "Jacobi", "ResidualNorm", "bicgstab_solve", "cg_solve", "diagonal",
    "gmres_solve", "pcg_solve", "reduce_microbench", "release",
]
