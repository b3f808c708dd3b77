"""ctypes binding of libwk_sparse.so (C ABI declared in include/wk_sparse.h).

The library is built in-tree (`make -C paper_2006_14290_b200`, or
`__graft_entry__.build()`); loading fails loudly if it is missing — there
is no CPU fallback anywhere in the package.
"""

import ctypes
import os

from .errors import (BreakdownError, DeviceError, DimensionMismatch, InvalidSliceSize, NativeLibraryMissing,
                     ParseError, UnsupportedFormat)

_HERE = os.path.dirname(os.path.abspath(__file__))
# WK_LIB_PATH: an alternative build of the same library (kernel A/B experiments)
LIB_PATH = os.environ.get("WK_LIB_PATH") or os.path.join(_HERE, "_lib", "libwk_sparse.so")

WK_OK = 0
WK_ERR_INVALID = 1001
WK_ERR_DIMENSION = 1002
WK_ERR_BREAKDOWN = 1003
WK_ERR_SLICE = 1004
WK_ERR_PARSE = 1005
WK_ERR_UNSUPPORTED = 1006

WK_FMT_CSR, WK_FMT_COO, WK_FMT_ELL, WK_FMT_SELLP, WK_FMT_HYBRID = range(5)
WK_CSR_STREAM, WK_CSR_SUBWARP, WK_CSR_ROWBLOCK, WK_CSR_MERGE, WK_CSR_LOAD_BALANCE = 0, 1, 2, 3, 4

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32
F64 = ctypes.c_double
U64 = ctypes.c_uint64


class WkMmHeader(ctypes.Structure):
    """Mirror of `wk_mm_header` (include/wk_sparse.h)."""

    _fields_ = [("nrows", I64), ("ncols", I64), ("nnz", I64), ("field", I32), ("symmetric", I32),
                ("body_offset", I64), ("body_line", I64)]


WK_PEER_MAX = 64


class WkPeerCtx(ctypes.Structure):
    """Mirror of `wk_peer_ctx` (include/wk_sparse.h)."""

    _fields_ = [("rank", I32), ("world", I32), ("arena", P * WK_PEER_MAX), ("seq", P), ("error", P)]


class WkPeerHalo(ctypes.Structure):
    """Mirror of `wk_peer_halo` (include/wk_sparse.h)."""

    _fields_ = [("n", I32), ("peer", I32 * 8), ("lo", I64 * 8), ("hi", I64 * 8), ("dst_off", I64 * 8),
                ("nrecv", I32), ("recv_peer", I32 * 8), ("int_lo", I64), ("int_hi", I64)]


class WkMatrix(ctypes.Structure):
    """Mirror of `wk_matrix` (include/wk_sparse.h)."""

    _fields_ = [
        ("format", I32), ("csr_strategy", I32), ("subwarp_size", I32), ("reserved", I32),
        ("nrows", I64), ("ncols", I64), ("nnz", I64),
        ("row_ptrs", P), ("row_idx", P), ("col_idx", P), ("values", P),
        ("slice_size", I64), ("slice_sets", P),
        ("width", I64), ("stride", I64), ("row_lengths", P),
        ("coo_nnz", I64), ("coo_row", P), ("coo_col", P), ("coo_val", P),
        ("plan", P),
    ]


class WkCgState(ctypes.Structure):
    _fields_ = [("rho", F64), ("pq", F64), ("rr", F64), ("threshold", F64), ("alpha", F64), ("beta", F64),
                ("iteration", I64), ("max_iters", I64), ("done", I32), ("breakdown", I32), ("xpend", I32),
                ("xdefer", I32), ("alpha_prev", F64)]


class WkBicgState(ctypes.Structure):
    _fields_ = [(n, F64) for n in ("rho", "rho_new", "alpha", "omega", "beta", "threshold", "rv", "ss", "tt", "ts",
                                   "rr", "rho_next")] + [("iteration", I64), ("max_iters", I64), ("done", I32),
                                             ("breakdown", I32), ("apply_half", I32), ("pad", I32)]


class WkGmresState(ctypes.Structure):
    _fields_ = [("beta", F64), ("threshold", F64), ("sq", F64), ("hn", F64), ("iteration", I64), ("max_iters", I64),
                ("done", I32), ("cycle_done", I32), ("j_done", I32), ("restart", I32)]


# name -> (restype, argtypes)
_SIGS = {
    "wk_last_error": (ctypes.c_char_p, []),
    "wk_version": (ctypes.c_int, []),
    "wk_device_sm_count": (ctypes.c_int, []),
    "wk_spmv_sellp_f64": (ctypes.c_int, [I64, I64, I64, P, P, P, P, P, P, P]),
    "wk_spmv_ell_f64": (ctypes.c_int, [I64, I64, I64, I64, P, P, P, P, P, P]),
    "wk_spmv_csr_f64": (ctypes.c_int, [I64, I64, I64, P, P, P, P, P, I32, I32, P, P]),
    "wk_csr_plan_chunks": (I64, [I64]),
    "wk_csr_plan_bytes": (I64, [I64]),
    "wk_csr_plan_build": (ctypes.c_int, [I64, I64, P, P, P]),
    "wk_csr_merge_plan_bytes": (I64, [I64, I64]),
    "wk_csr_merge_plan_build": (ctypes.c_int, [I64, I64, P, P, P]),
    "wk_csr_load_balance_plan_bytes": (I64, [I64, I64]),
    "wk_csr_load_balance_plan_build": (ctypes.c_int, [I64, I64, P, P, P]),
    "wk_mm_read_header": (ctypes.c_int, [P, I64, P]),
    "wk_mm_parse_entries": (ctypes.c_int, [P, I64, P, I32, P, P, P, I64, P]),
    "wk_mm_write": (ctypes.c_int, [I64, I64, I64, P, P, P, P, I64, P]),
    "wk_extract_diagonal": (ctypes.c_int, [P, P, P]),
    "wk_pcg_workspace_bytes": (I64, [I64]),
    "wk_pcg_jacobi_solve": (ctypes.c_int, [P, P, P, F64, I64, P, P, P, P, P]),
    "wk_reduce_microbench": (ctypes.c_int, [I32, I32, I32, P, P, P]),
    "wk_sym_alloc": (ctypes.c_int, [I64, P, P]),
    "wk_sym_open": (ctypes.c_int, [P, P]),
    "wk_sym_close": (ctypes.c_int, [P]),
    "wk_sym_free": (ctypes.c_int, [P]),
    "wk_peer_arena_header_bytes": (I64, []),
    "wk_cg_spmv_dot_peer": (ctypes.c_int, [P, P, P, P, P, P, P, P]),
    "wk_cg_update_xr_alpha_peer": (ctypes.c_int, [I64, P, P, P, P, P, P, P, P]),
    "wk_cg_replace_r_peer": (ctypes.c_int, [I64, P, P, P, P, P, P, P]),
    "wk_cg_update_p_beta_peer": (ctypes.c_int, [I64, P, P, P, P, P, P, P, P, P]),
    "wk_peer_allreduce": (ctypes.c_int, [P, P, P, I32, P]),
    "wk_peer_exchange": (ctypes.c_int, [P, P, I32, P, P, P, P, I32, P, P, P]),
    "wk_spmv_coo_f64": (ctypes.c_int, [I64, I64, I64, P, P, P, P, P, I32, P]),
    "wk_spmv_hybrid_f64": (ctypes.c_int, [I64, I64, I64, I64, P, P, P, I64, P, P, P, P, P, P]),
    "wk_spmv": (ctypes.c_int, [P, P, P, P]),
    "wk_spmv_masked": (ctypes.c_int, [P, P, P, P, P]),
    "wk_reduce_workspace_bytes": (I64, []),
    "wk_dot_f64": (ctypes.c_int, [I64, P, P, P, P, P]),
    "wk_norm2_f64": (ctypes.c_int, [I64, P, P, P, P]),
    "wk_axpy_f64": (ctypes.c_int, [I64, F64, P, P, P]),
    "wk_xpby_f64": (ctypes.c_int, [I64, P, F64, P, P]),
    "wk_scal_f64": (ctypes.c_int, [I64, F64, P, P]),
    "wk_multidot_f64": (ctypes.c_int, [I64, I64, P, I64, P, P, P, P]),
    "wk_gather_f64": (ctypes.c_int, [I64, P, P, P, P]),
    "wk_csr_row_lengths": (ctypes.c_int, [I64, P, P, P]),
    "wk_csr_max_row_length": (ctypes.c_int, [I64, P, P, P]),
    "wk_csr_row_length_histogram": (ctypes.c_int, [I64, P, I64, P, P]),
    "wk_csr_to_sellp_sets": (ctypes.c_int, [I64, I64, P, P, P, P, P]),
    "wk_csr_to_sellp_fill": (ctypes.c_int, [I64, I64, P, P, P, P, P, P, P]),
    "wk_csr_to_ell_fill": (ctypes.c_int, [I64, I64, I64, P, P, P, P, P, P, P]),
    "wk_hybrid_coo_offsets": (ctypes.c_int, [I64, I64, P, P, P, P]),
    "wk_sellp_zero_padding": (ctypes.c_int, [I64, I64, P, P, P, P, P]),
    "wk_ell_zero_padding": (ctypes.c_int, [I64, I64, I64, P, P, P, P]),
    "wk_hybrid_coo_fill": (ctypes.c_int, [I64, I64, P, P, P, P, P, P, P, P, I64, P]),
    "wk_hybrid_coo_fill_workspace": (ctypes.c_int64, [I64]),
    "wk_sort_pairs_workspace": (ctypes.c_int64, [I64]),
    "wk_sort_pairs_u64_f64": (ctypes.c_int, [I64, I32, P, P, P, P, P, I64, P]),
    "wk_coo_to_csr_ptrs": (ctypes.c_int, [I64, I64, P, P, P]),
    "wk_csr_to_coo_rows": (ctypes.c_int, [I64, P, P, P]),
    "wk_scan_workspace_bytes": (I64, [I64]),
    "wk_exclusive_scan_i64": (ctypes.c_int, [I64, P, P, P, P]),
    "wk_gen_stencil_csr": (ctypes.c_int, [I64, I64, I64, I32, P, P, P, P, P, P, P, P, P]),
    "wk_gen_rmat_edges": (ctypes.c_int, [I32, I32, F64, F64, F64, U64, I64, I64, P, P, P]),
    "wk_coo_dedup_tiles": (ctypes.c_int64, [I64]),
    "wk_coo_dedup_workspace": (ctypes.c_int64, [I64]),
    "wk_coo_dedup_count": (ctypes.c_int, [I64, P, P, P]),
    "wk_coo_dedup_scatter": (ctypes.c_int, [I64, I64, P, P, P, P, P, P, P]),
    "wk_cg_workspace_bytes": (I64, [I64]),
    "wk_cg_solve": (ctypes.c_int, [P, P, F64, I64, P, P, P, P, P]),
    "wk_bicgstab_workspace_bytes": (I64, [I64]),
    "wk_bicgstab_solve": (ctypes.c_int, [P, P, F64, I64, P, P, P, P, P]),
    "wk_gmres_workspace_bytes": (I64, [I64, I32]),
    "wk_gmres_solve": (ctypes.c_int, [P, P, F64, I64, I32, P, P, P, P, P]),
    "wk_cg_init_local": (ctypes.c_int, [I64, P, P, P, P, P, P, P]),
    "wk_cg_init_finish": (ctypes.c_int, [P, F64, I64, P, P]),
    "wk_cg_dot_pq": (ctypes.c_int, [I64, P, P, P, P, P]),
    "wk_cg_spmv_dot": (ctypes.c_int, [P, P, P, P, P, P]),
    "wk_cg_step_alpha": (ctypes.c_int, [P, P]),
    "wk_cg_update_xr": (ctypes.c_int, [I64, P, P, P, P, P, P, P]),
    "wk_cg_replace_r": (ctypes.c_int, [I64, P, P, P, P, P, P]),
    "wk_cg_step_beta": (ctypes.c_int, [P, P, P]),
    "wk_cg_update_xr_alpha": (ctypes.c_int, [I64, P, P, P, P, P, P, P]),
    "wk_cg_update_p_beta": (ctypes.c_int, [I64, P, P, P, P, P, P, P]),
    "wk_cg_update_p": (ctypes.c_int, [I64, P, P, P, P]),
    "wk_bicg_init": (ctypes.c_int, [I64, P, P, P, P, P, P, P, P, P]),
    "wk_bicg_init_finish": (ctypes.c_int, [P, F64, I64, P, P]),
    "wk_bicg_rho": (ctypes.c_int, [I64, P, P, P, P, P]),
    "wk_bicg_step_beta": (ctypes.c_int, [P, P]),
    "wk_bicg_update_p": (ctypes.c_int, [I64, P, P, P, P, P]),
    "wk_bicg_rv": (ctypes.c_int, [I64, P, P, P, P, P]),
    "wk_bicg_step_alpha": (ctypes.c_int, [P, P]),
    "wk_bicg_update_s": (ctypes.c_int, [I64, P, P, P, P, P, P]),
    "wk_bicg_step_s": (ctypes.c_int, [P, P, P]),
    "wk_bicg_half_x": (ctypes.c_int, [I64, P, P, P, P, P]),
    "wk_bicg_tt_ts": (ctypes.c_int, [I64, P, P, P, P, P]),
    "wk_bicg_step_omega": (ctypes.c_int, [P, P]),
    "wk_bicg_update_xr": (ctypes.c_int, [I64, P, P, P, P, P, P, P, P]),
    "wk_bicg_step_r": (ctypes.c_int, [P, P, P]),
    "wk_bicg_spmv_dots": (ctypes.c_int, [P, P, P, P, P, I32, P, P]),
    "wk_bicg_rho_first": (ctypes.c_int, [I64, P, P, P, P, P]),
    "wk_bicg_take_rho": (ctypes.c_int, [P, P]),
    "wk_bicg_update_xr_rho": (ctypes.c_int, [I64, P, P, P, P, P, P, P, P, P]),
    "wk_gmres_init": (ctypes.c_int, [I64, P, P, P, P, P, P]),
    "wk_gmres_init_finish": (ctypes.c_int, [P, F64, I64, I32, P, P]),
    "wk_gmres_cycle_start": (ctypes.c_int, [I64, P, P, P, P, P]),
    "wk_gmres_multidot": (ctypes.c_int, [I64, I32, P, I64, P, P, P, P, P]),
    "wk_gmres_orth": (ctypes.c_int, [I64, I32, P, I64, P, P, P, P, P]),
    "wk_gmres_givens": (ctypes.c_int, [I32, P, P, P, P, P, P, P]),
    "wk_gmres_next_basis": (ctypes.c_int, [I64, P, P, P, P]),
    "wk_gmres_update_x": (ctypes.c_int, [I64, P, I64, P, P, P, P, P, P]),
    "wk_gmres_orth_scaled": (ctypes.c_int, [I64, I32, P, I64, P, P, P, P, P, P]),
    "wk_gmres_givens_scaled": (ctypes.c_int, [I32, P, P, P, P, P, P, P, P]),
    "wk_gmres_update_x_scaled": (ctypes.c_int, [I64, P, I64, P, P, P, P, P, P, P]),
    "wk_gmres_residual": (ctypes.c_int, [I64, P, P, P, P, P, P]),
    "wk_gmres_restart": (ctypes.c_int, [P, P, P]),
}

EXPORTED = tuple(sorted(_SIGS))

_lib = None


def load():
    """Load (once) and return the ctypes library handle."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryMissing(
            f"{LIB_PATH} not found; build it with `make -C {_HERE}` or __graft_entry__.build() — "
            "this package has no CPU fallback")
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as exc:
        raise NativeLibraryMissing(f"cannot load {LIB_PATH}: {exc}") from exc
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().wk_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = ""):
    """Map a libwk_sparse status to the reference's exception types."""
    if rc == WK_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc == WK_ERR_BREAKDOWN:
        raise BreakdownError(msg)
    if rc == WK_ERR_DIMENSION:
        raise DimensionMismatch(msg)
    if rc == WK_ERR_SLICE:
        raise InvalidSliceSize(msg)
    if rc == WK_ERR_INVALID:
        raise ValueError(msg)
    if rc == WK_ERR_PARSE:
        raise ParseError(msg)
    if rc == WK_ERR_UNSUPPORTED:
        raise UnsupportedFormat(msg)
    raise DeviceError(rc, msg)


def call(name: str, *args):
    """Invoke `name` and raise on a non-zero status."""
    rc = getattr(load(), name)(*args)
    check(rc, name)
    return rc
