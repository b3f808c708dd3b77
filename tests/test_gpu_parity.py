"""Parity of the CUDA path (through the C ABI) against the CPU oracle and the
reference's golden vectors. Bars:
  * SELL-P, ELL, CSR-stream / -rowblock SpMV and every conversion: bitwise;
  * CSR-subwarp, CSR-merge, COO, Hybrid SpMV: max_scaled_rel_err <= 1e-12
    (integer-valued data: exact);
  * CG: equal iteration count, max |res_k - res_ref_k| / ||b|| <= 1e-10,
    max_scaled_rel_err(x) <= 1e-10.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import corpus_ref, krylov_ref, sparse_ref  # noqa: E402
from tests import golden_io  # noqa: E402

SPMV = golden_io.spmv_cases()
CG = golden_io.cg_cases()
TOL = 1e-12


@pytest.fixture(scope="module")
def wk():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2006_14290_b200 as wk

    return wk


@pytest.fixture
def ex(wk):
    return wk.make_executor("b200", device=0)


def _host(wk, ns, kind):
    if kind == "coo":
        return wk.CooMatrix(ns.nrows, ns.ncols, ns.row_idx, ns.col_idx, ns.values)
    if kind == "csr":
        return wk.CsrMatrix(ns.nrows, ns.ncols, ns.row_ptrs, ns.col_idx, ns.values)
    if kind == "sellp":
        return wk.SellpMatrix(ns.nrows, ns.ncols, ns.slice_size, ns.slice_sets, ns.col_idx, ns.values, ns.row_lengths)
    raise ValueError(kind)


def _is_int(case):
    return np.all(case.coo.values == np.round(case.coo.values)) and np.all(case.x == np.round(case.x))


# ---- SpMV on the reference's golden cases ---------------------------------------------------


@pytest.mark.parametrize("case", SPMV, ids=[c.name for c in SPMV])
def test_sellp_golden_bitwise(wk, ex, case):
    for s, sp in case.sellp.items():
        y = wk.spmv_sellp(_host(wk, sp, "sellp"), case.x, ex)
        assert y.tobytes() == case.y.tobytes(), f"slice {s}"


CSR_LONG_ROW = 256  # kCsrChunk: longer rows are split across work items (tolerance)


CSR_BITWISE_ROW = {"stream": 256, "rowblock": 64}  # rows up to this length fold bitwise


@pytest.mark.parametrize("case", SPMV, ids=[c.name for c in SPMV])
@pytest.mark.parametrize("strategy", ["stream", "rowblock", "merge", "load_balance", "auto"])
def test_csr_golden(wk, case, strategy):
    """stream / rowblock fold short rows bitwise; merge (merge-path tiles)
    reassociates rows cut by thread boundaries: 1e-12 scaled, exact on
    integer data; load_balance (seg8 warp ranges) adds the partial sums of a
    row cut by range boundaries in range order. Both are deterministic. auto
    resolves to rowblock or load_balance."""
    from paper_2006_14290_b200 import device as D

    e = wk.make_executor("b200", device=0, tuning={"csr_strategy": strategy})
    m = _host(wk, case.csr, "csr")
    y = wk.spmv_csr(m, case.x, e)
    lens = np.diff(case.csr.row_ptrs)
    assert sparse_ref.max_scaled_rel_err(y, case.y, lens) <= TOL
    if _is_int(case):
        assert np.array_equal(y, case.y)
    resolved = D.as_device(m, 0).auto_strategy() if strategy == "auto" else strategy
    if resolved in CSR_BITWISE_ROW:
        short = lens <= CSR_BITWISE_ROW[resolved]
        assert y[short].tobytes() == case.y[short].tobytes()
    elif resolved in ("merge", "load_balance"):
        assert wk.spmv_csr(m, case.x, e).tobytes() == y.tobytes()  # deterministic


@pytest.mark.parametrize("case", SPMV, ids=[c.name for c in SPMV])
def test_csr_subwarp_golden(wk, case):
    m = _host(wk, case.csr, "csr")
    nnz = sparse_ref.row_nnz(case.csr)
    for tile in (0, 1, 2, 4, 8, 16, 32):
        e = wk.make_executor("b200", device=0, tuning={"csr_strategy": "subwarp", "csr_subwarp_size": tile})
        y = wk.spmv_csr(m, case.x, e)
        if tile == 1 or _is_int(case):
            assert np.array_equal(y, case.y), tile
        else:
            assert sparse_ref.max_scaled_rel_err(y, case.y, nnz) <= TOL, tile


@pytest.mark.parametrize("case", SPMV, ids=[c.name for c in SPMV])
def test_coo_golden(wk, ex, case):
    y = wk.spmv_coo(_host(wk, case.coo, "coo"), case.x, ex)
    if _is_int(case):
        assert np.array_equal(y, case.y)
    else:
        assert sparse_ref.max_scaled_rel_err(y, case.y, sparse_ref.row_nnz(case.csr)) <= TOL


@pytest.mark.parametrize("aligned", [True, False])
@pytest.mark.parametrize("shape", ["skewed", "many_tiles", "one_row", "multi_range"])
def test_coo_hybrid_skewed(wk, ex, rng, shape, aligned):
    """COO and Hybrid (ELL + COO accumulate) on skewed / multi-range inputs
    (nnz not a multiple of 4: a tail past the last vector boundary); the
    unaligned case (device arrays offset by one element) takes the scalar-load
    path of the same kernel."""
    import torch

    from paper_2006_14290_b200 import device as D
    from paper_2006_14290_b200 import kernels as K

    ncols = 70000
    if shape == "one_row":
        lens = np.array([0, 60000, 0, 3])
    elif shape == "multi_range":
        lens = np.minimum((rng.pareto(1.2, size=900001) * 4).astype(np.int64), 5000)
        lens[rng.random(len(lens)) < 0.3] = 0
        lens[-1] = 7 - int(lens[:-1].sum()) % 4  # nnz % 4 == 3: a tail past the last 4-entry boundary
    else:
        n = 400000 if shape == "many_tiles" else 30000
        lens = np.minimum((rng.pareto(1.3, size=n) * 5).astype(np.int64), 20000)
        lens[rng.random(n) < 0.4] = 0
    ptrs, cols, vals = _banded_case(rng, lens, ncols)
    csr = wk.CsrMatrix(len(lens), ncols, ptrs, cols, vals)
    x = rng.standard_normal(ncols)
    y_ref = sparse_ref.spmv(csr, x)
    coo = wk.csr_to_coo(csr, ex)
    if aligned:
        assert sparse_ref.max_scaled_rel_err(wk.spmv_coo(coo, x, ex), y_ref, lens) <= TOL
        hyb = wk.csr_to_hybrid(csr, width=3, exec=ex)
        assert sparse_ref.max_scaled_rel_err(wk.spmv_hybrid(hyb, x, ex), y_ref, lens) <= TOL
    else:
        def off1(a, dt):
            t = torch.empty(len(a) + 1, dtype=dt, device="cuda")
            t[1:] = torch.as_tensor(np.asarray(a), dtype=dt, device="cuda")
            return t[1:]

        d = D.DeviceCoo(coo.nrows, coo.ncols, off1(coo.row_idx, torch.int32), off1(coo.col_idx, torch.int32),
                        off1(coo.values, torch.float64))
        y = K.spmv_device(d, torch.as_tensor(x, device="cuda")).cpu().numpy()
        assert sparse_ref.max_scaled_rel_err(y, y_ref, lens) <= TOL


@pytest.mark.parametrize("case", SPMV, ids=[c.name for c in SPMV])
def test_conversions_golden_bitwise(wk, ex, case):
    coo = _host(wk, case.coo, "coo")
    csr = wk.coo_to_csr(coo, ex)
    assert np.array_equal(csr.row_ptrs, case.csr.row_ptrs)
    assert np.array_equal(csr.col_idx, case.csr.col_idx)
    assert csr.values.tobytes() == case.csr.values.tobytes()
    for s, ref in case.sellp.items():
        got = wk.coo_to_sellp(coo, s, ex)
        assert np.array_equal(got.slice_sets, ref.slice_sets), s
        assert np.array_equal(got.row_lengths, ref.row_lengths), s
        assert np.array_equal(got.col_idx, ref.col_idx), s
        assert got.values.tobytes() == ref.values.tobytes(), s


@pytest.mark.parametrize("nrows,stride", [(1000, 1000), (4096, 4096), (4100, 4100), (130, 132), (999, 1004),
                                          (1001, 1001), (2000, 2050)])
def test_ell_strides_bitwise(wk, ex, rng, nrows, stride):
    """ELL through the TMA pipeline (stride % 4 == 0, partial last 64-row
    block) and the register kernel (other strides): bitwise vs the oracle,
    also with non-finite x[0] (padding must then be skipped via row_lengths)."""
    ncols = 3000
    lens = rng.integers(0, 30, size=nrows)
    lens[rng.random(nrows) < 0.1] = 0
    ptrs = np.concatenate(([0], np.cumsum(lens))).astype(np.int64)
    cols = np.concatenate([np.sort(rng.choice(ncols, size=int(L), replace=False)) for L in lens])
    csr = wk.CsrMatrix(nrows, ncols, ptrs, cols, rng.standard_normal(len(cols)))
    ell = wk.csr_to_ell(csr, stride=stride, exec=ex)
    ref = sparse_ref.csr_to_ell(csr, stride=stride)
    assert np.array_equal(ell.col_idx, ref.col_idx) and ell.values.tobytes() == ref.values.tobytes()
    for x0 in (0.5, np.inf):
        x = rng.standard_normal(ncols)
        x[0] = x0
        y_ref = sparse_ref.spmv(csr, x)
        assert wk.spmv_ell(ell, x, ex).tobytes() == y_ref.tobytes()


@pytest.mark.parametrize("nrows,stride", [(400003, 400004), (400000, 400000)])
def test_ell_many_tiles_bitwise(wk, ex, rng, nrows, stride):
    """More 512-row tiles than CTAs in the persistent grid (every ring stage
    reused across tiles), a partial last tile, a width that is not a multiple
    of the stage's column count; bitwise vs the oracle."""
    ncols = 50000
    lens = rng.integers(0, 11, size=nrows)
    lens[7] = 13
    ptrs = np.concatenate(([0], np.cumsum(lens))).astype(np.int64)
    rows = np.repeat(np.arange(nrows), lens)
    start = rng.integers(0, ncols - 13, size=nrows)
    cols = start[rows] + (np.arange(ptrs[-1]) - ptrs[rows])
    csr = wk.CsrMatrix(nrows, ncols, ptrs, cols, rng.standard_normal(len(cols)))
    ell = wk.csr_to_ell(csr, stride=stride, exec=ex)
    assert ell.width == 13
    x = rng.standard_normal(ncols)
    assert wk.spmv_ell(ell, x, ex).tobytes() == sparse_ref.spmv(csr, x).tobytes()


@pytest.mark.parametrize("case", SPMV, ids=[c.name for c in SPMV])
def test_ell_hybrid_golden(wk, ex, case):
    csr = _host(wk, case.csr, "csr")
    ell = wk.csr_to_ell(csr, exec=ex)
    ref = sparse_ref.csr_to_ell(case.csr)
    assert ell.width == ref.width and ell.stride == ref.stride
    assert np.array_equal(ell.col_idx, ref.col_idx) and ell.values.tobytes() == ref.values.tobytes()
    assert np.array_equal(ell.row_lengths, ref.row_lengths)
    assert wk.spmv_ell(ell, case.x, ex).tobytes() == case.y.tobytes()
    nnz = sparse_ref.row_nnz(case.csr)
    for k in (0, 1, 3, None):
        hyb = wk.csr_to_hybrid(csr, width=k, exec=ex)
        kk = hyb.ell.width
        href = sparse_ref.csr_to_hybrid(case.csr, kk)
        assert np.array_equal(hyb.ell.col_idx, href.ell.col_idx)
        assert hyb.ell.values.tobytes() == href.ell.values.tobytes()
        assert np.array_equal(hyb.coo.row_idx, href.coo.row_idx)
        assert np.array_equal(hyb.coo.col_idx, href.coo.col_idx)
        assert hyb.coo.values.tobytes() == href.coo.values.tobytes()
        y = wk.spmv_hybrid(hyb, case.x, ex)
        if _is_int(case):
            assert np.array_equal(y, case.y)
        else:
            assert sparse_ref.max_scaled_rel_err(y, case.y, nnz) <= TOL


def test_from_entries_duplicates(wk):
    case = next(c for c in SPMV if c.name == "duplicates")
    m = wk.CooMatrix.from_entries(3, 3, [2, 0, 2, 2, 1, 0], [1, 0, 1, 1, 2, 0], [0.1, 0.2, 0.3, 0.7, 1.0, 1e-17])
    assert np.array_equal(m.row_idx, case.coo.row_idx) and np.array_equal(m.col_idx, case.coo.col_idx)
    assert m.values.tobytes() == case.coo.values.tobytes()
    ez = next(c for c in SPMV if c.name == "explicit_zeros")
    m = wk.CooMatrix.from_entries(5, 5, [0, 0, 1, 2, 3, 3, 4], [0, 3, 1, 4, 0, 2, 4],
                                  [0.0, -1.5, 2.25, -0.0, 1e-300, -7.0, 3.0])
    assert m.values.tobytes() == ez.coo.values.tobytes()


@pytest.mark.parametrize("ss", [1, 4, 32, 64, 256, 512])
def test_sellp_fill_kernels_bitwise(wk, ex, rng, ss):
    """CSR -> SELL-P fill (TMA ring for 4 <= ss <= 256, staged scatter otherwise): many slices per CTA of
    the persistent grid, slices too wide for a stage (a 5000-entry row, direct
    path), empty slices, a last slice whose 16-byte-widened range would pass
    nnz; every array bitwise vs the oracle (sparse.py:219-242)."""
    nrows, ncols = 150001, 40000
    lens = rng.integers(0, 12, size=nrows)
    lens[1000:1000 + 3 * ss] = 0
    lens[77] = 5000
    lens[-1] = 3 - int(lens[:-1].sum()) % 4 + 4  # nnz % 4 == 3
    ptrs = np.concatenate(([0], np.cumsum(lens))).astype(np.int64)
    rows = np.repeat(np.arange(nrows), lens)
    start = rng.integers(0, ncols - 5000, size=nrows)
    cols = start[rows] + (np.arange(ptrs[-1]) - ptrs[rows])
    csr = wk.CsrMatrix(nrows, ncols, ptrs, cols, rng.standard_normal(len(cols)))
    assert csr.nnz % 4 == 3
    got = wk.csr_to_sellp(csr, ss, ex)
    ref = sparse_ref.csr_to_sellp(csr, ss)
    assert np.array_equal(got.slice_sets, ref.slice_sets)
    assert np.array_equal(got.row_lengths, ref.row_lengths)
    assert np.array_equal(got.col_idx, ref.col_idx)
    assert got.values.tobytes() == ref.values.tobytes()
    if ss != 64:
        return
    # the same kernels fill ELL (tiles of 2^k rows, stride padding rows) and the Hybrid ELL part (clipped rows)
    for stride in (nrows, nrows + 3, nrows + 1000):
        ell = wk.csr_to_ell(csr, stride=stride, exec=ex)
        eref = sparse_ref.csr_to_ell(csr, stride=stride)
        assert np.array_equal(ell.col_idx, eref.col_idx) and ell.values.tobytes() == eref.values.tobytes()
        assert np.array_equal(ell.row_lengths, eref.row_lengths)
    hyb = wk.csr_to_hybrid(csr, width=5, exec=ex)
    href = sparse_ref.csr_to_hybrid(csr, 5)
    assert np.array_equal(hyb.ell.col_idx, href.ell.col_idx)
    assert hyb.ell.values.tobytes() == href.ell.values.tobytes()
    assert np.array_equal(hyb.coo.col_idx, href.coo.col_idx) and hyb.coo.values.tobytes() == href.coo.values.tobytes()


# ---- edge cases -----------------------------------------------------------------------------


@pytest.mark.parametrize("x0", [np.inf, -np.inf, np.nan])
def test_nonfinite_x0_follows_oracle(wk, ex, x0, rng):
    m = corpus_ref.random_sparse(70, 70, 0.1, rng)
    csr = sparse_ref.coo_to_csr(m)
    x = rng.standard_normal(70)
    x[0] = x0
    y_ref = sparse_ref.spmv(csr, x)
    for s in (1, 8, 64):
        sp = sparse_ref.csr_to_sellp(csr, s)
        y = wk.spmv_sellp(_host(wk, sp, "sellp"), x, ex)
        assert np.array_equal(y, y_ref, equal_nan=True)
    hc = _host(wk, csr, "csr")
    y = wk.spmv_ell(wk.csr_to_ell(hc, exec=ex), x, ex)
    assert np.array_equal(y, y_ref, equal_nan=True)
    assert np.array_equal(wk.spmv_csr(hc, x, ex), y_ref, equal_nan=True)


def test_dimension_mismatch(wk, ex):
    case = SPMV[0]
    with pytest.raises(wk.DimensionMismatch):
        wk.spmv_coo(_host(wk, case.coo, "coo"), np.ones(5), ex)
    with pytest.raises(wk.DimensionMismatch):
        wk.spmv_sellp(_host(wk, case.sellp[2], "sellp"), np.ones(2), ex)
    with pytest.raises(wk.InvalidSliceSize):
        wk.coo_to_sellp(_host(wk, case.coo, "coo"), 12, ex)


def test_empty_matrices(wk, ex):
    z = wk.CsrMatrix(4, 3, [0, 0, 0, 0, 0], [], [])
    assert np.array_equal(wk.spmv_csr(z, np.ones(3), ex), np.zeros(4))
    sp = wk.csr_to_sellp(z, 2, ex)
    assert sp.slice_sets.tolist() == [0, 0, 0]
    assert np.array_equal(wk.spmv_sellp(sp, np.ones(3), ex), np.zeros(4))
    e = wk.CsrMatrix(0, 0, [0], [], [])
    assert wk.spmv_csr(e, np.zeros(0), ex).shape == (0,)


def test_long_rows_stream_kernel(wk, ex, rng):
    # rows much longer than the 1024-entry chunk: split across work items,
    # partials combined deterministically
    n, ncols = 600, 50000
    lens = np.zeros(n, dtype=np.int64)
    lens[[0, 1, 7, 300, 599]] = [30000, 2500, 1025, 40000, 9000]
    lens[lens == 0] = rng.integers(0, 40, size=int((lens == 0).sum()))
    ptrs = np.concatenate(([0], np.cumsum(lens)))
    cols = np.concatenate([np.sort(rng.choice(ncols, size=int(L), replace=False)) for L in lens])
    vals = rng.standard_normal(len(cols))
    csr = wk.CsrMatrix(n, ncols, ptrs, cols, vals)
    x = rng.standard_normal(ncols)
    y_ref = sparse_ref.spmv(csr, x)
    es = wk.make_executor("b200", device=0, tuning={"csr_strategy": "stream"})
    y = wk.spmv_csr(csr, x, es)
    short = lens <= CSR_LONG_ROW
    assert y[short].tobytes() == y_ref[short].tobytes()
    assert sparse_ref.max_scaled_rel_err(y, y_ref, lens) <= TOL
    assert wk.spmv_csr(csr, x, es).tobytes() == y.tobytes()  # deterministic
    ym = wk.spmv_csr(csr, x, ex)  # auto -> merge
    assert sparse_ref.max_scaled_rel_err(ym, y_ref, lens) <= TOL
    # forced row-block strategy: heavy blocks (long rows) take the warp-reduction path
    eb = wk.make_executor("b200", device=0, tuning={"csr_strategy": "rowblock"})
    yb = wk.spmv_csr(csr, x, eb)
    assert yb[lens <= 64].tobytes() == y_ref[lens <= 64].tobytes()
    assert sparse_ref.max_scaled_rel_err(yb, y_ref, lens) <= TOL
    coo = wk.csr_to_coo(csr, ex)
    assert sparse_ref.max_scaled_rel_err(wk.spmv_coo(coo, x, ex), y_ref, lens) <= TOL
    hyb = wk.csr_to_hybrid(csr, exec=ex)
    assert sparse_ref.max_scaled_rel_err(wk.spmv_hybrid(hyb, x, ex), y_ref, lens) <= TOL


def _merge_case(rng, lens, ncols, ints=False):
    ptrs = np.concatenate(([0], np.cumsum(lens))).astype(np.int64)
    cols = np.concatenate([np.sort(rng.choice(ncols, size=int(L), replace=False)) for L in lens]) if len(lens) else \
        np.zeros(0, np.int64)
    vals = rng.integers(1, 10, size=len(cols)).astype(np.float64) if ints else rng.standard_normal(len(cols))
    return ptrs, cols.astype(np.int64), vals


MERGE_TILE = 2048  # csr_merge.cuh kMgTile: merge items (row ends + nonzeros) per CTA


def _banded_case(rng, lens, ncols):
    """rows of consecutive columns at random offsets (vectorised; big cases)."""
    ptrs = np.concatenate(([0], np.cumsum(lens))).astype(np.int64)
    start = rng.integers(0, ncols - lens.max(initial=0) + 1, size=len(lens))
    rows = np.repeat(np.arange(len(lens)), lens)
    cols = start[rows] + (np.arange(ptrs[-1]) - ptrs[rows])
    return ptrs, cols.astype(np.int64), rng.standard_normal(int(ptrs[-1]))


@pytest.mark.parametrize("strategy", ["merge", "load_balance"])
@pytest.mark.parametrize("shape", ["tile_spanning_row", "empty_runs", "tile_aligned", "all_empty", "one_row",
                                   "skewed", "ints", "many_tiles", "multi_range"])
def test_csr_balanced_edge_cases(wk, rng, shape, strategy):
    """merge-path and load-balance CSR: rows spanning many tiles / warp
    ranges, long runs of empty rows crossing them, rows ending exactly on tile /
    thread boundaries, empty matrices; tolerance 1e-12, exact on integer data;
    both are deterministic."""
    ncols = 70000
    if shape == "tile_spanning_row":
        lens = np.array([3, 50000, 2, 0, 7000, 1] + [5] * 900)
    elif shape == "empty_runs":
        lens = np.zeros(20000, np.int64)
        lens[[5, 6000, 6001, 19999]] = [4000, 3, 2100, 9]
    elif shape == "tile_aligned":
        # every row is 2047 entries: row end + entries = one tile exactly; plus 7-item rows (thread boundaries)
        lens = np.array([MERGE_TILE - 1] * 6 + [7] * 3000)
    elif shape == "all_empty":
        lens = np.zeros(5000, np.int64)
    elif shape == "one_row":
        lens = np.array([60000])
    else:
        lens = np.minimum((rng.pareto(1.2, size=30000) * 3).astype(np.int64), ncols)
        lens[rng.random(30000) < 0.5] = 0
    if shape == "many_tiles":
        # > 2 tiles per CTA of the persistent grid: every pipeline stage is reused
        lens = np.minimum((rng.pareto(1.5, size=400000) * 6).astype(np.int64), 20000)
        lens[rng.random(400000) < 0.3] = 0
        ptrs, cols, vals = _banded_case(rng, lens, ncols)
    elif shape == "multi_range":
        # more 2048-entry warp ranges than warps in the persistent seg8 grid
        lens = np.minimum((rng.pareto(1.2, size=900001) * 4).astype(np.int64), 5000)
        lens[rng.random(len(lens)) < 0.3] = 0
        lens[-1] = 7 - int(lens[:-1].sum()) % 4  # nnz % 4 == 3
        ptrs, cols, vals = _banded_case(rng, lens, ncols)
    else:
        ptrs, cols, vals = _merge_case(rng, lens, ncols, ints=(shape == "ints"))
    if shape == "ints":
        lens = np.minimum((rng.pareto(1.2, size=20000) * 3).astype(np.int64), 3000)
        ptrs, cols, vals = _merge_case(rng, lens, ncols, ints=True)
    csr = wk.CsrMatrix(len(lens), ncols, ptrs, cols, vals)
    x = rng.integers(-5, 6, size=ncols).astype(np.float64) if shape == "ints" else rng.standard_normal(ncols)
    y_ref = sparse_ref.spmv(csr, x)
    e = wk.make_executor("b200", device=0, tuning={"csr_strategy": strategy})
    y = wk.spmv_csr(csr, x, e)
    assert sparse_ref.max_scaled_rel_err(y, y_ref, lens) <= TOL
    if shape == "ints":
        assert np.array_equal(y, y_ref)
    assert np.all(y[lens == 0] == 0.0)
    assert wk.spmv_csr(csr, x, e).tobytes() == y.tobytes()  # both deterministic (no atomics)
    if strategy == "merge":
        # rows folded inside one thread's 8 items are the reference fold exactly
        one = lens <= 1
        assert y[one].tobytes() == y_ref[one].tobytes()
    # masked SpMV through the solver entry point: skip flag set -> y untouched
    from paper_2006_14290_b200 import device as D
    from paper_2006_14290_b200 import _lib

    d = D.as_device(csr, 0).with_strategy(strategy)
    xt = torch.as_tensor(x, device="cuda")
    yt = torch.full((csr.nrows,), 7.0, dtype=torch.float64, device="cuda")
    flag = torch.ones(1, dtype=torch.int32, device="cuda")
    _lib.call("wk_spmv_masked", d.wk_ptr(), D._ptr(xt), D._ptr(yt), D._ptr(flag), D.stream_handle(d.device))
    assert torch.all(yt == 7.0)
    flag.zero_()
    _lib.call("wk_spmv_masked", d.wk_ptr(), D._ptr(xt), D._ptr(yt), D._ptr(flag), D.stream_handle(d.device))
    assert sparse_ref.max_scaled_rel_err(yt.cpu().numpy(), y_ref, lens) <= TOL


@pytest.mark.parametrize("shape", ["stencil", "random", "tiny"])
def test_spmv_pipeline_bitwise(wk, ex, rng, shape):
    """Host-to-host pipeline (chunked copy-in / sub-range SpMV launches /
    chunked copy-out on three streams, two alternating buffer sets) ==
    the one-launch SpMV, bit for bit, over several in-flight submissions."""
    from paper_2006_14290_b200 import corpus

    if shape == "stencil":
        m = corpus.stencil3d(20, 27).to_host()
    elif shape == "random":
        lens = rng.integers(0, 40, size=3000)
        ptrs, cols, vals = _banded_case(rng, lens, 5000)
        m = wk.CsrMatrix(3000, 5000, ptrs, cols, vals)
    else:
        m = wk.CsrMatrix(3, 2, [0, 1, 1, 3], [1, 0, 1], [2.0, 3.0, 4.0])
    sp = wk.csr_to_sellp(m, 64, ex)
    pipe = wk.SpmvPipeline(sp, chunks=7, pieces=5)
    xs = [torch.from_numpy(rng.standard_normal(m.ncols)).pin_memory() for _ in range(5)]
    ys = [torch.empty(m.nrows, dtype=torch.float64, pin_memory=True) for _ in range(5)]
    for xh, yh in zip(xs, ys):
        pipe.submit(xh, yh)
    pipe.synchronize()
    for xh, yh in zip(xs, ys):
        ref = sparse_ref.spmv(m, xh.numpy())
        assert yh.numpy().tobytes() == ref.tobytes()
    assert pipe(xs[0].numpy()).tobytes() == sparse_ref.spmv(m, xs[0].numpy()).tobytes()
    with pytest.raises(wk.DimensionMismatch):
        pipe.submit(torch.zeros(m.ncols + 1, dtype=torch.float64), ys[0])


# ---- generators ---------------------------------------------------------------------------


def test_device_generators_match_oracle(wk):
    from paper_2006_14290_b200 import corpus

    for dev, ref in (
        (corpus.poisson2d_matrix(17), corpus_ref.poisson2d(17)),
        (corpus.stencil3d(9, 7), corpus_ref.stencil(9, 9, 9, corpus_ref.points_7pt())),
        (corpus.stencil3d(8, 27), corpus_ref.stencil(8, 8, 8, corpus_ref.points_27pt())),
        (corpus.convection_diffusion3d(7), corpus_ref.stencil(7, 7, 7, corpus_ref.points_7pt(beta=(1.0, 0.5, 0.25)))),
    ):
        h = dev.to_host()
        assert np.array_equal(h.row_ptrs, ref.row_ptrs)
        assert np.array_equal(h.col_idx, ref.col_idx)
        assert h.values.tobytes() == ref.values.tobytes()
    r = corpus.rmat(12, edge_factor=8).to_host()
    rr = corpus_ref.rmat(12, edge_factor=8)
    assert np.array_equal(r.row_idx, rr.row_idx) and np.array_equal(r.col_idx, rr.col_idx)
    assert r.values.tobytes() == rr.values.tobytes()


# ---- BLAS-1 -------------------------------------------------------------------------------


def test_blas1(wk, ex, rng):
    for n in (0, 1, 31, 1000, 300001):
        a = rng.standard_normal(n)
        b = rng.standard_normal(n)
        d = wk.dot(a, b, ex)
        assert abs(d - float(a @ b)) <= 1e-12 * max(1.0, float(np.abs(a) @ np.abs(b)))
        assert abs(wk.norm2(a, ex) - float(np.linalg.norm(a))) <= 1e-12 * max(1.0, float(np.linalg.norm(a)))
        y = wk.axpy(0.37, a, b, ex)
        assert y.tobytes() == (b + 0.37 * a).tobytes()
    a = rng.standard_normal(123457)
    assert wk.dot(a, a, ex) == wk.dot(a, a, ex)  # deterministic


# ---- CG -------------------------------------------------------------------------------------


@pytest.mark.parametrize("case", CG, ids=[c.name for c in CG])
@pytest.mark.parametrize("fmt", ["sellp", "csr", "ell"])
def test_cg_golden(wk, ex, case, fmt):
    coo = _host(wk, case.coo, "coo")
    if fmt == "sellp":
        m = wk.coo_to_sellp(coo, 64, ex)
    elif fmt == "csr":
        m = wk.coo_to_csr(coo, ex)
    else:
        m = wk.csr_to_ell(wk.coo_to_csr(coo, ex), exec=ex)
    x, hist = wk.cg_solve(m, case.b, case.tol, case.max_iters, ex)
    assert len(hist) == len(case.hist)
    bn = max(float(np.linalg.norm(case.b)), 1e-300)
    assert np.max(np.abs(hist - case.hist)) / bn <= 1e-10
    assert sparse_ref.max_scaled_rel_err(x, case.x, sparse_ref.row_nnz(case.coo)) <= 1e-10


def test_cg_identity_and_2x2_exact(wk, ex):
    eye = wk.coo_to_sellp(wk.CooMatrix(3, 3, [0, 1, 2], [0, 1, 2], [1.0, 1.0, 1.0]), 64, ex)
    x, hist = wk.cg_solve(eye, np.array([1.0, 2.0, 3.0]), 1e-12, 50, ex)
    assert np.array_equal(x, [1.0, 2.0, 3.0]) and len(hist) == 2
    m = wk.coo_to_sellp(wk.CooMatrix(2, 2, [0, 0, 1, 1], [0, 1, 0, 1], [4.0, 1.0, 1.0, 3.0]), 64, ex)
    x, hist = wk.cg_solve(m, np.array([1.0, 2.0]), 1e-12, 10, ex)
    assert len(hist) - 1 <= 2 and np.max(np.abs(x - [1 / 11, 7 / 11])) <= 1e-12


def test_cg_errors(wk, ex):
    bad = wk.coo_to_sellp(wk.CooMatrix(2, 2, [0, 1], [0, 1], [1.0, -1.0]), 64, ex)
    with pytest.raises(wk.BreakdownError):
        wk.cg_solve(bad, np.array([0.0, 1.0]), 1e-10, 10, ex)
    rect = wk.coo_to_sellp(wk.CooMatrix(2, 3, [0], [1], [1.0]), 64, ex)
    with pytest.raises(wk.DimensionMismatch):
        wk.cg_solve(rect, np.ones(2), 1e-10, 5, ex)
    sq = wk.coo_to_sellp(wk.CooMatrix(3, 3, [0, 1, 2], [0, 1, 2], [2.0, 2.0, 2.0]), 64, ex)
    with pytest.raises(wk.DimensionMismatch):
        wk.cg_solve(sq, np.ones(4), 1e-10, 5, ex)
    with pytest.raises(ValueError):
        wk.cg_solve(sq, np.ones(3), 0.0, 5, ex)
    x, hist = wk.cg_solve(sq, np.zeros(3), 1e-10, 5, ex)
    assert np.array_equal(x, np.zeros(3)) and len(hist) == 1


def test_cg_device_resident_and_factory(wk, ex):
    from paper_2006_14290_b200 import corpus

    A = wk.csr_to_sellp(corpus.stencil3d(16, 7), 64, ex)
    b = torch.ones(A.nrows, dtype=torch.float64, device="cuda")
    x, hist = wk.cg_solve(A, b, 1e-10, 1000, ex)
    assert isinstance(x, torch.Tensor) and x.is_cuda
    Ah = A.to_host()
    xr, hr = krylov_ref.cg_solve(lambda v: sparse_ref.spmv(Ah, v), np.ones(A.nrows), 1e-10, 1000)
    assert len(hist) == len(hr)
    assert np.max(np.abs(hist.cpu().numpy() - hr)) / np.sqrt(A.nrows) <= 1e-10
    solver = wk.Cg([wk.Iteration(1000), wk.ResidualNorm(1e-10)], ex).generate(A)
    xs = solver.apply(b)
    assert solver.iterations == len(hr) - 1
    assert torch.equal(xs, x)


# ---- Jacobi PCG, diagonal, reduction microbenchmark -----------------------


def _shifted_stencil(wk, n, rng):
    """7-point 3-D Laplacian scaled symmetrically, S A S with S = diag(10^u),
    u ~ U(-1.5, 1.5): SPD, rows of very different scale (Jacobi undoes the
    scaling; plain CG struggles)."""
    from paper_2006_14290_b200 import corpus

    h = corpus.stencil3d(n, 7).to_host()
    rows = np.repeat(np.arange(h.nrows), np.diff(h.row_ptrs))
    cols = np.asarray(h.col_idx)
    sc = 10.0 ** rng.uniform(-1.5, 1.5, size=h.nrows)
    vals = np.array(h.values, dtype=np.float64) * sc[rows] * sc[cols]
    return wk.CsrMatrix(h.nrows, h.ncols, h.row_ptrs, h.col_idx, vals), vals[rows == cols]


@pytest.mark.parametrize("fmt", ["csr", "sellp", "ell", "coo", "hybrid"])
def test_diagonal_all_formats(wk, ex, rng, fmt):
    A, d_ref = _shifted_stencil(wk, 9, rng)
    m = {"csr": lambda: A, "sellp": lambda: wk.csr_to_sellp(A, 64, ex), "ell": lambda: wk.csr_to_ell(A, exec=ex),
         "coo": lambda: wk.csr_to_coo(A, ex), "hybrid": lambda: wk.csr_to_hybrid(A, width=3, exec=ex)}[fmt]()
    d = wk.diagonal(m, ex).cpu().numpy()
    assert d.tobytes() == d_ref.tobytes()
    z = wk.CsrMatrix(3, 3, [0, 1, 1, 2], [1, 0], [5.0, 6.0])  # rows without a diagonal entry -> 0.0
    assert wk.diagonal(z, ex).cpu().numpy().tolist() == [0.0, 0.0, 0.0]


@pytest.mark.parametrize("fmt", ["sellp", "csr"])
@pytest.mark.parametrize("n", [10, 15])
def test_pcg_jacobi_matches_oracle(wk, ex, rng, fmt, n):
    """> 50 iterations (residual replacement), equal counts, history within
    1e-10 ||b||; Jacobi takes fewer iterations than plain CG here."""
    A, d_ref = _shifted_stencil(wk, n, rng)
    m = wk.csr_to_sellp(A, 64, ex) if fmt == "sellp" else A
    b = rng.standard_normal(A.nrows)
    x, hist = wk.pcg_solve(m, b, 1e-13, 2000, ex)
    f = lambda v: sparse_ref.spmv(A, v)  # noqa: E731
    xr, hr = krylov_ref.pcg_jacobi_solve(f, d_ref, b, 1e-13, 2000)
    assert len(hist) == len(hr) and len(hr) > 51
    assert np.max(np.abs(hist - hr)) / np.linalg.norm(b) <= 1e-10
    assert sparse_ref.max_scaled_rel_err(x, xr, sparse_ref.row_nnz(A)) <= 1e-10
    _, hc = wk.cg_solve(m, b, 1e-13, 500, ex)
    assert len(hist) < len(hc)
    solver = wk.Cg([wk.Iteration(2000), wk.ResidualNorm(1e-13)], ex, preconditioner=wk.Jacobi()).generate(m)
    xs = solver.apply(b)
    assert solver.iterations == len(hr) - 1 and np.array_equal(xs, x)


def test_pcg_breakdown_and_errors(wk, ex):
    bad = wk.coo_to_sellp(wk.CooMatrix(2, 2, [0, 1], [0, 1], [1.0, -1.0]), 64, ex)
    with pytest.raises(wk.BreakdownError):
        wk.pcg_solve(bad, np.array([0.0, 1.0]), 1e-10, 10, ex, diag=np.ones(2))
    sq = wk.coo_to_sellp(wk.CooMatrix(3, 3, [0, 1, 2], [0, 1, 2], [2.0, 4.0, 8.0]), 64, ex)
    x, hist = wk.pcg_solve(sq, np.array([2.0, 4.0, 8.0]), 1e-12, 10, ex)
    assert np.array_equal(x, [1.0, 1.0, 1.0]) and len(hist) == 2  # exact in one step
    x, hist = wk.pcg_solve(sq, np.zeros(3), 1e-10, 5, ex)
    assert np.array_equal(x, np.zeros(3)) and len(hist) == 1
    with pytest.raises(ValueError):
        wk.pcg_solve(sq, np.ones(3), -1.0, 5, ex)


@pytest.mark.parametrize("shared", [False, True])
def test_reduce_microbench(wk, ex, shared):
    """kernels.py:341-364: every tile of `size` lanes reduces ranks 1..size."""
    for size in (1, 2, 4, 8, 16, 32):
        out, cycles = wk.reduce_microbench(size, 100, ex, shared_memory=shared)
        assert out.tolist() == [float(size * (size + 1) // 2)] * size
        assert cycles > 0
    with pytest.raises(ValueError):
        wk.reduce_microbench(3, 1, ex)


# ---- BiCGSTAB / GMRES (no reference: vs the oracle restatement) ----------------------------------


@pytest.mark.parametrize("n", [1, 7, 1000, 300001])
def test_bicg_steps_vector_and_scalar_paths(wk, rng, n):
    """The BiCGSTAB step kernels take the vectorised path (vmap_kernel) for
    16-byte aligned vectors and the scalar map/reduce path otherwise: same
    element arithmetic (bitwise vectors), dots within 1e-13 relative; the
    half-step x update runs only while apply_half is set and clears it."""
    import ctypes

    from paper_2006_14290_b200 import _lib

    L = _lib.load()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    ws = torch.zeros(int(L.wk_reduce_workspace_bytes()), dtype=torch.uint8, device="cuda")
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    host = {k: rng.standard_normal(n) for k in ("x", "p", "sv", "t", "r", "v", "rh")}

    def run(offset):
        buf = {k: torch.zeros(n + 2, dtype=torch.float64, device="cuda") for k in host}
        vec = {k: buf[k][offset: offset + n] for k in host}
        for k in host:
            vec[k].copy_(torch.from_numpy(host[k]))
        h = _lib.WkBicgState()
        h.alpha, h.omega, h.beta, h.apply_half = 0.37, -1.25, 0.81, 1
        state = torch.frombuffer(bytearray(bytes(h)), dtype=torch.uint8).to("cuda")
        S = P(state)
        _lib.check(L.wk_bicg_update_xr(n, P(vec["p"]), P(vec["sv"]), P(vec["t"]), P(vec["x"]), P(vec["r"]), S,
                                       P(ws), st), "xr")
        _lib.check(L.wk_bicg_update_p(n, P(vec["r"]), P(vec["v"]), P(vec["p"]), S, st), "p")
        _lib.check(L.wk_bicg_update_s(n, P(vec["r"]), P(vec["v"]), P(vec["sv"]), S, P(ws), st), "s")
        _lib.check(L.wk_bicg_tt_ts(n, P(vec["t"]), P(vec["sv"]), S, P(ws), st), "tt")
        _lib.check(L.wk_bicg_rho(n, P(vec["rh"]), P(vec["r"]), S, P(ws), st), "rho")
        _lib.check(L.wk_bicg_rv(n, P(vec["rh"]), P(vec["v"]), S, P(ws), st), "rv")
        _lib.check(L.wk_bicg_half_x(n, P(vec["p"]), P(vec["x"]), S, P(ws), st), "half")
        x_after_one = vec["x"].clone()
        _lib.check(L.wk_bicg_half_x(n, P(vec["p"]), P(vec["x"]), S, P(ws), st), "half again")  # flag now clear
        torch.cuda.synchronize()
        out = _lib.WkBicgState.from_buffer_copy(bytes(state.cpu().numpy()))
        assert out.apply_half == 0 and torch.equal(vec["x"], x_after_one)
        return {k: vec[k].cpu().numpy() for k in ("x", "r", "p", "sv")}, out

    va, sa = run(0)   # aligned: vectorised
    vs, ss = run(1)   # offset by one element: scalar fallback
    for k in va:
        assert va[k].tobytes() == vs[k].tobytes(), k
    for f in ("rr", "ss", "tt", "ts", "rho_new", "rv"):
        a, b = getattr(sa, f), getattr(ss, f)
        assert abs(a - b) <= 1e-13 * max(1.0, abs(b)), f
    # element arithmetic against numpy (kernels.py-style separate roundings)
    x0, p0, sv0, t0 = host["x"], host["p"], host["sv"], host["t"]
    x1 = (x0 + 0.37 * p0) + (-1.25) * sv0
    r1 = sv0 - (-1.25) * t0
    assert np.array_equal(va["r"], r1)
    assert np.allclose(va["x"], x1 + 0.37 * (r1 + 0.81 * (p0 - (-1.25) * host["v"])), rtol=0, atol=1e-12)


@pytest.mark.parametrize("grid", [12, 11])
@pytest.mark.parametrize("solver", ["bicgstab", "gmres"])
def test_nonsymmetric_solvers_match_oracle(wk, ex, solver, grid):
    from paper_2006_14290_b200 import corpus

    A = corpus.convection_diffusion3d(grid)
    Ah = A.to_host()
    b = np.ones(A.nrows)
    f = lambda v: sparse_ref.spmv(Ah, v)  # noqa: E731
    if solver == "bicgstab":
        x, hist = wk.bicgstab_solve(A, b, 1e-10, 500, ex)
        xr, hr = krylov_ref.bicgstab_solve(f, b, 1e-10, 500)
    else:
        x, hist = wk.gmres_solve(A, b, 1e-10, 500, ex, restart=30)
        xr, hr = krylov_ref.gmres_solve(f, b, 1e-10, 500, restart=30)
    x = x.cpu().numpy() if hasattr(x, "cpu") else x
    hist = hist.cpu().numpy() if hasattr(hist, "cpu") else hist
    assert len(hist) == len(hr)
    assert np.max(np.abs(hist - hr)) / np.linalg.norm(b) <= 1e-10
    assert sparse_ref.max_scaled_rel_err(x, xr, sparse_ref.row_nnz(Ah)) <= 1e-10
    assert hist[-1] <= 1e-10 * np.linalg.norm(b)


@pytest.mark.parametrize("n", [0, 1, 2, 2047, 2048, 2049, 32767, 32768, 32769, 100003, (1 << 20) + 7])
@pytest.mark.parametrize("key_bits", [1, 7, 9, 17, 48, 63])
def test_sort_pairs_stable(wk, n, key_bits):
    """csrc/sort.cu against numpy's stable argsort: keys with many duplicates
    (values = input positions, so stability is checked exactly), sub-tile /
    chunk boundaries, odd and even pass counts."""
    import torch

    from paper_2006_14290_b200 import device as D

    rng = np.random.default_rng(n * 64 + key_bits)
    hi = 1 << key_bits
    pool = rng.integers(0, hi, size=max(1, n // 3), dtype=np.uint64)  # ~3 copies per key
    keys = pool[rng.integers(0, len(pool), size=n)].astype(np.int64) if n else np.zeros(0, np.int64)
    vals = np.arange(n, dtype=np.float64)
    kt = torch.as_tensor(keys, device="cuda")
    vt = torch.as_tensor(vals, device="cuda")
    sk, sv = D.sort_pairs(kt, vt, key_bits=key_bits)
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(sk.cpu().numpy(), keys[order])
    assert np.array_equal(sv.cpu().numpy(), vals[order])
    assert np.array_equal(kt.cpu().numpy(), keys)  # not in place by default


def test_from_entries_rmat_matches_oracle(wk):
    """Device ingestion of R-MAT scale 16 (sort + duplicate fold) against the
    oracle's np.lexsort + np.add.at restatement, bitwise."""
    from paper_2006_14290_b200 import corpus
    from oracle import corpus_ref

    d = corpus.rmat(16).to_host()
    r = corpus_ref.rmat(16)
    assert np.array_equal(d.row_idx, r.row_idx) and np.array_equal(d.col_idx, r.col_idx)
    assert d.values.tobytes() == r.values.tobytes()


@pytest.mark.parametrize("shape", ["short_with_long_rows", "empty_rows", "exactly_8", "mean_above_8"])
def test_csr_rowblock_short_kernel_edges(wk, ex, rng, shape):
    """The rowblock strategy's thread-per-row kernel (mean row length <= 8)
    on rows longer than its 8-entry batch (one of 3000 entries), runs of
    empty rows, rows of exactly 8, and the TMA row-block path just above the
    mean threshold: bitwise against the reference fold, also with x[0] = inf
    (padding never enters a CSR fold)."""
    n, ncols = 50000, 60000
    lens = rng.integers(0, 9, size=n)
    if shape == "short_with_long_rows":
        lens[[3, 777, n - 1]] = [3000, 17, 9]
    elif shape == "empty_rows":
        lens[1000:9000] = 0
    elif shape == "exactly_8":
        lens[:] = 8
    else:
        lens = rng.integers(6, 13, size=n)  # mean ~9: the TMA row-block kernel
    ptrs, cols, vals = _banded_case(rng, lens, ncols)
    csr = wk.CsrMatrix(n, ncols, ptrs, cols, vals)
    e = wk.make_executor("b200", device=0, tuning={"csr_strategy": "rowblock"})
    for x0 in (0.25, np.inf):
        x = rng.standard_normal(ncols)
        x[0] = x0
        y = wk.spmv_csr(csr, x, e)
        assert y.tobytes() == sparse_ref.spmv(csr, x).tobytes()


@pytest.mark.parametrize("width", [0, 1, 4])
def test_hybrid_fill_long_row_boundaries(wk, ex, rng, width):
    """CSR -> Hybrid COO remainder around the fill's thresholds: rows whose
    overflow is 255 / 256 / 257 entries (flattened run vs long-row queue),
    4095 / 4096 / 4097 and 12289 (segment boundaries of the queue), 32-row
    groups full of long rows, and empty groups; bitwise against the oracle."""
    n, ncols = 4000, 20000
    lens = rng.integers(0, 6, size=n)
    specials = [255, 256, 257, 4095, 4096, 4097, 12289]
    for i, L in enumerate(specials):
        lens[100 + i] = L + width
    lens[640:672] = 300 + width       # a 32-row group of long rows
    lens[2000:2100] = 0               # empty groups
    ptrs, cols, vals = _banded_case(rng, lens, ncols)
    csr = wk.CsrMatrix(n, ncols, ptrs, cols, vals)
    hyb = wk.csr_to_hybrid(csr, width=width, exec=ex)
    ref = sparse_ref.csr_to_hybrid(csr, width)
    assert np.array_equal(hyb.coo.row_idx, ref.coo.row_idx)
    assert np.array_equal(hyb.coo.col_idx, ref.coo.col_idx)
    assert hyb.coo.values.tobytes() == ref.coo.values.tobytes()
    x = rng.standard_normal(ncols)
    assert sparse_ref.max_scaled_rel_err(wk.spmv_hybrid(hyb, x, ex), sparse_ref.spmv(csr, x), lens) <= TOL


def test_cg_pending_x_update_flushed_on_breakdown(wk, ex):
    """diag(1, 1, -1.5), b = ones: iteration 1 (alpha 6) is the even half of a
    paired x update (cg_update_xp_pair<0> defers x += alpha p), iteration 2
    breaks down (p.Ap = 4050 - 5400 < 0) before its x pass. wk_cg_solve must
    still leave x = x_1 = 6 * ones (the deferred update applied) and report
    the breaking iteration, 2 (the reference's "at iteration 2")."""
    import ctypes

    import torch

    from paper_2006_14290_b200 import _lib
    from paper_2006_14290_b200 import device as D

    A = wk.coo_to_sellp(wk.CooMatrix(3, 3, [0, 1, 2], [0, 1, 2], [1.0, 1.0, -1.5]), 64, ex)
    d = D.as_device(A, ex.device)
    b = torch.ones(3, dtype=torch.float64, device=d.device)
    x = torch.full((3,), -7.0, dtype=torch.float64, device=d.device)
    hist = torch.zeros(11, dtype=torch.float64, device=d.device)
    iters = ctypes.c_int64(-1)
    L = _lib.load()
    ws = torch.zeros(int(L.wk_cg_workspace_bytes(3)), dtype=torch.uint8, device=d.device)
    rc = L.wk_cg_solve(d.wk_ptr(), D._ptr(b), 1e-12, 10, D._ptr(x), D._ptr(hist), ctypes.byref(iters),
                       D._ptr(ws), D.stream_handle(d.device))
    torch.cuda.synchronize()
    assert rc == _lib.WK_ERR_BREAKDOWN
    assert iters.value == 2
    assert x.cpu().tolist() == [6.0, 6.0, 6.0]
    with pytest.raises(wk.BreakdownError):
        wk.cg_solve(A, np.ones(3), 1e-12, 10, ex)


@pytest.mark.parametrize("n", [2, 3, 4, 5])
def test_cg_converging_on_either_half_of_a_pair(wk, ex, n):
    """Diagonal systems with k distinct eigenvalues converge in exactly k
    iterations, so k = 2..5 ends the solve on the even (x update otherwise
    deferred) and the odd (both updates applied) iteration of a pair; x and
    the history must match the reference CG (dot products may reassociate:
    1e-12 relative)."""
    from oracle import krylov_ref

    vals = [1.0, 2.0, 4.0, 8.0, 16.0][:n]
    m = wk.coo_to_sellp(wk.CooMatrix(n, n, list(range(n)), list(range(n)), vals), 64, ex)
    b = np.arange(1.0, n + 1.0)
    x, hist = wk.cg_solve(m, b, 1e-14, 50, ex)
    rx, rh = krylov_ref.cg_solve(lambda v: np.asarray(vals) * v, b, 1e-14, 50)
    assert len(hist) == len(rh) == n + 1
    assert np.max(np.abs(np.asarray(x) - rx)) <= 1e-12 * np.max(np.abs(rx))
    assert np.max(np.abs(np.asarray(hist) - rh)) <= 1e-12 * rh[0]


@pytest.mark.parametrize("restart", [1, 2, 5, 31])
def test_gmres_restart_lengths_match_oracle(wk, ex, restart):
    """GMRES with deferred normalisation (wk_gmres_solve keeps the basis
    unscaled, v_i = sig_i u_i) against the restatement's explicit
    normalisation, for restart lengths from 1 to the maximum, odd n."""
    from paper_2006_14290_b200 import corpus

    A = corpus.convection_diffusion3d(7)
    Ah = A.to_host()
    b = np.linspace(1.0, 2.0, A.nrows)
    f = lambda v: sparse_ref.spmv(Ah, v)  # noqa: E731
    x, hist = wk.gmres_solve(A, b, 1e-10, 400, ex, restart=restart)
    xr, hr = krylov_ref.gmres_solve(f, b, 1e-10, 400, restart=restart)
    x = x.cpu().numpy() if hasattr(x, "cpu") else x
    hist = hist.cpu().numpy() if hasattr(hist, "cpu") else hist
    assert len(hist) == len(hr)
    assert np.max(np.abs(hist - hr)) / np.linalg.norm(b) <= 1e-10
    assert sparse_ref.max_scaled_rel_err(x, xr, sparse_ref.row_nnz(Ah)) <= 1e-10


@pytest.mark.parametrize("k", [1, 2, 3])
def test_gmres_lucky_breakdown(wk, ex, k):
    """A diagonal matrix with k distinct eigenvalues: the Krylov space is
    exhausted after k steps (||w|| = 0: the next basis scale is never used)
    and GMRES returns the exact solution."""
    n = 64
    vals = [1.0 + (i % k) for i in range(n)]
    m = wk.coo_to_sellp(wk.CooMatrix(n, n, list(range(n)), list(range(n)), vals), 64, ex)
    b = np.ones(n)
    x, hist = wk.gmres_solve(m, b, 1e-14, 50, ex, restart=10)
    x = x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)
    assert len(hist) - 1 == k
    assert np.max(np.abs(x - 1.0 / np.asarray(vals))) <= 1e-14
