"""Property-based tests (hypothesis), after the reference's own round-trip
property test of the conversions (pkg/tests/test_sparse.py:135-146, 60
examples): random COO matrices (duplicates, empty rows/columns, explicit
zeros, 0..120 rows), every slice size.

CPU: the oracle's conversions round-trip to the same dense matrix and its
SpMV folds agree bitwise across formats (test_sparse.py:291-300).
GPU: the device conversions (from_entries with duplicate summing, COO->CSR,
CSR->SELL-P / ELL / Hybrid) are bitwise the oracle's, and every SpMV kernel
matches the oracle fold — bitwise for SELL-P / ELL / CSR row-block, within
1e-12 scaled for the reassociating CSR strategies, COO and Hybrid."""

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from oracle import sparse_ref

SLICES = [1, 2, 4, 8, 16, 32, 64]


@st.composite
def coo_matrices(draw):
    nrows = draw(st.integers(0, 120))
    ncols = draw(st.integers(1, 120))
    n = draw(st.integers(0, 400)) if nrows else 0
    rows = draw(st.lists(st.integers(0, max(nrows - 1, 0)), min_size=n, max_size=n))
    cols = draw(st.lists(st.integers(0, ncols - 1), min_size=n, max_size=n))
    ints = draw(st.booleans())
    if ints:
        vals = draw(st.lists(st.integers(-9, 9).map(float), min_size=n, max_size=n))
    else:
        vals = draw(st.lists(st.floats(-1e3, 1e3, allow_nan=False, width=64), min_size=n, max_size=n))
    seed = draw(st.integers(0, 2**31 - 1))
    return nrows, ncols, rows, cols, vals, ints, seed


@settings(max_examples=60, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(coo_matrices(), st.sampled_from(SLICES))
def test_oracle_round_trip(m, ss):
    nrows, ncols, rows, cols, vals, ints, seed = m
    coo = sparse_ref.coo_from_entries(nrows, ncols, rows, cols, vals)
    csr = sparse_ref.coo_to_csr(coo)
    sp = sparse_ref.csr_to_sellp(csr, ss)
    dense = sparse_ref.to_dense(coo)
    assert np.array_equal(sparse_ref.to_dense(csr), dense)
    assert np.array_equal(sparse_ref.to_dense(sp), dense)
    x = np.random.default_rng(seed).standard_normal(ncols)
    y = sparse_ref.spmv(csr, x)
    assert sparse_ref.spmv(sp, x).tobytes() == y.tobytes()
    assert sparse_ref.spmv(coo, x).tobytes() == y.tobytes()
    assert sparse_ref.spmv(sparse_ref.csr_to_ell(csr), x).tobytes() == y.tobytes()


@pytest.mark.gpu
@settings(max_examples=60, deadline=None, suppress_health_check=[HealthCheck.too_slow,
                                                                 HealthCheck.function_scoped_fixture])
@given(m=coo_matrices(), ss=st.sampled_from(SLICES))
def test_device_conversions_and_spmv(m, ss):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2006_14290_b200 as wk

    nrows, ncols, rows, cols, vals, ints, seed = m
    ex = wk.make_executor("b200", device=0)
    ref_coo = sparse_ref.coo_from_entries(nrows, ncols, rows, cols, vals)
    coo = wk.CooMatrix.from_entries(nrows, ncols, np.asarray(rows, np.int64), np.asarray(cols, np.int64),
                                    np.asarray(vals, np.float64))
    H = lambda a: a.to_host() if hasattr(a, "to_host") else a  # noqa: E731
    ch = H(coo)
    assert np.array_equal(np.asarray(ch.row_idx, np.int64), ref_coo.row_idx)
    assert np.array_equal(np.asarray(ch.col_idx, np.int64), ref_coo.col_idx)
    assert np.asarray(ch.values, np.float64).tobytes() == ref_coo.values.tobytes()
    ref_csr = sparse_ref.coo_to_csr(ref_coo)
    csr = wk.coo_to_csr(coo, ex)
    assert np.array_equal(np.asarray(H(csr).row_ptrs, np.int64), ref_csr.row_ptrs)
    sp = wk.coo_to_sellp(coo, ss, ex)
    sh = H(sp)
    ref_sp = sparse_ref.csr_to_sellp(ref_csr, ss)
    assert np.array_equal(np.asarray(sh.slice_sets, np.int64), ref_sp.slice_sets)
    assert np.array_equal(np.asarray(sh.col_idx, np.int64), ref_sp.col_idx)
    assert np.asarray(sh.values, np.float64).tobytes() == ref_sp.values.tobytes()
    if nrows == 0:
        return
    rng = np.random.default_rng(seed)
    x = rng.integers(-5, 6, size=ncols).astype(np.float64) if ints else rng.standard_normal(ncols)
    y_ref = sparse_ref.spmv(ref_csr, x)
    lens = sparse_ref.row_nnz(ref_csr)
    asnp = lambda v: v.cpu().numpy() if hasattr(v, "cpu") else np.asarray(v)  # noqa: E731
    assert asnp(wk.spmv_sellp(sp, x, ex)).tobytes() == y_ref.tobytes()
    ell = wk.csr_to_ell(csr, exec=ex)
    assert asnp(wk.spmv_ell(ell, x, ex)).tobytes() == y_ref.tobytes()
    outs = []
    for strat in ("rowblock", "load_balance", "merge", "stream", "subwarp"):
        e = wk.make_executor("b200", device=0, tuning={"csr_strategy": strat})
        y = asnp(wk.spmv_csr(csr, x, e))
        if strat == "rowblock":  # rows of <= 64 entries: the lane's sequential fold
            short = lens <= 64
            assert y[short].tobytes() == y_ref[short].tobytes()
        outs.append(y)
    outs.append(asnp(wk.spmv_coo(coo, x, ex)))
    outs.append(asnp(wk.spmv_hybrid(wk.csr_to_hybrid(csr, width=2, exec=ex), x, ex)))
    for y in outs:
        if ints:
            assert np.array_equal(y, y_ref)
        else:
            assert sparse_ref.max_scaled_rel_err(y, y_ref, lens) <= 1e-12


@st.composite
def spd_systems(draw):
    """Random sparse symmetric strictly diagonally dominant (hence SPD) systems."""
    n = draw(st.integers(1, 300))
    m = draw(st.integers(0, 4 * n))
    i = draw(st.lists(st.integers(0, n - 1), min_size=m, max_size=m))
    j = draw(st.lists(st.integers(0, n - 1), min_size=m, max_size=m))
    v = draw(st.lists(st.floats(-1.0, 1.0, allow_nan=False, width=64), min_size=m, max_size=m))
    seed = draw(st.integers(0, 2**31 - 1))
    return n, i, j, v, seed


@pytest.mark.gpu
@settings(max_examples=30, deadline=None, suppress_health_check=[HealthCheck.too_slow,
                                                                 HealthCheck.function_scoped_fixture])
@given(sys_=spd_systems(), fmt=st.sampled_from(["sellp", "csr", "ell"]))
def test_cg_random_spd(sys_, fmt):
    """CG (wk_cg_solve: device loop, CUDA graph, L2 ping-pong) on random SPD
    systems against the oracle CG (kernels.py:283-331 update order): same
    starting residual, converged to the tolerance, iteration counts within
    one (dot summation orders differ), solutions within 1e-8."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2006_14290_b200 as wk
    from oracle import krylov_ref

    n, i, j, v, seed = sys_
    rows = np.concatenate([np.asarray(i, np.int64), np.asarray(j, np.int64), np.arange(n)])
    cols = np.concatenate([np.asarray(j, np.int64), np.asarray(i, np.int64), np.arange(n)])
    vals = np.concatenate([np.asarray(v), np.asarray(v), np.zeros(n)])
    off = np.zeros(n)
    np.add.at(off, rows[: 2 * len(i)], np.abs(vals[: 2 * len(i)]))
    vals[2 * len(i):] = off + 1.0  # strict diagonal dominance
    ref_coo = sparse_ref.coo_from_entries(n, n, rows, cols, vals)
    ref_csr = sparse_ref.coo_to_csr(ref_coo)
    ex = wk.make_executor("b200", device=0)
    coo = wk.CooMatrix(n, n, ref_coo.row_idx, ref_coo.col_idx, ref_coo.values)
    A = {"sellp": lambda: wk.coo_to_sellp(coo, 64, ex), "csr": lambda: wk.coo_to_csr(coo, ex),
         "ell": lambda: wk.csr_to_ell(wk.coo_to_csr(coo, ex), exec=ex)}[fmt]()
    b = np.random.default_rng(seed).standard_normal(n)
    tol = 1e-10
    x, hist = wk.cg_solve(A, b, tol, 1000, ex)
    xr, hr = krylov_ref.cg_solve(lambda z: sparse_ref.spmv(ref_csr, z), b, tol, 1000)
    x = x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)
    hist = hist.cpu().numpy() if hasattr(hist, "cpu") else np.asarray(hist)
    assert abs(hist[0] - hr[0]) <= 1e-14 * hr[0]
    assert abs(len(hist) - len(hr)) <= 1
    bn = float(np.linalg.norm(b))
    assert hist[-1] <= tol * bn or len(hist) - 1 == 1000
    assert np.max(np.abs(x - xr)) <= 1e-8 * max(1.0, float(np.max(np.abs(xr))))
