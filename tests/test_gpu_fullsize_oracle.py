"""Whole-output parity at BASELINE.json's full sizes against the C oracle.

The C restatement (oracle/csrc/oracle.c) builds every full-size matrix on the
host independently of the device -- stencil generator, CSR -> SELL-P
conversion, R-MAT generator + stable radix sort + duplicate fold -- and folds
SpMV on all host cores. So each device array is compared entry for entry and
each device y over ALL rows, not a sample:

  cfg 1: 5-point Poisson 1000^2   CSR arrays bitwise; y bitwise (every
                                  sequential-fold CSR kernel)
  cfg 2: 27-point 200^3           CSR + SELL-P(64) + ELL arrays bitwise; y bitwise
                                  for SELL-P / ELL / CSR rowblock + stream,
                                  1e-12 scaled for the reassociating CSR kernels
  cfg 3: R-MAT scale 24           raw edges, device radix sort and dedup ->
                                  COO arrays bitwise (268M edges), Hybrid(4)
                                  ELL part + COO remainder bitwise; y: CSR
                                  rowblock bitwise on rows <= 64 entries, COO /
                                  load_balance / merge / Hybrid (and rowblock's
                                  long rows) within 1e-12 scaled
  cfg 4, 5: 7-point 256^3, convection-diffusion 512^3 (the solver operators):
                                  CSR + SELL-P arrays and y bitwise

Tolerance (reassociating kernels): |y - y_ref| <= 1e-12 * max(1, len(row)) *
max(1, |y_ref|) per row, sparse_ref.max_scaled_rel_err.
"""

import numpy as np
import pytest
from types import SimpleNamespace

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import corpus_ref, native, sparse_ref  # noqa: E402

TOL = 1e-12


@pytest.fixture(scope="module")
def wk():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2006_14290_b200 as wk

    return wk


def _h(t):
    return t.cpu().numpy()


def _spmv(d, x):
    from paper_2006_14290_b200 import kernels

    y = kernels.spmv_device(d, x)
    torch.cuda.synchronize()
    return _h(y)


def _x(n, seed):
    x = np.random.default_rng(seed).random(n)
    return x, torch.as_tensor(x, device="cuda")


def _same_csr(dev, host):
    assert np.array_equal(_h(dev.row_ptrs).astype(np.int64), host.row_ptrs)
    assert np.array_equal(_h(dev.col_idx), host.col_idx)
    assert _h(dev.values).tobytes() == host.values.tobytes()


def _entry_pos(ptrs):
    """Position of every CSR entry inside its row."""
    ptrs = np.asarray(ptrs, dtype=np.int64)
    lens = np.diff(ptrs)
    return np.arange(ptrs[-1], dtype=np.int64) - np.repeat(ptrs[:-1], lens)


def _same_ell(ell, csr, width=None):
    """ELL(width, stride) image of a host CSR (sparse.py:233-241 layout with
    one slice of stride n: entry j of row r at j * stride + r, padding (0,
    0.0); entries past `width` excluded)."""
    ptrs = np.asarray(csr.row_ptrs, dtype=np.int64)
    n = len(ptrs) - 1
    lens = np.diff(ptrs)
    w = int(lens.max()) if width is None else int(width)
    assert ell.width == w
    pos = _entry_pos(ptrs)
    rows = np.repeat(np.arange(n, dtype=np.int64), lens)
    m = pos < w
    slot = pos[m] * ell.stride + rows[m]
    col = np.zeros(w * ell.stride, dtype=np.int32)
    val = np.zeros(w * ell.stride, dtype=np.float64)
    col[slot] = np.asarray(csr.col_idx)[m]
    val[slot] = np.asarray(csr.values)[m]
    assert np.array_equal(_h(ell.col_idx)[: w * ell.stride], col)
    assert _h(ell.values)[: w * ell.stride].tobytes() == val.tobytes()
    assert np.array_equal(_h(ell.row_lengths_t).astype(np.int64), np.minimum(lens, w))


def _bitwise(y, ref, what):
    bad = np.flatnonzero(y.view(np.int64) != ref.view(np.int64))
    assert bad.size == 0, f"{what}: {bad.size} rows differ, first {bad[:5]}"


def _close(y, ref, lens, what):
    err = sparse_ref.max_scaled_rel_err(y, ref, lens)
    assert err <= TOL, f"{what}: max scaled rel err {err:.3e}"


def test_cfg1_poisson_1000_whole_vector(wk):
    from paper_2006_14290_b200 import corpus

    A = corpus.poisson2d_matrix(1000)
    H = native.stencil_csr(1000, 1000, 1, corpus_ref.points_5pt())
    _same_csr(A, H)
    x, xd = _x(A.ncols, 1)
    ref = native.Prepared(H).spmv(x)
    for strat in ("auto", "rowblock", "stream"):
        A.with_strategy(strat)
        _bitwise(_spmv(A, xd), ref, strat)
    lens = np.diff(H.row_ptrs)
    for strat in ("load_balance", "merge", "subwarp"):
        A.with_strategy(strat)
        _close(_spmv(A, xd), ref, lens, strat)


def test_cfg2_27pt_200_whole_vector(wk):
    from paper_2006_14290_b200 import corpus
    from paper_2006_14290_b200 import device as D

    A = corpus.stencil3d(200, 27)
    H = native.stencil_csr(200, 200, 200, corpus_ref.points_27pt())
    _same_csr(A, H)
    x, xd = _x(A.ncols, 5)
    ref = native.Prepared(H).spmv(x)
    lens = np.diff(H.row_ptrs)

    sp = D.csr_to_sellp(A, 64)
    hs = native.csr_to_sellp(H, 64)
    assert np.array_equal(_h(sp.slice_sets).astype(np.int64), hs.slice_sets)
    assert np.array_equal(_h(sp.row_lengths_t).astype(np.int64), hs.row_lengths)
    assert np.array_equal(_h(sp.col_idx), hs.col_idx)
    assert _h(sp.values).tobytes() == hs.values.tobytes()
    del hs
    _bitwise(_spmv(sp, xd), ref, "sellp64")
    del sp
    ell = D.csr_to_ell(A)
    _same_ell(ell, H)
    _bitwise(_spmv(ell, xd), ref, "ell")
    del ell
    for strat in ("rowblock", "stream"):
        A.with_strategy(strat)
        _bitwise(_spmv(A, xd), ref, strat)
    for strat in ("load_balance", "merge", "subwarp"):
        A.with_strategy(strat)
        _close(_spmv(A, xd), ref, lens, strat)


def test_cfg3_rmat24_whole_pipeline(wk):
    from paper_2006_14290_b200 import corpus
    from paper_2006_14290_b200 import device as D

    H = native.rmat_coo(24)
    R = corpus.rmat(24)
    assert R.nnz == len(H.values)
    assert np.array_equal(_h(R.row_idx), H.row_idx)
    assert np.array_equal(_h(R.col_idx), H.col_idx)
    assert _h(R.values).tobytes() == H.values.tobytes()

    x, xd = _x(R.ncols, 3)
    hp = native.Prepared(H)
    ref = hp.spmv(x)
    lens = np.bincount(H.row_idx, minlength=H.nrows)
    ptrs = np.concatenate([[0], np.cumsum(lens)])
    hrow, hcol, hval = H.row_idx, H.col_idx, H.values
    del hp, H
    _close(_spmv(R, xd), ref, lens, "coo")
    C = D.coo_to_csr(R)
    C.with_strategy("rowblock")
    # rowblock folds rows of <= 64 entries sequentially per lane (bitwise);
    # longer rows take a warp-wide reduction (csr_tma.cuh, heavy blocks)
    y = _spmv(C, xd)
    short = lens <= 64
    _bitwise(y[short], ref[short], "csr rowblock, rows <= 64")
    _close(y, ref, lens, "csr rowblock")
    for strat in ("load_balance", "merge"):
        C.with_strategy(strat)
        _close(_spmv(C, xd), ref, lens, strat)
    Hy = D.csr_to_hybrid(C, width=4)
    # conversion arrays: the ELL part holds each row's first 4 entries, the COO
    # remainder the rest in row-major order (sparse_ref.csr_to_hybrid)
    _same_ell(Hy.ell, SimpleNamespace(row_ptrs=ptrs, col_idx=hcol, values=hval), width=4)
    keep = _entry_pos(ptrs) >= 4
    assert np.array_equal(_h(Hy.coo.row_idx), hrow[keep])
    assert np.array_equal(_h(Hy.coo.col_idx), hcol[keep])
    assert _h(Hy.coo.values).tobytes() == hval[keep].tobytes()
    _close(_spmv(Hy, xd), ref, lens, "hybrid")


@pytest.mark.parametrize("n,beta", [(256, None), (512, "conv")])
def test_cfg4_cfg5_solver_operators_whole_vector(wk, n, beta):
    """The solver operators of configs 4 (7-point Laplacian 256^3) and 5
    (7-point convection-diffusion 512^3, 134M rows): generator and SELL-P(64)
    arrays entry for entry, operator SpMV bitwise over every row."""
    from paper_2006_14290_b200 import corpus
    from paper_2006_14290_b200 import device as D

    if beta is None:
        A, pts = corpus.stencil3d(n, 7), corpus_ref.points_7pt()
    else:
        A, pts = corpus.convection_diffusion3d(n), corpus_ref.points_7pt(6.0, corpus.CONV_DIFF_BETA)
    H = native.stencil_csr(n, n, n, pts)
    _same_csr(A, H)
    sp = D.csr_to_sellp(A, 64)
    del A
    hs = native.csr_to_sellp(H, 64)
    del H
    assert np.array_equal(_h(sp.slice_sets).astype(np.int64), hs.slice_sets)
    assert np.array_equal(_h(sp.col_idx), hs.col_idx)
    assert _h(sp.values).tobytes() == hs.values.tobytes()
    x, xd = _x(sp.ncols, 11)
    ref = native.Prepared(hs).spmv(x)
    _bitwise(_spmv(sp, xd), ref, f"sellp64 {n}^3")
