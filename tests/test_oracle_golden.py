"""Pin the CPU oracle against golden vectors produced by the reference
(warpkit) itself. CPU only: this is what makes the oracle trustworthy before
it is used to judge the CUDA path."""

import numpy as np
import pytest

from oracle import corpus_ref, krylov_ref, sparse_ref
from tests import golden_io

SPMV = golden_io.spmv_cases()
CG = golden_io.cg_cases()


@pytest.mark.parametrize("case", SPMV, ids=[c.name for c in SPMV])
def test_conversions_bit_exact(case):
    csr = sparse_ref.coo_to_csr(case.coo)
    assert np.array_equal(csr.row_ptrs, case.csr.row_ptrs)
    assert np.array_equal(csr.col_idx, case.coo.col_idx)
    for s, ref in case.sellp.items():
        got = sparse_ref.csr_to_sellp(csr, s)
        for field in ("slice_sets", "col_idx", "values", "row_lengths"):
            a, b = getattr(got, field), getattr(ref, field)
            assert a.dtype == b.dtype, field
            assert np.array_equal(a, b), (s, field)
        # byte-level equality of the values, signed zeros included
        assert got.values.tobytes() == ref.values.tobytes()


@pytest.mark.parametrize("case", SPMV, ids=[c.name for c in SPMV])
def test_spmv_fold_bitwise(case):
    y = case.y
    assert sparse_ref.spmv(case.coo, case.x).tobytes() == y.tobytes()
    assert sparse_ref.spmv(case.csr, case.x).tobytes() == y.tobytes()
    for s, sp in case.sellp.items():
        assert sparse_ref.spmv(sp, case.x).tobytes() == y.tobytes()
    assert sparse_ref.spmv_loop(case.csr, case.x).tobytes() == y.tobytes()


@pytest.mark.parametrize("case", SPMV, ids=[c.name for c in SPMV])
def test_ell_and_hybrid_restatements_fold_like_csr(case):
    # parity unpinned by the reference (no ELL/Hybrid there), but both are
    # defined to fold each row in column order, so they must equal the
    # reference's CSR result bitwise.
    ell = sparse_ref.csr_to_ell(case.csr)
    assert sparse_ref.spmv(ell, case.x).tobytes() == case.y.tobytes()
    assert np.array_equal(sparse_ref.to_dense(ell), sparse_ref.to_dense(case.csr))
    for k in (0, 1, 3):
        hyb = sparse_ref.csr_to_hybrid(case.csr, k)
        assert sparse_ref.spmv(hyb, case.x).tobytes() == case.y.tobytes()
        assert np.array_equal(sparse_ref.to_dense(hyb), sparse_ref.to_dense(case.csr))


def test_from_entries_duplicate_order():
    case = next(c for c in SPMV if c.name == "duplicates")
    # rebuild from the raw triplets used in make_golden.py
    m = sparse_ref.coo_from_entries(3, 3, [2, 0, 2, 2, 1, 0], [1, 0, 1, 1, 2, 0],
                                    [0.1, 0.2, 0.3, 0.7, 1.0, 1e-17])
    assert np.array_equal(m.row_idx, case.coo.row_idx)
    assert m.values.tobytes() == case.coo.values.tobytes()


@pytest.mark.parametrize("case", CG, ids=[c.name for c in CG])
def test_cg_restatement_bitwise(case):
    sp = sparse_ref.csr_to_sellp(sparse_ref.coo_to_csr(case.coo), 64)
    x, hist = krylov_ref.cg_solve(lambda v: sparse_ref.spmv(sp, v), case.b, case.tol, case.max_iters)
    assert len(hist) == len(case.hist)
    # OPENBLAS_NUM_THREADS may differ from the fixture's (1) in this process,
    # and ddot's summation order depends on it -> tolerance,
    # normalised by ||b|| as in BASELINE.md §2.
    bn = max(np.linalg.norm(case.b), 1.0)
    assert np.max(np.abs(hist - case.hist)) / bn <= 1e-12
    assert sparse_ref.max_scaled_rel_err(x, case.x, np.full(len(x), 5)) <= 1e-12


def test_generators_match_reference_corpus():
    z = np.load(golden_io.os.path.join(golden_io.GOLDEN, "spmv_cases.npz"))
    for name, gen in (("poisson6", corpus_ref.poisson2d(6)), ("tridiag48", corpus_ref.tridiagonal(48))):
        assert np.array_equal(gen.col_idx, z[f"{name}__col_idx"])
        assert np.array_equal(gen.values, z[f"{name}__values"])
        assert np.array_equal(gen.row_ptrs, z[f"{name}__csr_row_ptrs"])


def test_c_oracle_matches_numpy_oracle(rng):
    from oracle import native
    m = corpus_ref.stencil(9, 7, 5, corpus_ref.points_27pt())
    x = rng.standard_normal(m.ncols)
    y = sparse_ref.spmv(m, x)
    assert native.Prepared(m).spmv(x).tobytes() == y.tobytes()
    sp = sparse_ref.csr_to_sellp(m, 32)
    assert native.Prepared(sp).spmv(x).tobytes() == y.tobytes()
    ell = sparse_ref.csr_to_ell(m)
    assert native.Prepared(ell).spmv(x).tobytes() == y.tobytes()
    coo = sparse_ref.csr_to_coo(m)
    assert native.Prepared(coo).spmv(x, nthreads=3).tobytes() == y.tobytes()
    case = next(c for c in CG if c.name == "poisson30")
    sp = sparse_ref.csr_to_sellp(sparse_ref.coo_to_csr(case.coo), 64)
    xs, hist = native.Prepared(sp).cg(case.b, case.tol, case.max_iters, nthreads=1)
    assert len(hist) == len(case.hist)
    assert np.max(np.abs(hist - case.hist)) / np.linalg.norm(case.b) <= 1e-12


def test_bicgstab_and_gmres_restatements_solve():
    # unpinned by the reference: check they actually solve a nonsymmetric
    # convection-diffusion system and report consistent histories
    m = corpus_ref.stencil(8, 8, 8, corpus_ref.points_7pt(beta=(1.0, 0.5, 0.25)))
    b = np.ones(m.nrows)
    A = sparse_ref.to_dense(m)
    xs = np.linalg.solve(A, b)
    f = lambda v: sparse_ref.spmv(m, v)  # noqa: E731
    x, hist = krylov_ref.bicgstab_solve(f, b, 1e-10, 500)
    assert hist[-1] <= 1e-10 * np.linalg.norm(b)
    assert np.max(np.abs(x - xs)) <= 1e-8
    x, hist = krylov_ref.gmres_solve(f, b, 1e-10, 2000, restart=30)
    assert hist[-1] <= 1e-10 * np.linalg.norm(b)
    assert np.max(np.abs(x - xs)) <= 1e-8
    assert np.isclose(hist[-1], np.linalg.norm(b - A @ x), rtol=1e-6, atol=1e-14)


def test_rmat_generator_statistics():
    m = corpus_ref.rmat(10, edge_factor=8)
    assert m.nrows == 1024
    keys = m.row_idx * m.ncols + m.col_idx
    assert np.all(np.diff(keys) > 0)
    counts = np.bincount(m.row_idx, minlength=m.nrows)
    # skew: quadrant a=0.57 concentrates edges on low row indices
    assert counts[:256].sum() > counts[768:].sum() * 4


def test_c_generators_equal_numpy_restatements():
    """oracle.native.stencil_csr / csr_to_sellp (the C builders of the
    full-size CPU baseline) equal corpus_ref.stencil / sparse_ref.csr_to_sellp
    (sparse.py:219-242) exactly."""
    from oracle import corpus_ref, native, sparse_ref

    cases = [(7, 5, 6, corpus_ref.points_27pt(), 0, None),
             (9, 8, 7, corpus_ref.points_7pt(beta=(1.0, 0.5, 0.25)), 50, 300),
             (30, 1, 1, corpus_ref.points_5pt(), 0, None)]
    for nx, ny, nz, pts, lo, hi in cases:
        a = native.stencil_csr(nx, ny, nz, pts, lo, hi)
        b = corpus_ref.stencil(nx, ny, nz, pts, lo, hi)
        assert np.array_equal(a.row_ptrs, b.row_ptrs) and np.array_equal(a.col_idx, b.col_idx)
        assert a.values.tobytes() == b.values.tobytes()
        for ss in (1, 4, 64):
            sa, sb = native.csr_to_sellp(a, ss), sparse_ref.csr_to_sellp(b, ss)
            for k in ("slice_sets", "col_idx", "row_lengths"):
                assert np.array_equal(getattr(sa, k), getattr(sb, k)), k
            assert sa.values.tobytes() == sb.values.tobytes()


def test_c_rmat_pipeline_equals_numpy_restatement():
    """oracle.native.rmat_coo (the C R-MAT generator + stable radix sort +
    duplicate fold used by the full-size config-3 parity test) equals
    corpus_ref.rmat (np.lexsort + np.add.at, sparse.py:63-80) entry for entry."""
    from oracle import native

    for scale, ef, seed in ((6, 16, 42), (11, 8, 7), (13, 16, 42)):
        a = native.rmat_coo(scale, ef, seed=seed)
        b = corpus_ref.rmat(scale, ef, seed=seed)
        assert np.array_equal(a.row_idx, b.row_idx) and np.array_equal(a.col_idx, b.col_idx)
        assert a.values.tobytes() == b.values.tobytes()


@pytest.mark.parametrize("nthreads", [1, 3, 8])
def test_c_sort_pairs_is_stable(nthreads):
    from oracle import native

    rng = np.random.default_rng(nthreads)
    for n, bits in ((0, 8), (1, 16), (1000, 10), (100_003, 40), (50_000, 64)):
        k = rng.integers(0, 1 << min(bits, 62), n, dtype=np.int64)
        if bits == 64:
            k = k ^ (rng.integers(0, 2, n, dtype=np.int64) << 63)  # negative keys sort as u64
        k[: n // 3] = k[n // 3: 2 * (n // 3)]  # duplicates
        v = rng.random(n)
        order = np.argsort(k.view(np.uint64), kind="stable")
        ks, vs = native.sort_pairs(k.copy(), v.copy(), bits, nthreads)
        assert np.array_equal(ks, k[order]) and vs.tobytes() == v[order].tobytes()
