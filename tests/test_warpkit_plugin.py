"""Drop-in into the reference's own registry and harness.

The reference package (`warpkit`) is importable from `baseline/_ref` (the
offline install of /root/reference, git-ignored, shipped to the GPU box) or,
in the build container, from /root/reference/pkg/src. Without either, these
tests skip. CPU part: registration only. GPU part: warpkit's own public
functions and its benchmark harness (`run_benchmark`, which checks every
result against warpkit's sequential oracle) run on the b200 executor."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for cand in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(cand, "warpkit")) and cand not in sys.path:
        sys.path.append(cand)
        break

warpkit = pytest.importorskip("warpkit")


@pytest.fixture(scope="module")
def installed():
    from paper_2006_14290_b200 import warpkit_plugin

    return warpkit_plugin.install(warpkit)


def test_registration(installed):
    import importlib

    wd = importlib.import_module("warpkit.dispatch")

    assert "b200" in wd.EXEC_KINDS
    ex = wd.make_executor("b200")
    assert ex.kind == "b200"
    for name in ("spmv_coo", "spmv_csr", "spmv_sellp", "cg", "reduce_microbench"):
        assert wd.get_operation(name).impls["b200"] is not None
    # the reference's own executors are untouched
    assert wd.make_executor("ref").kind == "reference"
    from warpkit.bench import BenchConfig

    BenchConfig(corpus=".", execs=("ref", "b200"))  # accepted by the harness' validation


@pytest.mark.gpu
def test_reference_api_on_b200(installed):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from warpkit.corpus import poisson2d_matrix, random_sparse_matrix
    from warpkit.kernels import cg_solve, spmv_coo, spmv_csr, spmv_sellp
    from warpkit.sparse import coo_to_csr, coo_to_sellp, dense_spmv_reference

    ex = warpkit.make_executor("b200")
    ref = warpkit.make_executor("ref")
    rng = np.random.default_rng(1234)
    m = random_sparse_matrix(80, 80, 0.2, rng)
    x = rng.random(80)
    y = dense_spmv_reference(m, x)
    assert np.array_equal(spmv_sellp(coo_to_sellp(m, 64), x, ex), y)
    assert np.array_equal(spmv_csr(coo_to_csr(m), x, ex), y)
    assert np.max(np.abs(spmv_coo(m, x, ex) - y)) <= 1e-12 * max(1.0, np.abs(y).max()) * 80
    assert ex.counters.lane_steps == m.nnz
    sp = coo_to_sellp(poisson2d_matrix(12), 64)
    b = np.ones(sp.nrows)
    xr, hr = cg_solve(sp, b, 1e-10, 500, ref)
    xg, hg = warpkit.dispatch("cg", ex, sp, b, 1e-10, 500)
    assert len(hg) == len(hr)
    assert np.max(np.abs(hg - hr)) / np.linalg.norm(b) <= 1e-10
    for size in (4, 8, 32):  # the reduction microbenchmark runs on the GPU now
        assert np.array_equal(warpkit.dispatch("reduce_microbench", ex, size, 10),
                              warpkit.dispatch("reduce_microbench", ref, size, 10))


@pytest.mark.gpu
def test_reference_harness_on_b200(installed, tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from warpkit.bench import BenchConfig, run_benchmark
    from warpkit.corpus import generate_corpus

    generate_corpus(tmp_path)
    cfg = BenchConfig(corpus=tmp_path, kernels=("coo", "csr", "sellp", "cg"), execs=("ref", "b200"),
                      warmup_iters=1, timed_iters=2)
    res = run_benchmark(cfg)
    rows = [r for r in res.records if r.exec == "b200"]
    assert rows, "no b200 records"
    bad = [(r.matrix, r.kernel, r.max_rel_err) for r in rows if not r.correct]
    assert not bad, bad


def test_plugin_raises_warpkit_errors(installed):
    """With the b200 slot installed, warpkit's own entry points still raise
    warpkit.errors classes (the checks run before any device work)."""
    from warpkit.corpus import poisson2d_matrix
    from warpkit.kernels import spmv_coo, spmv_csr, spmv_sellp
    from warpkit.sparse import coo_to_csr, coo_to_sellp

    ex = warpkit.make_executor("b200")
    m = poisson2d_matrix(4)
    for fn, mm in ((spmv_coo, m), (spmv_csr, coo_to_csr(m)), (spmv_sellp, coo_to_sellp(m, 4))):
        with pytest.raises(warpkit.errors.DimensionMismatch):
            fn(mm, np.ones(m.ncols + 1), ex)
    with pytest.raises(warpkit.errors.DimensionMismatch):
        warpkit.dispatch("cg", ex, coo_to_sellp(m, 4), np.ones(3), 1e-8, 10)
    with pytest.raises(ValueError):
        warpkit.dispatch("cg", ex, coo_to_sellp(m, 4), np.ones(m.nrows), 0.0, 10)


@pytest.mark.gpu
def test_plugin_breakdown_is_warpkit_breakdown(installed):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from warpkit.sparse import CooMatrix, coo_to_sellp

    # indefinite: p.Ap < 0 at the first iteration (kernels.py:317-318)
    m = CooMatrix.from_entries(2, 2, [0, 1], [0, 1], [-1.0, -2.0])
    with pytest.raises(warpkit.errors.BreakdownError):
        warpkit.dispatch("cg", warpkit.make_executor("b200"), coo_to_sellp(m, 2), np.ones(2), 1e-8, 10)


@pytest.mark.gpu
def test_reference_cli_strict_on_b200(installed, tmp_path):
    """The reference's own command line (bench.py:434-500) with the b200
    executor: --strict exits 0 only if every record validates against the
    reference oracle, and results.csv carries the b200 rows."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import csv

    from warpkit.bench import main
    from warpkit.corpus import generate_corpus

    corpus, out = tmp_path / "corpus", tmp_path / "out"
    corpus.mkdir()
    generate_corpus(corpus)
    rc = main(["--corpus", str(corpus), "--out", str(out), "--execs", "ref,b200", "--kernels", "coo,csr,sellp,cg",
               "--warmup", "1", "--iters", "2", "--strict"])
    assert rc == 0
    with open(out / "results.csv") as fh:
        rows = list(csv.DictReader(fh))
    b200 = [r for r in rows if r.get("exec") == "b200"]
    assert b200 and {r["kernel"] for r in b200} == {"coo", "csr", "sellp", "cg"}
    assert all(r["correct"] in ("True", "true", "1") for r in b200), [r for r in b200 if r["correct"] not in ("True", "true", "1")]
