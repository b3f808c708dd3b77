"""Generate golden fixtures from the REFERENCE itself (warpkit).

Run in the build container, where the read-only reference is importable:

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py

It imports `warpkit` from /root/reference/pkg/src, builds the matrices with
the reference's own constructors / conversions (`CooMatrix.from_entries`,
`coo_to_csr`, `coo_to_sellp`, corpus generators) and records the reference's
outputs (`dense_spmv_reference`, `cg_solve` on the "reference" executor).
The GPU box has no /root/reference, so the committed `.npz` files are what
the oracle and the CUDA path are pinned against there.
"""

import json
import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

import warpkit  # noqa: E402
from warpkit.corpus import diagonal_matrix, poisson2d_matrix, random_sparse_matrix, tridiagonal_matrix  # noqa: E402
from warpkit.dispatch import make_executor  # noqa: E402
from warpkit.kernels import cg_solve  # noqa: E402
from warpkit.sparse import CooMatrix, coo_to_csr, coo_to_sellp, dense_spmv_reference  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
SLICES = (1, 2, 4, 8, 16, 32, 64)


def spmv_cases():
    rng = np.random.default_rng(1234)
    cases = []
    A = CooMatrix.from_entries(3, 3, [0, 0, 1, 2, 2], [0, 2, 1, 0, 2], [1.0, 2.0, 3.0, 4.0, 5.0])
    cases.append(("hand", A, np.ones(3)))
    cases.append(("identity40", diagonal_matrix(40, 1.0), rng.standard_normal(40)))
    m = random_sparse_matrix(64, 64, 0.3, rng, integer=True)
    cases.append(("int64x64", m, rng.integers(-5, 6, size=64).astype(np.float64)))
    cases.append(("real60", random_sparse_matrix(60, 60, 0.4, rng), rng.random(60)))
    cases.append(("empty_rows", CooMatrix.from_entries(4, 4, [1, 3], [0, 2], [2.0, 5.0]), np.ones(4)))
    cols = np.arange(20)
    cases.append(("long_row", CooMatrix(2, 20, np.zeros(20, dtype=int), cols,
                                        rng.integers(1, 5, 20).astype(float)), np.ones(20)))
    cases.append(("padding65", random_sparse_matrix(65, 65, 0.2, rng), rng.random(65)))
    cases.append(("rect64x48", random_sparse_matrix(64, 48, 0.5, rng), rng.random(48)))
    cases.append(("zero3", CooMatrix(3, 3, [], [], []), np.ones(3)))
    cases.append(("diag48", diagonal_matrix(48), rng.random(48)))
    cases.append(("tridiag48", tridiagonal_matrix(48), rng.random(48)))
    cases.append(("poisson6", poisson2d_matrix(6), rng.random(36)))
    cases.append(("poisson12_normal", poisson2d_matrix(12), rng.standard_normal(144)))
    # explicit zeros and signed values
    zr = CooMatrix.from_entries(5, 5, [0, 0, 1, 2, 3, 3, 4], [0, 3, 1, 4, 0, 2, 4],
                                [0.0, -1.5, 2.25, -0.0, 1e-300, -7.0, 3.0])
    cases.append(("explicit_zeros", zr, np.array([-2.0, 0.5, 1e300, -0.0, 3.0])))
    # duplicate summation order (from_entries, sparse.py:63-80)
    dup = CooMatrix.from_entries(3, 3, [2, 0, 2, 2, 1, 0], [1, 0, 1, 1, 2, 0],
                                 [0.1, 0.2, 0.3, 0.7, 1.0, 1e-17])
    cases.append(("duplicates", dup, rng.random(3)))
    # acceptance-criterion-4 style sweep (test_acceptance.py:173-213)
    rng99 = np.random.default_rng(99)
    for i in range(40):
        nrows = int(rng99.integers(1, 65))
        ncols = int(rng99.integers(1, 65))
        density = float(rng99.random())
        integer = i % 2 == 0
        m = random_sparse_matrix(nrows, ncols, density, rng99, integer=integer)
        x = rng99.integers(-4, 5, size=ncols).astype(float) if integer else rng99.random(ncols)
        cases.append((f"sweep{i:02d}", m, x))
    # a larger power-law-ish matrix with rows far longer than a warp
    rows = np.concatenate([np.zeros(700, int), np.full(300, 5), rng.integers(0, 300, 3000)])
    cols = np.concatenate([np.arange(700), rng.integers(0, 700, 300), rng.integers(0, 700, 3000)])
    cases.append(("skewed300", CooMatrix.from_entries(300, 700, rows, cols, rng.standard_normal(4000)),
                  rng.standard_normal(700)))
    return cases


def write_spmv():
    out = {}
    names = []
    for name, coo, x in spmv_cases():
        names.append(name)
        p = f"{name}__"
        out[p + "shape"] = np.array([coo.nrows, coo.ncols], dtype=np.int64)
        out[p + "row_idx"] = coo.row_idx
        out[p + "col_idx"] = coo.col_idx
        out[p + "values"] = coo.values
        out[p + "x"] = np.asarray(x, dtype=np.float64)
        y = dense_spmv_reference(coo, x)
        out[p + "y"] = y
        csr = coo_to_csr(coo)
        out[p + "csr_row_ptrs"] = csr.row_ptrs
        assert np.array_equal(dense_spmv_reference(csr, x), y)
        for s in SLICES:
            sp = coo_to_sellp(coo, s)
            q = f"{p}sellp{s}_"
            out[q + "slice_sets"] = sp.slice_sets
            out[q + "col_idx"] = sp.col_idx
            out[q + "values"] = sp.values
            out[q + "row_lengths"] = sp.row_lengths
            assert np.array_equal(dense_spmv_reference(sp, x), y)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "spmv_cases.npz"), **out)
    return names


def cg_cases():
    return [
        ("identity3", diagonal_matrix(3, 1.0), np.array([1.0, 2.0, 3.0]), 1e-12, 50),
        ("spd2x2", CooMatrix.from_entries(2, 2, [0, 0, 1, 1], [0, 1, 0, 1], [4.0, 1.0, 1.0, 3.0]),
         np.array([1.0, 2.0]), 1e-12, 10),
        ("poisson10", poisson2d_matrix(10), np.ones(100), 1e-10, 1000),
        ("tridiag24", tridiagonal_matrix(24), np.linspace(1.0, 2.0, 24), 1e-12, 200),
        ("poisson30", poisson2d_matrix(30), np.ones(900), 1e-12, 1000),
        ("poisson40_cap", poisson2d_matrix(40), np.linspace(-1.0, 1.0, 1600), 1e-14, 120),
        ("poisson100", poisson2d_matrix(100), np.ones(10000), 1e-8, 10000),
    ]


def write_cg():
    out = {}
    names = []
    ex = make_executor("ref")
    for name, coo, b, tol, max_iters in cg_cases():
        names.append(name)
        p = f"{name}__"
        sp = coo_to_sellp(coo, 64)
        x, hist = cg_solve(sp, b, tol, max_iters, ex)
        out[p + "shape"] = np.array([coo.nrows, coo.ncols], dtype=np.int64)
        out[p + "row_idx"] = coo.row_idx
        out[p + "col_idx"] = coo.col_idx
        out[p + "values"] = coo.values
        out[p + "b"] = b
        out[p + "params"] = np.array([tol, max_iters], dtype=np.float64)
        out[p + "x"] = x
        out[p + "hist"] = hist
        print(f"cg {name}: {len(hist) - 1} iterations, final {hist[-1]:.3e}")
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "cg_cases.npz"), **out)
    return names


def main():
    spmv_names = write_spmv()
    cg_names = write_cg()
    manifest = {
        "generator": "tests/golden/make_golden.py",
        "reference": "warpkit " + warpkit.__version__ + " from /root/reference/pkg/src",
        "numpy": np.__version__,
        "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS"),
        "spmv_cases": spmv_names,
        "sellp_slice_sizes": list(SLICES),
        "cg_cases": cg_names,
        "cg_slice_size": 64,
    }
    with open(os.path.join(HERE, "manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=1)
        fh.write("\n")


if __name__ == "__main__":
    main()
