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

import io
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


def mm_texts():
    """MatrixMarket inputs: the reference's own test texts (test_sparse.py:149-266)
    plus whitespace / line-ending / literal / symmetry / size edge cases."""
    rng = np.random.default_rng(99)
    H = "%%MatrixMarket matrix coordinate"
    t = {}
    t["diag"] = "\n".join([H + " real general", "3 3 3", "1 1 1.0", "2 2 2.0", "3 3 3.0"])
    t["symmetric"] = "\n".join([H + " real symmetric", "3 3 3", "1 1 2.0", "2 1 5.0", "3 3 1.0"])
    t["pattern"] = "\n".join([H + " pattern general", "2 2 2", "1 1", "2 2"])
    t["integer"] = "\n".join([H + " integer general", "2 2 1", "2 1 7"])
    t["duplicates"] = "\n".join([H + " real general", "2 2 2", "1 1 1.5", "1 1 2.5"])
    t["comments_blank"] = "\n".join([H + " real general", "% a comment", "", "2 2 1", "% another", "1 2 3.0"])
    t["crlf_tabs"] = "\r\n".join([H + " real general", "  3\t3  2 ", "\t1 3\t-4.25  ", "3 1 1e-3", ""])
    t["upper_banner"] = "\n".join(["%%MATRIXMARKET Matrix Coordinate REAL General", "2 3 2", "1 3 2.0", "2 1 -1.0"])
    t["literals"] = "\n".join([H + " real general", "4 4 10", "1 1 +1.5", "1 2 1E5", "1 3 .5", "1 4 5.",
                                "2 1 -0.0", "2 2 4.9e-324", "2 3 1.7976931348623157e308", "2 4 inf",
                                "3 3 -Infinity", "4 4 0.1000000000000000055511151231257827"])
    t["int_literals"] = "\n".join([H + " integer general", "3 3 3", "+1 1 +7", "002 3 -0", "3 002 12345678901"])
    t["empty_matrix"] = H + " real general\n0 0 0\n"
    t["no_final_newline"] = H + " real general\n1 1 1\n1 1 2.5"
    t["cr_only"] = "\r".join([H + " pattern symmetric", "3 3 3", "2 1", "3 3", "3 2"])
    t["sym_diag_dups"] = "\n".join([H + " real symmetric", "3 3 5", "1 1 1.0", "2 1 2.0", "2 1 3.0", "1 1 4.0",
                                     "3 2 0.5"])
    # random general matrix with duplicates, values in repr form
    n, m, k = 300, 200, 3000
    r = rng.integers(1, n + 1, k)
    c = rng.integers(1, m + 1, k)
    v = rng.standard_normal(k) * 10.0 ** rng.integers(-30, 30, k)
    t["random_general"] = H + " real general\n% generated\n" + f"{n} {m} {k}\n" + "".join(
        f"{a} {b} {repr(float(x))}\n" for a, b, x in zip(r, c, v))
    r2 = rng.integers(1, 121, 900)
    c2 = np.minimum(r2, rng.integers(1, 121, 900))
    t["random_symmetric"] = H + " real symmetric\n" + "120 120 900\n" + "".join(
        f"{a} {b} {x!r}\n" for a, b, x in zip(r2, c2, rng.random(900).tolist()))
    errors = {
        "err_complex": H + " complex general\n1 1 1\n1 1 1.0 2.0",
        "err_array": "%%MatrixMarket matrix array real general\n2 2\n1.0\n2.0\n3.0\n4.0",
        "err_skew": H + " real skew-symmetric\n2 2 1\n2 1 1.0",
        "err_hermitian": H + " real hermitian\n2 2 1\n2 1 1.0",
        "err_banner": "%%NotMatrixMarket whatever\n1 1 1\n1 1 1.0",
        "err_banner_short": "%%MatrixMarket matrix coordinate real\n1 1 1\n1 1 1.0",
        "err_count_low": H + " real general\n2 2 2\n1 1 1.0",
        "err_count_high": H + " real general\n2 2 1\n1 1 1.0\n2 2 1.0",
        "err_fields": H + " real general\n2 2 1\n1 x 1.0",
        "err_fields_count": H + " real general\n2 2 1\n1 1",
        "err_pattern_extra": H + " pattern general\n2 2 1\n1 1 1.0",
        "err_bounds": H + " real general\n3 3 1\n4 1 1.0",
        "err_zero_index": H + " real general\n3 3 1\n0 1 1.0",
        "err_size_fields": H + " real general\n3 3\n1 1 1.0",
        "err_negative": H + " real general\n-3 3 0",
        "err_missing_size": H + " real general\n% only a comment\n",
        "err_empty": "",
        "err_float_index": H + " real general\n3 3 1\n1.0 1 1.0",
        "err_bad_value": H + " real general\n3 3 1\n1 1 abc",
        "err_hex_value": H + " real general\n3 3 1\n1 1 0x1p3",
    }
    t.update(errors)
    return t


def write_mm():
    """Record the reference reader's results (or error type) for every text,
    and the reference writer's output for a few matrices."""
    from warpkit.errors import ParseError, UnsupportedFormat
    from warpkit.sparse import read_matrix_market, write_matrix_market

    texts = mm_texts()
    cases = {}
    arrays = {}
    for name, text in texts.items():
        try:
            m = read_matrix_market(text if text else io.BytesIO(b""))
        except (ParseError, UnsupportedFormat) as exc:
            cases[name] = {"text": text, "error": type(exc).__name__}
            continue
        cases[name] = {"text": text, "shape": [m.nrows, m.ncols]}
        arrays[name + "__row_idx"] = np.asarray(m.row_idx, dtype=np.int64)
        arrays[name + "__col_idx"] = np.asarray(m.col_idx, dtype=np.int64)
        arrays[name + "__values"] = np.asarray(m.values, dtype=np.float64)
    # non-ASCII bytes
    try:
        read_matrix_market(io.BytesIO(b"%%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 1.0\xff"))
    except ParseError:
        cases["err_non_ascii"] = {"text_bytes_hex": (b"%%MatrixMarket matrix coordinate real general\n1 1 1\n"
                                                     b"1 1 1.0\xff").hex(), "error": "ParseError"}
    rng = np.random.default_rng(7)
    writes = {}
    for name, (n, m_, dens) in {"w_small": (8, 8, 0.5), "w_rect": (23, 31, 0.2)}.items():
        mm = random_sparse_matrix(n, m_, dens, rng)
        vals = mm.values * np.logspace(-120, 100, mm.nnz) * np.where(np.arange(mm.nnz) % 2, -1, 1)
        mm = CooMatrix(mm.nrows, mm.ncols, mm.row_idx, mm.col_idx, vals)
        writes[name] = write_matrix_market(mm)
        arrays[name + "__row_idx"] = np.asarray(mm.row_idx, dtype=np.int64)
        arrays[name + "__col_idx"] = np.asarray(mm.col_idx, dtype=np.int64)
        arrays[name + "__values"] = np.asarray(mm.values, dtype=np.float64)
        arrays[name + "__shape"] = np.array([mm.nrows, mm.ncols])
    with open(os.path.join(HERE, "mm_cases.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py (mm)", "reads": cases, "writes": writes}, fh, indent=1)
        fh.write("\n")
    np.savez_compressed(os.path.join(HERE, "mm_cases.npz"), **arrays)
    print(f"mm: {len(cases)} read cases, {len(writes)} write cases")


def main():
    if "--only-mm" in sys.argv:
        write_mm()
        return
    spmv_names = write_spmv()
    cg_names = write_cg()
    write_mm()
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
