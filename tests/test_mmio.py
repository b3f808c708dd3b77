"""MatrixMarket ingestion: the native parser
(csrc/mmio.cpp through the C ABI) against the reference reader's own results
(tests/golden/mm_cases.json, written by warpkit) and the line-by-line oracle
restatement (oracle/mm_ref.py).

CPU tests pin the parse (triplets in file order + the oracle's duplicate sum)
and the writer; the GPU test runs the full product path, whose duplicate sum
is the device sort + fold."""

import io
import json
import os

import numpy as np
import pytest

from oracle import mm_ref, sparse_ref
from tests.golden_io import GOLDEN

wk = pytest.importorskip("paper_2006_14290_b200")

with open(os.path.join(GOLDEN, "mm_cases.json")) as _fh:
    MM = json.load(_fh)
ARR = np.load(os.path.join(GOLDEN, "mm_cases.npz"))
READS = MM["reads"]
OK = sorted(k for k, v in READS.items() if "error" not in v)
ERR = sorted(k for k, v in READS.items() if "error" in v)


def _text(case):
    if "text_bytes_hex" in case:
        return bytes.fromhex(case["text_bytes_hex"])
    return case["text"]


def _golden(name):
    return ARR[name + "__row_idx"], ARR[name + "__col_idx"], ARR[name + "__values"]


@pytest.mark.parametrize("name", OK)
def test_oracle_matches_reference_reader(name):
    m = mm_ref.read(_text(READS[name]))
    r, c, v = _golden(name)
    assert [m.nrows, m.ncols] == READS[name]["shape"]
    assert np.array_equal(m.row_idx, r) and np.array_equal(m.col_idx, c)
    assert m.values.tobytes() == v.tobytes()


@pytest.mark.parametrize("name", OK)
def test_native_parse_matches_reference(name):
    text = _text(READS[name])
    nrows, ncols, rows, cols, vals = wk.read_matrix_market_entries(text)
    er = mm_ref.read_entries(text)
    assert (nrows, ncols) == (er[0], er[1])
    assert rows.tolist() == er[2] and cols.tolist() == er[3]
    assert vals.tobytes() == np.asarray(er[4], dtype=np.float64).tobytes()
    m = sparse_ref.coo_from_entries(nrows, ncols, rows, cols, vals)
    r, c, v = _golden(name)
    assert np.array_equal(m.row_idx, r) and np.array_equal(m.col_idx, c)
    assert m.values.tobytes() == v.tobytes()


@pytest.mark.parametrize("name", ERR)
def test_native_errors_match_reference(name):
    case = READS[name]
    exc = {"ParseError": wk.ParseError, "UnsupportedFormat": wk.UnsupportedFormat}[case["error"]]
    with pytest.raises(exc):
        wk.read_matrix_market_entries(_text(case))
    with pytest.raises(mm_ref.MMError) as info:
        mm_ref.read_entries(_text(case))
    assert info.value.kind == case["error"]


@pytest.mark.parametrize("name", sorted(MM["writes"]))
def test_writer_matches_reference_text(name):
    m = wk.CooMatrix(int(ARR[name + "__shape"][0]), int(ARR[name + "__shape"][1]), ARR[name + "__row_idx"],
                     ARR[name + "__col_idx"], ARR[name + "__values"])
    assert wk.write_matrix_market(m) == MM["writes"][name]
    assert mm_ref.write(m) == MM["writes"][name]


def test_sources(tmp_path):
    text = READS["symmetric"]["text"]
    want = wk.read_matrix_market_entries(text)
    path = tmp_path / "a.mtx"
    path.write_text(text)
    for src in (str(path), path, text.encode(), io.BytesIO(text.encode()), io.StringIO(text)):
        got = wk.read_matrix_market_entries(src)
        assert got[:2] == want[:2] and np.array_equal(got[2], want[2]) and np.array_equal(got[4], want[4])
    out = io.StringIO()
    m = wk.CooMatrix(2, 2, [0, 1], [1, 0], [0.5, -2.0])
    assert wk.write_matrix_market(m, out) == out.getvalue()
    wk.write_matrix_market(m, tmp_path / "b.mtx")
    assert (tmp_path / "b.mtx").read_text() == out.getvalue()


@pytest.mark.parametrize("nthreads", [1, 3, 8])
@pytest.mark.parametrize("eol", ["\n", "\r\n", "\r"])
def test_threaded_parse_large(rng, nthreads, eol):
    """Multi-megabyte body: chunk cuts at line boundaries (incl. CRLF pairs),
    comments / blank lines inside the body, symmetric mirrors; the entry
    error reported is the first in file order."""
    n, k = 5000, 200000
    r = rng.integers(1, n + 1, k)
    c = np.minimum(r, rng.integers(1, n + 1, k))
    v = rng.standard_normal(k)
    lines = [f"{a} {b} {x!r}" for a, b, x in zip(r.tolist(), c.tolist(), v.tolist())]
    for pos in (10, 50000, 123457):
        lines.insert(pos, "% comment inside the body")
        lines.insert(pos, "   ")
    text = eol.join(["%%MatrixMarket matrix coordinate real symmetric", f"{n} {n} {k}"] + lines) + eol
    got = wk.read_matrix_market_entries(text, nthreads=nthreads)
    want = mm_ref.read_entries(text)
    assert np.array_equal(got[2], want[2]) and np.array_equal(got[3], want[3])
    assert got[4].tobytes() == np.asarray(want[4]).tobytes()
    # two bad lines: the earlier one is reported
    bad = list(lines)
    bad[150000] = "1 2 x"
    bad[160000] = "9999999 1 1.0"
    text = eol.join(["%%MatrixMarket matrix coordinate real symmetric", f"{n} {n} {k}"] + bad)
    with pytest.raises(wk.ParseError, match="line 150003"):
        wk.read_matrix_market_entries(text, nthreads=nthreads)


@pytest.mark.gpu
@pytest.mark.parametrize("name", OK)
def test_read_matrix_market_device_path(name):
    """Full product path: native parse + device sort / duplicate fold."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    m = wk.read_matrix_market(_text(READS[name]))
    r, c, v = _golden(name)
    assert [m.nrows, m.ncols] == READS[name]["shape"]
    assert np.array_equal(m.row_idx, r) and np.array_equal(m.col_idx, c)
    assert m.values.tobytes() == v.tobytes()
    d = wk.read_matrix_market(_text(READS[name]), device=0)
    h = d.to_host()
    assert np.array_equal(h.row_idx, r) and h.values.tobytes() == v.tobytes()
