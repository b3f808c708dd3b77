"""CPU oracle (TEST INFRASTRUCTURE ONLY): MatrixMarket coordinate reader and
writer of the reference `warpkit.sparse` (sparse.py:269-354), restated line
by line in plain Python for the parity tests of the native parser
(`paper_2006_14290_b200/csrc/mmio.cpp`). Pinned against the reference's own
outputs in `tests/golden/mm_cases.json` (tests/golden/make_golden.py).

`read_entries` stops before `CooMatrix.from_entries` (the triplets in file
order, symmetric mirrors interleaved); `read` adds the duplicate sum
(`sparse_ref.coo_from_entries`, the `np.add.at` order of sparse.py:73-79).
Errors are reported as ("ParseError" | "UnsupportedFormat", message).
"""

from . import sparse_ref


class MMError(Exception):
    def __init__(self, kind, msg):
        super().__init__(msg)
        self.kind = kind


def read_entries(text):
    """sparse.py:269-335 without the final from_entries."""
    if isinstance(text, bytes):
        try:
            text = text.decode("ascii")
        except UnicodeDecodeError as exc:  # sparse.py:277-280
            raise MMError("ParseError", str(exc))
    lines = text.splitlines()
    if not lines:  # sparse.py:282-283
        raise MMError("ParseError", "empty MatrixMarket stream")
    banner = lines[0].strip().lower().split()  # sparse.py:284-286
    if len(banner) != 5 or banner[0] != "%%matrixmarket" or banner[1] != "matrix":
        raise MMError("ParseError", "malformed banner")
    layout, field, symmetry = banner[2], banner[3], banner[4]
    if layout != "coordinate":  # sparse.py:288-293
        raise MMError("UnsupportedFormat", layout)
    if field not in ("real", "integer", "pattern"):
        raise MMError("UnsupportedFormat", field)
    if symmetry not in ("general", "symmetric"):
        raise MMError("UnsupportedFormat", symmetry)
    body = [(n, ln) for n, ln in enumerate(lines[1:], start=2) if ln.strip() and not ln.lstrip().startswith("%")]
    if not body:  # sparse.py:299-300
        raise MMError("ParseError", "missing size line")
    size_no, size_line = body[0]
    parts = size_line.split()
    if len(parts) != 3:  # sparse.py:302-303
        raise MMError("ParseError", f"line {size_no}: size line")
    try:
        nrows, ncols, nnz = (int(p) for p in parts)
    except ValueError:
        raise MMError("ParseError", f"line {size_no}: size literal")
    if nrows < 0 or ncols < 0 or nnz < 0:
        raise MMError("ParseError", f"line {size_no}: negative size")
    entries = body[1:]
    if len(entries) != nnz:  # sparse.py:311-312
        raise MMError("ParseError", f"expected {nnz} entries, found {len(entries)}")
    pattern = field == "pattern"
    want = 2 if pattern else 3
    rows, cols, vals = [], [], []
    for line_no, ln in entries:  # sparse.py:316-334
        p = ln.split()
        if len(p) != want:
            raise MMError("ParseError", f"line {line_no}: fields")
        try:
            i, j = int(p[0]), int(p[1])
            v = 1.0 if pattern else float(p[2])
        except ValueError:
            raise MMError("ParseError", f"line {line_no}: literal")
        if not (1 <= i <= nrows and 1 <= j <= ncols):
            raise MMError("ParseError", f"line {line_no}: bounds")
        rows.append(i - 1)
        cols.append(j - 1)
        vals.append(v)
        if symmetry == "symmetric" and i != j:
            rows.append(j - 1)
            cols.append(i - 1)
            vals.append(v)
    return nrows, ncols, rows, cols, vals


def read(text):
    nrows, ncols, rows, cols, vals = read_entries(text)
    return sparse_ref.coo_from_entries(nrows, ncols, rows, cols, vals)


def write(m):
    """sparse.py:338-353."""
    out = ["%%MatrixMarket matrix coordinate real general\n", f"{m.nrows} {m.ncols} {len(m.values)}\n"]
    for r, c, v in zip(m.row_idx, m.col_idx, m.values):
        out.append(f"{int(r) + 1} {int(c) + 1} {float(v):.17g}\n")
    return "".join(out)
