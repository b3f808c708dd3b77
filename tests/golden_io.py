"""Loader for the golden fixtures written by tests/golden/make_golden.py."""

import os
from types import SimpleNamespace

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SLICES = (1, 2, 4, 8, 16, 32, 64)


def _load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def spmv_cases():
    z = _load("spmv_cases.npz")
    out = []
    for name in z["names"].tolist():
        p = f"{name}__"
        nrows, ncols = (int(v) for v in z[p + "shape"])
        coo = SimpleNamespace(nrows=nrows, ncols=ncols, row_idx=z[p + "row_idx"],
                              col_idx=z[p + "col_idx"], values=z[p + "values"])
        sellp = {}
        for s in SLICES:
            q = f"{p}sellp{s}_"
            sellp[s] = SimpleNamespace(nrows=nrows, ncols=ncols, slice_size=s,
                                       slice_sets=z[q + "slice_sets"], col_idx=z[q + "col_idx"],
                                       values=z[q + "values"], row_lengths=z[q + "row_lengths"])
        csr = SimpleNamespace(nrows=nrows, ncols=ncols, row_ptrs=z[p + "csr_row_ptrs"],
                              col_idx=z[p + "col_idx"], values=z[p + "values"])
        out.append(SimpleNamespace(name=name, coo=coo, csr=csr, sellp=sellp, x=z[p + "x"], y=z[p + "y"]))
    return out


def cg_cases():
    z = _load("cg_cases.npz")
    out = []
    for name in z["names"].tolist():
        p = f"{name}__"
        nrows, ncols = (int(v) for v in z[p + "shape"])
        coo = SimpleNamespace(nrows=nrows, ncols=ncols, row_idx=z[p + "row_idx"],
                              col_idx=z[p + "col_idx"], values=z[p + "values"])
        tol, max_iters = z[p + "params"]
        out.append(SimpleNamespace(name=name, coo=coo, b=z[p + "b"], tol=float(tol),
                                   max_iters=int(max_iters), x=z[p + "x"], hist=z[p + "hist"]))
    return out
