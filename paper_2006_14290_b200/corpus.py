"""Synthetic matrix families generated directly in HBM.

* `poisson2d_matrix` — the reference's 5-point Poisson (corpus.py:33-50):
  diag 4, off -1, natural order r = j*nx + i.
* `stencil3d` — 3-D 7-point (diag 6) and 27-point (diag 26) Laplacians
  (BASELINE configs 2 and 4).
* `convection_diffusion3d` — nonsymmetric 7-point -Lap(u) + beta.grad(u),
  central differences: neighbour +d gets -1 + beta_d/2, -d gets -1 - beta_d/2
  (BASELINE config 5).
* `rmat` — R-MAT / Graph500 power-law matrix (BASELINE config 3) from a
  counter-based hash; duplicates summed with `from_entries` semantics.

All return device twins (`device.DeviceCsr` / `DeviceCoo`); call
`.to_host()` for the reference's host dataclasses. The CPU oracle
(`oracle/corpus_ref.py`) regenerates the same matrices bit for bit.
"""

import numpy as np
import torch

from . import _lib
from . import device as D

POINTS_5PT = [(0, -1, 0, -1.0), (-1, 0, 0, -1.0), (0, 0, 0, 4.0), (1, 0, 0, -1.0), (0, 1, 0, -1.0)]


def points_7pt(diag=6.0, beta=(0.0, 0.0, 0.0)):
    bx, by, bz = beta
    return [(0, 0, -1, -1.0 - bz / 2), (0, -1, 0, -1.0 - by / 2), (-1, 0, 0, -1.0 - bx / 2), (0, 0, 0, diag),
            (1, 0, 0, -1.0 + bx / 2), (0, 1, 0, -1.0 + by / 2), (0, 0, 1, -1.0 + bz / 2)]


def points_27pt():
    return [(dx, dy, dz, 26.0 if (dx, dy, dz) == (0, 0, 0) else -1.0)
            for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]


def stencil(nx, ny, nz, points, device=None) -> D.DeviceCsr:
    """CSR of a constant-coefficient stencil, built by `wk_gen_stencil_csr`."""
    dev = D._dev(device)
    n = nx * ny * nz
    pts = list(points)
    dx = np.array([p[0] for p in pts], dtype=np.int32)
    dy = np.array([p[1] for p in pts], dtype=np.int32)
    dz = np.array([p[2] for p in pts], dtype=np.int32)
    vals = np.array([p[3] for p in pts], dtype=np.float64)
    hp = [a.ctypes.data_as(_lib.P) for a in (dx, dy, dz, vals)]
    st = D.stream_handle(dev)
    ws = D.workspace(dev)
    ptrs = torch.empty(n + 1, dtype=torch.int32, device=dev)
    _lib.call("wk_gen_stencil_csr", nx, ny, nz, len(pts), *hp, D._ptr(ptrs), None, None, D._ptr(ws.scan_ws(n)), st)
    nnz = int(ptrs[-1].item())
    col = torch.empty(nnz, dtype=torch.int32, device=dev)
    val = torch.empty(nnz, dtype=torch.float64, device=dev)
    _lib.call("wk_gen_stencil_csr", nx, ny, nz, len(pts), *hp, D._ptr(ptrs), D._ptr(col), D._ptr(val),
              D._ptr(ws.scan_ws(n)), st)
    return D.DeviceCsr(n, n, ptrs, col, val)


def poisson2d_matrix(nx, ny=None, device=None) -> D.DeviceCsr:
    """corpus.py:33-50 as a device CSR."""
    ny = nx if ny is None else ny
    return stencil(nx, ny, 1, POINTS_5PT, device)


def stencil3d(n, points=7, device=None) -> D.DeviceCsr:
    pts = points_7pt() if points == 7 else points_27pt() if points == 27 else points
    return stencil(n, n, n, pts, device)


CONV_DIFF_BETA = (1.0, 0.5, 0.25)


def convection_diffusion3d(n, beta=CONV_DIFF_BETA, device=None) -> D.DeviceCsr:
    return stencil(n, n, n, points_7pt(6.0, beta), device)


def rmat_edge_keys(scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=42, device=None, chunk=1 << 26):
    """The raw R-MAT edge list as (row * 2**scale + col int64 keys, U[0,1)
    values), in edge order (duplicates present)."""
    dev = D._dev(device)
    nedges = (1 << scale) * edge_factor
    keys = torch.empty(nedges, dtype=torch.int64, device=dev)
    vals = torch.empty(nedges, dtype=torch.float64, device=dev)
    st = D.stream_handle(dev)
    for lo in range(0, nedges, chunk):
        cnt = min(chunk, nedges - lo)
        _lib.call("wk_gen_rmat_edges", scale, edge_factor, a, b, c, seed, lo, cnt,
                  D._ptr(keys[lo:lo + cnt]), D._ptr(vals[lo:lo + cnt]), st)
    return keys, vals


def rmat(scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=42, device=None, chunk=1 << 26) -> D.DeviceCoo:
    """R-MAT(scale, edge_factor) as a sorted, duplicate-summed device COO."""
    keys, vals = rmat_edge_keys(scale, edge_factor, a, b, c, seed, device, chunk)
    n = 1 << scale
    return D.coo_from_keys(n, n, keys, vals, sum_duplicates=True, owned=True)
