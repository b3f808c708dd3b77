"""CPU oracle (TEST INFRASTRUCTURE ONLY): synthetic matrix families.

* `diagonal`, `tridiagonal`, `poisson2d`, `random_sparse` restate
  `warpkit/corpus.py:18-66` (values, natural ordering, ascending columns).
* `stencil` generalises the 5-point Poisson rule (corpus.py:33-50) to any
  3-D stencil: row r = (k*ny + j)*nx + i, one entry per in-bounds stencil
  point, points ordered by linear offset so columns ascend. It is the CPU
  restatement of the device generator `wk_gen_stencil_csr`.
* `rmat` is the R-MAT / Graph500 generator of BASELINE config 3 restated on
  top of the same counter-based hash (splitmix64) as the device generator
  `wk_gen_rmat_coo`, so both sides build the identical matrix.
"""

import numpy as np

from .sparse_ref import coo_from_entries, coo_to_csr
from types import SimpleNamespace


def diagonal(n, value=2.0):
    idx = np.arange(n, dtype=np.int64)
    return SimpleNamespace(nrows=n, ncols=n, row_idx=idx, col_idx=idx.copy(), values=np.full(n, value))


def tridiagonal(n, diag=2.0, off=-1.0):
    return stencil(n, 1, 1, [(-1, 0, 0, off), (0, 0, 0, diag), (1, 0, 0, off)])


def random_sparse(nrows, ncols, density, rng, integer=False):
    """corpus.py:53-66: Bernoulli(density) pattern, U[0,1) or int 1..9 values."""
    mask = rng.random((nrows, ncols)) < density
    rows, cols = np.nonzero(mask)
    if integer:
        vals = rng.integers(1, 10, size=len(rows)).astype(np.float64)
    else:
        vals = rng.random(len(rows))
    return coo_from_entries(nrows, ncols, rows, cols, vals)


# -- stencils -------------------------------------------------------------------

def points_5pt():
    return [(0, -1, 0, -1.0), (-1, 0, 0, -1.0), (0, 0, 0, 4.0), (1, 0, 0, -1.0), (0, 1, 0, -1.0)]


def points_7pt(diag=6.0, beta=(0.0, 0.0, 0.0)):
    """3-D 7-point: diag `diag`; neighbour along +d gets -1 + beta_d/2 and
    along -d gets -1 - beta_d/2 (central-difference convection term; beta = 0
    gives the Laplacian)."""
    bx, by, bz = beta
    return [(0, 0, -1, -1.0 - bz / 2), (0, -1, 0, -1.0 - by / 2), (-1, 0, 0, -1.0 - bx / 2),
            (0, 0, 0, diag),
            (1, 0, 0, -1.0 + bx / 2), (0, 1, 0, -1.0 + by / 2), (0, 0, 1, -1.0 + bz / 2)]


def points_27pt():
    pts = []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                pts.append((dx, dy, dz, 26.0 if (dx, dy, dz) == (0, 0, 0) else -1.0))
    return pts


def _sorted_points(points, nx, ny):
    return sorted(points, key=lambda p: p[2] * nx * ny + p[1] * nx + p[0])


def stencil(nx, ny, nz, points, row_lo=0, row_hi=None):
    """CSR of a constant-coefficient stencil on an nx*ny*nz grid; with
    row_lo/row_hi only those rows (global column indices), e.g. a z-slab
    sample of a large grid."""
    pts = _sorted_points(points, nx, ny)
    ncols = nx * ny * nz
    row_hi = ncols if row_hi is None else row_hi
    r = np.arange(row_lo, row_hi, dtype=np.int64)
    n = len(r)
    i = r % nx
    j = (r // nx) % ny
    k = r // (nx * ny)
    masks = []
    for dx, dy, dz, _ in pts:
        masks.append((i + dx >= 0) & (i + dx < nx) & (j + dy >= 0) & (j + dy < ny)
                     & (k + dz >= 0) & (k + dz < nz))
    lengths = np.sum(masks, axis=0).astype(np.int64)
    ptrs = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lengths, out=ptrs[1:])
    nnz = int(ptrs[-1])
    col = np.empty(nnz, dtype=np.int64)
    val = np.empty(nnz, dtype=np.float64)
    pos = np.zeros(n, dtype=np.int64)
    local = np.arange(n, dtype=np.int64)
    for (dx, dy, dz, v), mk in zip(pts, masks):
        rows = local[mk]
        dst = ptrs[rows] + pos[rows]
        col[dst] = r[mk] + dz * nx * ny + dy * nx + dx
        val[dst] = v
        pos[rows] += 1
    return SimpleNamespace(nrows=n, ncols=ncols, row_ptrs=ptrs, col_idx=col, values=val)


def poisson2d(nx, ny=None):
    """corpus.py:33-50 (2-D 5-point, diag 4, off -1) as CSR."""
    ny = nx if ny is None else ny
    return stencil(nx, ny, 1, points_5pt())


# -- R-MAT ------------------------------------------------------------------------

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(z):
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def uniform(seed, counter):
    """U[0,1) double from 53 hash bits of (seed, counter)."""
    with np.errstate(over="ignore"):
        h = splitmix64(np.uint64(seed) * np.uint64(0xD1B54A32D192ED03) + np.asarray(counter, dtype=np.uint64))
    return (h >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def rmat_edges(scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=42, edge_lo=0, edge_hi=None):
    """Edges [edge_lo, edge_hi) of R-MAT(scale): for edge e and level l the
    uniform u(seed, e*(scale+1) + l) picks the quadrant (a | b | c | d) that
    sets bit (scale-1-l) of (row, col); u(seed, e*(scale+1) + scale) is the
    value. No vertex permutation (BASELINE config 3)."""
    nedges = (1 << scale) * edge_factor
    edge_hi = nedges if edge_hi is None else edge_hi
    e = np.arange(edge_lo, edge_hi, dtype=np.uint64)
    rows = np.zeros(len(e), dtype=np.int64)
    cols = np.zeros(len(e), dtype=np.int64)
    L = np.uint64(scale + 1)
    for lvl in range(scale):
        u = uniform(seed, e * L + np.uint64(lvl))
        bit = np.int64(1) << np.int64(scale - 1 - lvl)
        row_bit = u >= a + b
        col_bit = ((u >= a) & (u < a + b)) | (u >= a + b + c)
        rows |= np.where(row_bit, bit, 0)
        cols |= np.where(col_bit, bit, 0)
    vals = uniform(seed, e * L + np.uint64(scale))
    return rows, cols, vals


def rmat(scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=42):
    """R-MAT matrix as sorted, duplicate-summed COO (from_entries semantics,
    sparse.py:63-80): duplicates are summed in edge order."""
    n = 1 << scale
    rows, cols, vals = rmat_edges(scale, edge_factor, a, b, c, seed)
    return coo_from_entries(n, n, rows, cols, vals)


def to_csr(m):
    return m if hasattr(m, "row_ptrs") else coo_to_csr(m)
