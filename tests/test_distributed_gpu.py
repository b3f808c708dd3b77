"""The row-block distributed path with the real device kernels: two ranks
share cuda:0 over a gloo group (the GPU box has one GPU; NCCL refuses two
ranks on one device), so halo exchange and all-reduces are staged through
host memory while packing, SpMV and the fused CG steps are libwk_sparse.
Checks: distributed SpMV bitwise == single-GPU SpMV; distributed CG has the
oracle's iteration count and residual history within 1e-10 * ||b||."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import corpus_ref, krylov_ref, sparse_ref  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2006_14290_b200 import corpus
        from paper_2006_14290_b200 import distributed as DI
        from paper_2006_14290_b200 import kernels

        res = {}
        # weak-scaled 27-point slabs, SELL-P local format
        op = DI.stencil_slab_operator(12, 10, 6, corpus.points_27pt(), dist, fmt="sellp")
        x = op.new_vector()
        g = torch.Generator(device="cuda").manual_seed(5 + rank)
        x[: op.n_local] = torch.rand(op.n_local, dtype=torch.float64, device="cuda", generator=g)
        y = torch.zeros(op.n_local, dtype=torch.float64, device="cuda")
        op.spmv(x, y)
        res["slab_x"] = x[: op.n_local].cpu().numpy()
        res["slab_y"] = y.cpu().numpy()
        # strong partition of a generic CSR (csr and ell local formats)
        m = corpus_ref.poisson2d(20)
        for fmt in ("csr", "ell", "hybrid"):
            opc = DI.partition_csr(m, DI.Comm(), fmt=fmt)
            xg = np.random.default_rng(9).standard_normal(m.nrows)
            xe = opc.new_vector()
            lo, hi = opc.bounds[rank], opc.bounds[rank + 1]
            xe[: opc.n_local] = torch.from_numpy(xg[lo:hi]).cuda()
            yy = torch.zeros(opc.n_local, dtype=torch.float64, device="cuda")
            opc.spmv(xe, yy)
            res[f"y_{fmt}"] = yy.cpu().numpy()
        # distributed CG on the strong-partitioned 7-point 12^3 Laplacian
        opg = DI.stencil_slab_operator(12, 12, None, corpus.points_7pt(), dist, fmt="sellp", weak=False, nz=12)
        b = torch.ones(opg.n_local, dtype=torch.float64, device="cuda")
        xs, hist = DI.cg_solve(opg, b, 1e-10, 500)
        res["cg_x"] = xs.cpu().numpy()
        res["cg_hist"] = hist.cpu().numpy()
        # nonsymmetric convection-diffusion: distributed BiCGSTAB and GMRES(30)
        opn = DI.stencil_slab_operator(10, 10, None, corpus.points_7pt(6.0, corpus.CONV_DIFF_BETA), dist,
                                       fmt="csr", weak=False, nz=10)
        bn = torch.ones(opn.n_local, dtype=torch.float64, device="cuda")
        xs, hist = DI.bicgstab_solve(opn, bn, 1e-10, 500)
        res["bicg_x"], res["bicg_hist"] = xs.cpu().numpy(), hist.cpu().numpy()
        xs, hist = DI.gmres_solve(opn, bn, 1e-10, 500, restart=30)
        res["gmres_x"], res["gmres_hist"] = xs.cpu().numpy(), hist.cpu().numpy()
        out[rank] = res
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def parts():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    return [out[0], out[1]]


def test_slab_spmv_bitwise(parts):
    m = corpus_ref.stencil(12, 10, 12, corpus_ref.points_27pt())
    x = np.concatenate([p["slab_x"] for p in parts])
    y = np.concatenate([p["slab_y"] for p in parts])
    assert y.tobytes() == sparse_ref.spmv(m, x).tobytes()


@pytest.mark.parametrize("fmt", ["csr", "ell", "hybrid"])
def test_partitioned_formats(parts, fmt):
    m = corpus_ref.poisson2d(20)
    xg = np.random.default_rng(9).standard_normal(m.nrows)
    y = np.concatenate([p[f"y_{fmt}"] for p in parts])
    ref = sparse_ref.spmv(m, xg)
    if fmt == "hybrid":
        assert sparse_ref.max_scaled_rel_err(y, ref, sparse_ref.row_nnz(m)) <= 1e-12
    else:
        assert y.tobytes() == ref.tobytes()


def _nccl_worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    try:
        from paper_2006_14290_b200 import corpus
        from paper_2006_14290_b200 import distributed as DI

        opg = DI.stencil_slab_operator(24, 24, None, corpus.points_7pt(), dist, fmt="sellp", weak=False, nz=24)
        b = torch.ones(opg.n_local, dtype=torch.float64, device="cuda")
        res = {}
        for graph in (False, True):
            xs, hist = DI.cg_solve(opg, b, 1e-13, 500, graph=graph)
            res[f"x_{graph}"] = xs.cpu().numpy()
            res[f"hist_{graph}"] = hist.cpu().numpy()
            opn = DI.stencil_slab_operator(16, 16, None, corpus.points_7pt(6.0, corpus.CONV_DIFF_BETA), dist,
                                           fmt="sellp", weak=False, nz=16)
            bn = torch.ones(opn.n_local, dtype=torch.float64, device="cuda")
            xs, hist = DI.bicgstab_solve(opn, bn, 1e-12, 500, graph=graph)
            res[f"bicg_hist_{graph}"] = hist.cpu().numpy()
            xs, hist = DI.gmres_solve(opn, bn, 1e-12, 500, restart=10, graph=graph)
            res[f"gmres_hist_{graph}"] = hist.cpu().numpy()
        out[rank] = res
    finally:
        dist.destroy_process_group()


def test_distributed_cg_nccl_graph_single_rank():
    """The NCCL + CUDA-graph path of the distributed CG (one rank: the
    all-reduces are real NCCL calls captured in the graph)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_nccl_worker, args=(1, _free_port(), out), nprocs=1, join=True)
    res = out[0]
    assert len(res["hist_True"]) > 51  # several graph replays
    assert np.array_equal(res["hist_True"], res["hist_False"])
    for k in ("bicg", "gmres"):
        assert len(res[f"{k}_hist_True"]) > 12
        assert np.array_equal(res[f"{k}_hist_True"], res[f"{k}_hist_False"])
    assert np.array_equal(res["x_True"], res["x_False"])
    m = corpus_ref.stencil(24, 24, 24, corpus_ref.points_7pt())
    sp = sparse_ref.csr_to_sellp(m, 64)
    b = np.ones(m.nrows)
    xr, hr = krylov_ref.cg_solve(lambda v: sparse_ref.spmv(sp, v), b, 1e-13, 500)
    assert len(res["hist_True"]) == len(hr)
    assert np.max(np.abs(res["hist_True"] - hr)) / np.linalg.norm(b) <= 1e-10


def test_distributed_cg(parts):
    m = corpus_ref.stencil(12, 12, 12, corpus_ref.points_7pt())
    b = np.ones(m.nrows)
    sp = sparse_ref.csr_to_sellp(m, 64)
    xr, hr = krylov_ref.cg_solve(lambda v: sparse_ref.spmv(sp, v), b, 1e-10, 500)
    h0, h1 = parts[0]["cg_hist"], parts[1]["cg_hist"]
    assert np.array_equal(h0, h1)
    assert len(h0) == len(hr)
    assert np.max(np.abs(h0 - hr)) / np.linalg.norm(b) <= 1e-10
    x = np.concatenate([p["cg_x"] for p in parts])
    assert sparse_ref.max_scaled_rel_err(x, xr, sparse_ref.row_nnz(m)) <= 1e-10


@pytest.mark.parametrize("solver", ["bicg", "gmres"])
def test_distributed_nonsymmetric(parts, solver):
    m = corpus_ref.stencil(10, 10, 10, corpus_ref.points_7pt(beta=(1.0, 0.5, 0.25)))
    b = np.ones(m.nrows)
    f = lambda v: sparse_ref.spmv(m, v)  # noqa: E731
    if solver == "bicg":
        xr, hr = krylov_ref.bicgstab_solve(f, b, 1e-10, 500)
    else:
        xr, hr = krylov_ref.gmres_solve(f, b, 1e-10, 500, restart=30)
    h0, h1 = parts[0][f"{solver}_hist"], parts[1][f"{solver}_hist"]
    assert np.array_equal(h0, h1)
    assert len(h0) == len(hr)
    assert np.max(np.abs(h0 - hr)) / np.linalg.norm(b) <= 1e-10
    x = np.concatenate([p[f"{solver}_x"] for p in parts])
    assert sparse_ref.max_scaled_rel_err(x, xr, sparse_ref.row_nnz(m)) <= 1e-10
