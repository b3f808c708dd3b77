"""Row-block partitioning, halo exchange and the distributed CG control flow,
exercised on CPU with world-size-2 gloo process groups.

The product's local kernels need a GPU, so the rank-local compute is
replaced by `NumpyOps` — a CPU restatement (test infrastructure, built on the
oracle) of the same building blocks (gather, SpMV, wk_cg_* steps) — while
the partition planner, the exchange, the all-reduces and the CG driver are
the product code in paper_2006_14290_b200.distributed.
"""

import ctypes
import math
import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import corpus_ref, krylov_ref, sparse_ref
from paper_2006_14290_b200 import _lib
from paper_2006_14290_b200 import distributed as DI

ST = _lib.WkCgState
OFF = {name: getattr(ST, name).offset for name, _ in ST._fields_}


class NumpyOps:
    """CPU restatement of DeviceOps (same update order as krylov.cu)."""

    device = torch.device("cpu")

    def zeros(self, n):
        return torch.zeros(n, dtype=torch.float64)

    def index(self, arr):
        return torch.as_tensor(np.asarray(arr, dtype=np.int64))

    def gather(self, idx, src, dst):
        dst.copy_(src[idx])

    def spmv(self, local, x_ext, y):
        y[: local.nrows] = torch.from_numpy(sparse_ref.spmv(local, x_ext.numpy()))

    def spmv_masked(self, local, x_ext, y, state):
        if not self._get(state, "done"):
            self.spmv(local, x_ext, y)

    def spmv_dot(self, local, p_ext, q, state):
        self.spmv_masked(local, p_ext, q, state)
        self.cg("wk_cg_dot_pq", local.nrows, p_ext, q, state)

    def new_state(self):
        return torch.zeros(ctypes.sizeof(ST), dtype=torch.uint8)

    def _get(self, st, name):
        ctype = dict(ST._fields_)[name]
        return ctype.from_buffer_copy(st.numpy().tobytes()[OFF[name]:OFF[name] + ctypes.sizeof(ctype)]).value

    def _set(self, st, name, value):
        ctype = dict(ST._fields_)[name]
        raw = bytes(ctype(value))
        st[OFF[name]:OFF[name] + len(raw)] = torch.frombuffer(bytearray(raw), dtype=torch.uint8)

    def read_state(self, st):
        return ST.from_buffer_copy(st.numpy().tobytes())

    def cg(self, name, *a):
        g, s = self._get, self._set
        if name == "wk_cg_init_local":
            n, b, x, r, p, st = a
            x[:n] = 0.0
            r[:] = b
            p[:n] = b
            s(st, "rho", float(b.numpy() @ b.numpy()))
            s(st, "iteration", 0)
            s(st, "done", 0)
            s(st, "breakdown", 0)
        elif name == "wk_cg_init_finish":
            st, tol, max_iters, hist = a
            bn = math.sqrt(g(st, "rho"))
            hist[0] = bn
            s(st, "threshold", tol * bn)
            s(st, "max_iters", max_iters)
            s(st, "done", int(not (bn != 0.0 and 0 < max_iters and bn > tol * bn)))
        elif name == "wk_cg_dot_pq":
            n, p, q, st = a
            if not g(st, "done"):
                s(st, "pq", float(p[:n].numpy() @ q[:n].numpy()))
        elif name == "wk_cg_step_alpha":
            (st,) = a
            if g(st, "done"):
                return
            pq = g(st, "pq")
            s(st, "iteration", g(st, "iteration") + 1)
            if pq <= 0.0:
                s(st, "breakdown", 1)
                s(st, "done", 1)
                return
            s(st, "alpha", g(st, "rho") / pq)
        elif name == "wk_cg_update_xr":
            n, p, q, x, r, st = a
            if g(st, "done"):
                return
            al = g(st, "alpha")
            x[:n] = x[:n] + al * p[:n]
            if g(st, "iteration") % 50 != 0:
                r[:] = r - al * q[:n]
                s(st, "rr", float(r.numpy() @ r.numpy()))
        elif name == "wk_cg_replace_r":
            n, b, q, r, st = a
            if g(st, "done") or g(st, "iteration") % 50 != 0:
                return
            r[:] = b - q[:n]
            s(st, "rr", float(r.numpy() @ r.numpy()))
        elif name == "wk_cg_step_beta":
            st, hist = a
            if g(st, "done"):
                return
            rr = g(st, "rr")
            it = g(st, "iteration")
            hist[it] = math.sqrt(rr)
            s(st, "beta", rr / g(st, "rho"))
            s(st, "rho", rr)
            s(st, "done", int(not (it < g(st, "max_iters") and math.sqrt(rr) > g(st, "threshold"))))
        elif name == "wk_cg_update_xr_alpha":
            self.cg("wk_cg_step_alpha", a[5])
            self.cg("wk_cg_update_xr", *a)
        elif name == "wk_cg_update_p_beta":
            n, r, p, st, hist = a
            if g(st, "done"):
                return
            beta = g(st, "rr") / g(st, "rho")
            p[:n] = r + beta * p[:n]
            self.cg("wk_cg_step_beta", st, hist)
        elif name == "wk_cg_update_p":
            n, r, p, st = a
            if not g(st, "done"):
                p[:n] = r + g(st, "beta") * p[:n]
        else:
            raise KeyError(name)


def _upload_cpu(nrows, ncols, ptrs, cols, vals):
    return SimpleNamespace(nrows=nrows, ncols=ncols, row_ptrs=ptrs, col_idx=cols, values=vals)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = DI.Comm()
        m = case["matrix"]
        op = DI.partition_csr(m, comm, ops=NumpyOps(), upload=_upload_cpu)
        lo, hi = op.bounds[rank], op.bounds[rank + 1]
        x = case["x"]
        x_ext = op.new_vector()
        x_ext[: op.n_local] = torch.from_numpy(x[lo:hi])
        y = torch.zeros(op.n_local, dtype=torch.float64)
        op.spmv(x_ext, y)
        res = {"y": y.numpy().copy(), "lo": lo, "hi": hi, "n_halo": op.n_halo}
        if case.get("cg"):
            b = torch.from_numpy(case["b"][lo:hi].copy())
            xs, hist = DI.cg_solve(op, b, case["tol"], case["max_iters"])
            res["x"] = xs.numpy().copy()
            res["hist"] = hist.numpy().copy()
        out[rank] = res
    finally:
        dist.destroy_process_group()


def _run(case, world=2):
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), case, out), nprocs=world, join=True)
    return [out[r] for r in range(world)]


def test_row_blocks_aligned():
    b = DI.row_blocks(1000, 3)
    assert b[0] == 0 and b[-1] == 1000
    assert all(v % 64 == 0 for v in b[1:-1])
    assert DI.row_blocks(10, 4)[-1] == 10


def test_localize_columns_keeps_global_order():
    halo = np.array([3, 9, 40], dtype=np.int64)
    got = DI.localize_columns([3, 10, 11, 40, 9], 10, 20, halo)
    assert got.tolist() == [10, 0, 1, 12, 11]


def test_plan_matches_needs():
    bounds = [0, 64, 128, 192]
    needs = [np.array([64, 65, 130]), np.array([0, 129, 191]), np.array([127])]
    plan = DI._plan_from_needs(1, bounds, needs)
    assert plan.recv_ranges == {0: (0, 1), 2: (1, 2)}
    assert {q: v.tolist() for q, v in plan.send_idx.items()} == {0: [0, 1], 2: [63]}


@pytest.mark.parametrize("kind", ["stencil", "random"])
def test_distributed_spmv_bitwise(kind):
    rng = np.random.default_rng(3)
    if kind == "stencil":
        m = corpus_ref.stencil(6, 5, 7, corpus_ref.points_27pt())
    else:
        m = sparse_ref.coo_to_csr(corpus_ref.random_sparse(300, 300, 0.03, rng))
    x = rng.standard_normal(m.ncols)
    parts = _run({"matrix": m, "x": x})
    y = np.concatenate([p["y"] for p in parts])
    assert y.tobytes() == sparse_ref.spmv(m, x).tobytes()
    assert parts[0]["n_halo"] > 0


def test_distributed_cg_matches_oracle():
    m = corpus_ref.poisson2d(16)  # 256 rows -> 2 blocks of 128
    b = np.ones(m.nrows)
    tol, max_iters = 1e-10, 500
    parts = _run({"matrix": m, "x": np.zeros(m.nrows), "cg": True, "b": b, "tol": tol, "max_iters": max_iters})
    sp = sparse_ref.csr_to_sellp(m, 64)
    xr, hr = krylov_ref.cg_solve(lambda v: sparse_ref.spmv(sp, v), b, tol, max_iters)
    hist = parts[0]["hist"]
    assert np.array_equal(hist, parts[1]["hist"])  # identical control on both ranks
    assert len(hist) == len(hr)
    assert np.max(np.abs(hist - hr)) / np.linalg.norm(b) <= 1e-10
    x = np.concatenate([p["x"] for p in parts])
    assert sparse_ref.max_scaled_rel_err(x, xr, sparse_ref.row_nnz(m)) <= 1e-10


def test_distributed_cg_long_run_with_replacement():
    m = corpus_ref.poisson2d(24)  # > 50 iterations: covers the residual replacement
    b = np.linspace(-1.0, 1.0, m.nrows)
    parts = _run({"matrix": m, "x": np.zeros(m.nrows), "cg": True, "b": b, "tol": 1e-12, "max_iters": 400})
    sp = sparse_ref.csr_to_sellp(m, 64)
    xr, hr = krylov_ref.cg_solve(lambda v: sparse_ref.spmv(sp, v), b, 1e-12, 400)
    hist = parts[0]["hist"]
    assert len(hr) > 51 and len(hist) == len(hr)
    assert np.max(np.abs(hist - hr)) / np.linalg.norm(b) <= 1e-10
