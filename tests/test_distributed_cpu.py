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

    def read_state(self, st, cls=None):
        return (cls or ST).from_buffer_copy(st.numpy().tobytes())

    def new_struct(self, cls):
        return torch.zeros(ctypes.sizeof(cls), dtype=torch.uint8)

    def spmv_flag(self, local, x_ext, y, state, offset):
        if int(np.frombuffer(state.numpy().tobytes()[offset:offset + 4], dtype=np.int32)[0]) == 0:
            self.spmv(local, x_ext, y)

    def bicg_spmv_dots(self, local, x_ext, y, state, w, mode):
        self.spmv_flag(local, x_ext, y, state, _lib.WkBicgState.done.offset)
        n = local.nrows
        if mode == 1:
            _bicg_step("rv", n, w, y, state)
        else:
            _bicg_step("tt_ts", n, y, x_ext, state)

    def step(self, name, *a, ws=False):
        """BiCGSTAB / GMRES step kernels of csrc/krylov_steps.cu restated
        (same statement order; the state struct is edited in place)."""
        if name.startswith("wk_bicg_"):
            return _bicg_step(name[len("wk_bicg_"):], *a)
        if name.startswith("wk_gmres_"):
            return _gmres_step(name[len("wk_gmres_"):], *a)
        raise KeyError(name)

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
            # x += alpha p only on replacement iterations (else in the p update)
            self.cg("wk_cg_step_alpha", a[5])
            n, p, q, x, r, st = a
            if g(st, "done"):
                return
            al = g(st, "alpha")
            if g(st, "iteration") % 50 == 0:
                x[:n] = x[:n] + al * p[:n]
            else:
                r[:] = r - al * q[:n]
                s(st, "rr", float(r.numpy() @ r.numpy()))
        elif name == "wk_cg_update_p_beta":
            n, r, p, x, st, hist = a
            if g(st, "done"):
                return
            if g(st, "iteration") % 50 != 0:
                x[:n] = x[:n] + g(st, "alpha") * p[:n]
            beta = g(st, "rr") / g(st, "rho")
            p[:n] = r + beta * p[:n]
            self.cg("wk_cg_step_beta", st, hist)
        elif name == "wk_cg_update_p":
            n, r, p, st = a
            if not g(st, "done"):
                p[:n] = r + g(st, "beta") * p[:n]
        else:
            raise KeyError(name)


def _dot(a, b):
    return float(a.numpy() @ b.numpy())


def _bicg_step(name, *a):
    """krylov_steps.cu bicg_* (wk_bicg_state via ctypes.from_buffer)."""
    st = a[-1] if name in ("init", "rho", "update_p", "rv", "update_s", "half_x", "tt_ts", "update_xr",
                           "rho_first", "update_xr_rho") else None
    if name in ("init_finish", "step_beta", "step_alpha", "step_s", "step_omega", "step_r", "take_rho"):
        st = a[0]
    s = _lib.WkBicgState.from_buffer(st.numpy())
    if name == "init":
        n, b, x, r, rh, p, v, _ = a
        x[:n] = 0.0
        r[:n] = b
        rh[:n] = b
        p[:] = 0.0
        v[:n] = 0.0
        s.rr = _dot(b, b)
    elif name == "init_finish":
        _, tol, max_iters, hist = a
        bn = math.sqrt(s.rr)
        hist[0] = bn
        s.rho = s.alpha = s.omega = 1.0
        s.threshold = tol * bn
        s.iteration, s.max_iters, s.breakdown, s.apply_half = 0, max_iters, 0, 0
        s.done = int(not (bn != 0.0 and 0 < max_iters and bn > s.threshold))
    elif name == "rho":
        n, rh, r, _ = a
        if not s.done:
            s.rho_new = _dot(rh[:n], r[:n])
    elif name == "step_beta":
        if s.done:
            return
        if s.rho_new == 0.0:
            s.breakdown, s.done = 1, 1
            s.iteration += 1
            return
        s.beta = (s.rho_new / s.rho) * (s.alpha / s.omega)
    elif name == "update_p":
        n, r, v, p, _ = a
        if not s.done:
            p[:n] = r[:n] + s.beta * (p[:n] - s.omega * v[:n])
    elif name == "rv":
        n, rh, v, _ = a
        if not s.done:
            s.rv = _dot(rh[:n], v[:n])
    elif name == "step_alpha":
        if s.done:
            return
        if s.rv == 0.0:
            s.breakdown, s.done = 1, 1
            s.iteration += 1
            return
        s.alpha = s.rho_new / s.rv
    elif name == "update_s":
        n, r, v, sv, _ = a
        if not s.done:
            sv[:n] = r[:n] - s.alpha * v[:n]
            s.ss = _dot(sv[:n], sv[:n])
    elif name == "step_s":
        _, hist = a
        if s.done:
            return
        s.iteration += 1
        sn = math.sqrt(s.ss)
        if sn <= s.threshold:
            hist[s.iteration] = sn
            s.apply_half, s.done = 1, 1
    elif name == "half_x":
        n, p, x, _ = a
        if s.apply_half:
            x[:n] = x[:n] + s.alpha * p[:n]
            s.apply_half = 0
    elif name == "tt_ts":
        n, t, sv, _ = a
        if not s.done:
            s.tt = _dot(t[:n], t[:n])
            s.ts = _dot(t[:n], sv[:n])
    elif name == "step_omega":
        if s.done:
            return
        if s.tt == 0.0:
            s.breakdown, s.done = 1, 1
            return
        s.omega = s.ts / s.tt
    elif name == "update_xr":
        n, p, sv, t, x, r, _ = a
        if not s.done:
            x[:n] = (x[:n] + s.alpha * p[:n]) + s.omega * sv[:n]
            r[:n] = sv[:n] - s.omega * t[:n]
            s.rr = _dot(r[:n], r[:n])
    elif name == "rho_first":
        n, rh, r, _ = a
        if not s.done:
            s.rho_next = _dot(rh[:n], r[:n])
    elif name == "take_rho":
        if not s.done:
            s.rho_new = s.rho_next
    elif name == "update_xr_rho":
        n, p, sv, t, rh, x, r, _ = a
        if not s.done:
            x[:n] = (x[:n] + s.alpha * p[:n]) + s.omega * sv[:n]
            r[:n] = sv[:n] - s.omega * t[:n]
            s.rr = _dot(r[:n], r[:n])
            s.rho_next = _dot(rh[:n], r[:n])
    elif name == "step_r":
        _, hist = a
        if s.done:
            return
        rn = math.sqrt(s.rr)
        hist[s.iteration] = rn
        s.rho = s.rho_new
        s.done = int(not (s.iteration < s.max_iters and rn > s.threshold))
    else:
        raise KeyError(name)


def _gmres_step(name, *a):
    """krylov_steps.cu gmres_* (wk_gmres_state via ctypes.from_buffer)."""
    idx = {"init": 4, "init_finish": 0, "cycle_start": 4, "multidot": 6, "orth": 6, "givens": 5,
           "next_basis": 3, "update_x": 7, "residual": 4, "restart": 0, "orth_scaled": 7, "givens_scaled": 6,
           "update_x_scaled": 8}[name]
    s = _lib.WkGmresState.from_buffer(a[idx].numpy())
    if name == "init":
        n, b, x, r, _ = a
        x[:n] = 0.0
        r[:n] = b
        s.sq = _dot(b, b)
    elif name == "init_finish":
        _, tol, max_iters, restart, hist = a
        bn = math.sqrt(s.sq)
        hist[0] = bn
        s.beta, s.threshold = bn, tol * bn
        s.iteration, s.max_iters, s.restart = 0, max_iters, restart
        s.done = int(not (bn != 0.0 and 0 < max_iters and bn > s.threshold))
        s.cycle_done, s.j_done = s.done, 0
    elif name == "cycle_start":
        n, r, V0, g, _ = a
        if s.done:
            return
        V0[:n] = r[:n] / s.beta
        g[: s.restart + 1] = 0.0
        g[0] = s.beta
        s.j_done, s.cycle_done = 0, 0
    elif name == "multidot":
        n, j, V, ld, w, Hj, _ = a
        if not s.cycle_done:
            for q in range(j + 1):
                Hj[q] = _dot(V[q * ld: q * ld + n], w[:n])
    elif name == "orth":
        n, j, V, ld, w, Hj, _ = a
        if not s.cycle_done:
            for q in range(j + 1):
                w[:n] = w[:n] - float(Hj[q]) * V[q * ld: q * ld + n]
            s.sq = _dot(w[:n], w[:n])
    elif name == "orth_scaled":
        n, j, V, ld, w, Hj, sig, _ = a
        if not s.cycle_done:
            sj = float(sig[j])
            h = [float(sig[q]) * sj * float(Hj[q]) for q in range(j + 1)]
            w[:n] = sj * w[:n]
            for q in range(j + 1):
                w[:n] = w[:n] - h[q] * float(sig[q]) * V[q * ld: q * ld + n]
                Hj[q] = h[q]
            s.sq = _dot(w[:n], w[:n])
    elif name == "givens_scaled":
        j, H, cs, sn, g, sig, st, hist = a
        if not s.cycle_done:
            hn = math.sqrt(s.sq)
            sig[j + 1] = 1.0 / hn if hn != 0.0 else 0.0
        _gmres_step("givens", j, H, cs, sn, g, st, hist)
    elif name == "update_x_scaled":
        n, V, ld, H, g, y, x, sig, st = a
        if s.done:
            return
        m, jd = s.restart, s.j_done
        for i in range(jd - 1, -1, -1):
            acc = float(g[i])
            for k in range(i + 1, jd):
                acc = acc - float(H[i + k * (m + 1)]) * float(y[k])
            y[i] = acc / float(H[i + i * (m + 1)])
        for q in range(jd):
            x[:n] = x[:n] + float(y[q]) * float(sig[q]) * V[q * ld: q * ld + n]
    elif name == "givens":
        j, H, cs, sn, g, _, hist = a
        if s.cycle_done:
            return
        m = s.restart
        Hj = H[j * (m + 1):]
        hn = math.sqrt(s.sq)
        s.hn = hn
        Hj[j + 1] = hn
        for i in range(j):
            aa, cc = float(Hj[i]), float(Hj[i + 1])
            Hj[i] = cs[i].item() * aa + sn[i].item() * cc
            Hj[i + 1] = -sn[i].item() * aa + cs[i].item() * cc
        c, sj = krylov_ref.givens(float(Hj[j]), float(Hj[j + 1]))
        cs[j], sn[j] = c, sj
        Hj[j] = c * float(Hj[j]) + sj * float(Hj[j + 1])
        Hj[j + 1] = 0.0
        g[j + 1] = -sj * float(g[j])
        g[j] = c * float(g[j])
        s.iteration += 1
        s.j_done = j + 1
        res = abs(float(g[j + 1]))
        hist[s.iteration] = res
        if res <= s.threshold or s.iteration >= s.max_iters or hn == 0.0 or j + 1 == m:
            s.cycle_done = 1
    elif name == "next_basis":
        n, w, Vn, _ = a
        if not s.cycle_done:
            Vn[:n] = w[:n] / s.hn
    elif name == "update_x":
        n, V, ld, H, g, y, x, _ = a
        if s.done:
            return
        m, jd = s.restart, s.j_done
        for i in range(jd - 1, -1, -1):
            acc = float(g[i])
            for k in range(i + 1, jd):
                acc = acc - float(H[i + k * (m + 1)]) * float(y[k])
            y[i] = acc / float(H[i + i * (m + 1)])
        for q in range(jd):
            x[:n] = x[:n] + float(y[q]) * V[q * ld: q * ld + n]
    elif name == "residual":
        n, b, w, r, _ = a
        if not s.done:
            r[:n] = b[:n] - w[:n]
            s.sq = _dot(r[:n], r[:n])
    elif name == "restart":
        _, hist = a
        if s.done:
            return
        bt = math.sqrt(s.sq)
        s.beta = bt
        hist[s.iteration] = bt
        s.done = int(not (s.iteration < s.max_iters and bt > s.threshold))
        s.cycle_done = s.done
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
        if case.get("peer_fail"):
            _install_failing_peer_lib(rank, case["peer_fail"])
        comm = DI.Comm()
        m = case["matrix"]
        op = DI.partition_csr(m, comm, ops=NumpyOps(), upload=_upload_cpu, bounds=case.get("bounds"))
        res = {}
        if case.get("peer_fail"):
            res["mode"] = DI.maybe_enable_peer(op)
            res["peer"] = op.peer is not None or comm.peer is not None
        lo, hi = op.bounds[rank], op.bounds[rank + 1]
        x = case["x"]
        x_ext = op.new_vector()
        x_ext[: op.n_local] = torch.from_numpy(x[lo:hi])
        y = torch.zeros(op.n_local, dtype=torch.float64)
        op.spmv(x_ext, y)
        res.update({"y": y.numpy().copy(), "lo": lo, "hi": hi, "n_halo": op.n_halo})
        b = torch.from_numpy(case["b"][lo:hi].copy()) if "b" in case else None
        for kind in case.get("solvers", ("cg",) if case.get("cg") else ()):
            if kind == "cg":
                xs, hist = DI.cg_solve(op, b, case["tol"], case["max_iters"])
            elif kind == "bicgstab":
                xs, hist = DI.bicgstab_solve(op, b, case["tol"], case["max_iters"], chunk=3)
            else:
                xs, hist = DI.gmres_solve(op, b, case["tol"], case["max_iters"], restart=case.get("restart", 30))
            res[kind] = (xs[: op.n_local].numpy().copy(), hist.numpy().copy())
            if kind == "cg":
                res["x"], res["hist"] = res[kind]
        out[rank] = res
    finally:
        dist.destroy_process_group()


def _install_failing_peer_lib(rank, where):
    """Replace the native library seen by peer.PeerComm with a stub whose
    arena allocation (where="alloc") or IPC open (where="open") fails on
    rank 1 only: the set-up must fail on EVERY rank together and
    maybe_enable_peer must fall back to the process-group path everywhere."""
    from paper_2006_14290_b200 import peer as PE

    class Stub:
        freed = 0

        def wk_peer_arena_header_bytes(self):
            return 256

        def wk_sym_alloc(self, nbytes, base_ref, handle):
            if where == "alloc" and rank == 1:
                return 2
            base_ref._obj.value = 0x1000
            return 0

        def wk_sym_open(self, h, p_ref):
            if where == "open" and rank == 1:
                return 2
            p_ref._obj.value = 0x2000
            return 0

        def wk_sym_free(self, base):
            Stub.freed += 1
            return 0

        def wk_sym_close(self, p):
            return 0

        def __getattr__(self, name):
            return lambda *a: 0

    PE._lib = SimpleNamespace(load=lambda: Stub(), last_error=lambda: "stub failure", WkPeerCtx=_lib.WkPeerCtx)


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


# ---- world sizes 4 and 8: slab plans, the process-group exchange and all three solvers ----------


def _slab_bounds(nx, ny, nz, world):
    return DI.SlabLayout(nx, ny, world, 0, weak=False, nz=nz).bounds


@pytest.mark.parametrize("world", [4, 8])
def test_slab_layout_equals_generic_plan(world):
    """The z-slab plan of stencil_slab_operator (SlabLayout: one halo plane
    per side, columns remapped to [owned | lo plane | hi plane]) equals the
    generic plan partition_csr derives from the global matrix's columns, for
    every rank, including uneven plane splits (nz % world != 0)."""
    nx, ny, nz = 5, 4, 2 * world + 3
    pts = corpus_ref.points_7pt(beta=(1.0, 0.5, 0.25))
    m = corpus_ref.stencil(nx, ny, nz, pts)
    ptrs = np.asarray(m.row_ptrs, np.int64)
    cols = np.asarray(m.col_idx, np.int64)
    for g in range(world):
        lay = DI.SlabLayout(nx, ny, world, g, weak=False, nz=nz)
        bounds = lay.bounds
        needed = []
        for q in range(world):
            lo, hi = bounds[q], bounds[q + 1]
            c = cols[ptrs[lo]:ptrs[hi]]
            needed.append(np.unique(c[(c < lo) | (c >= hi)]))
        ref = DI._plan_from_needs(g, bounds, needed)
        assert np.array_equal(lay.plan.halo_cols, ref.halo_cols)
        assert lay.plan.recv_ranges == ref.recv_ranges
        assert {q: v.tolist() for q, v in lay.plan.send_idx.items()} == {q: v.tolist() for q, v in ref.send_idx.items()}
        # the local columns: extended-slab numbering -> [owned | halo] equals
        # the generic global -> local map
        ext = corpus_ref.stencil(nx, ny, lay.e1 - lay.e0, pts)
        eptr = np.asarray(ext.row_ptrs, np.int64)
        ecol = torch.as_tensor(np.asarray(ext.col_idx, np.int64)[eptr[lay.lo_rows]:eptr[lay.lo_rows + lay.n_local]])
        lo, hi = bounds[g], bounds[g + 1]
        want = DI.localize_columns(cols[ptrs[lo]:ptrs[hi]], lo, hi, ref.halo_cols)
        assert np.array_equal(lay.localize(ecol).numpy(), want)


@pytest.mark.parametrize("world", [4, 8])
def test_distributed_spmv_and_solvers_world(world):
    """World 4 / 8 over gloo with z-slab bounds: SpMV bitwise, CG equal to
    the reference CG (counts, history 1e-10, x 1e-10), GMRES(8) equal to the
    restatement, BiCGSTAB on a diagonally dominant operator (non-chaotic)
    within 1e-10 of the restatement. The exchange and all-reduces are the
    process-group path the NCCL backend uses (batch_isend_irecv /
    all_reduce)."""
    nx, ny, nz = 6, 5, 2 * world + 1
    m = corpus_ref.stencil(nx, ny, nz, corpus_ref.points_7pt(diag=8.0, beta=(1.0, 0.5, 0.25)))
    rng = np.random.default_rng(world)
    x = rng.standard_normal(m.nrows)
    b = rng.standard_normal(m.nrows)
    case = {"matrix": m, "x": x, "b": b, "tol": 1e-10, "max_iters": 200, "restart": 8,
            "solvers": ("bicgstab", "gmres"), "bounds": _slab_bounds(nx, ny, nz, world)}
    parts = _run(case, world)
    y = np.concatenate([p["y"] for p in parts])
    assert y.tobytes() == sparse_ref.spmv(m, x).tobytes()
    spmv = lambda v: sparse_ref.spmv(m, v)  # noqa: E731
    nnz = sparse_ref.row_nnz(m)
    for kind, ref in (("bicgstab", krylov_ref.bicgstab_solve(spmv, b, 1e-10, 200)),
                      ("gmres", krylov_ref.gmres_solve(spmv, b, 1e-10, 200, restart=8))):
        xr, hr = ref
        hists = [p[kind][1] for p in parts]
        for h in hists[1:]:
            assert np.array_equal(h, hists[0]), kind  # identical control on every rank
        assert len(hists[0]) == len(hr), (kind, len(hists[0]), len(hr))
        assert np.max(np.abs(hists[0] - hr)) / np.linalg.norm(b) <= 1e-10, kind
        xd = np.concatenate([p[kind][0] for p in parts])
        assert sparse_ref.max_scaled_rel_err(xd, xr, nnz) <= 1e-10, kind


@pytest.mark.parametrize("world", [4, 8])
def test_distributed_cg_world(world):
    nx, ny, nz = 6, 6, 3 * world
    m = corpus_ref.stencil(nx, ny, nz, corpus_ref.points_7pt())
    b = np.ones(m.nrows)
    parts = _run({"matrix": m, "x": np.zeros(m.nrows), "cg": True, "b": b, "tol": 1e-10, "max_iters": 500,
                  "bounds": _slab_bounds(nx, ny, nz, world)}, world)
    sp = sparse_ref.csr_to_sellp(m, 64)
    xr, hr = krylov_ref.cg_solve(lambda v: sparse_ref.spmv(sp, v), b, 1e-10, 500)
    for p in parts[1:]:
        assert np.array_equal(p["hist"], parts[0]["hist"])
    assert len(parts[0]["hist"]) == len(hr)
    assert np.max(np.abs(parts[0]["hist"] - hr)) / np.linalg.norm(b) <= 1e-10
    x = np.concatenate([p["x"] for p in parts])
    assert sparse_ref.max_scaled_rel_err(x, xr, sparse_ref.row_nnz(m)) <= 1e-10


@pytest.mark.parametrize("where", ["alloc", "open"])
def test_peer_setup_failure_falls_back_on_every_rank(where):
    """One rank failing the peer-arena set-up (allocation or IPC open) makes
    maybe_enable_peer fall back to the process-group path on ALL ranks (no
    rank left waiting in a peer kernel), and the SpMV stays bitwise."""
    m = corpus_ref.stencil(6, 5, 8, corpus_ref.points_27pt())
    x = np.random.default_rng(5).standard_normal(m.nrows)
    parts = _run({"matrix": m, "x": x, "peer_fail": where})
    assert [p["mode"] for p in parts] == ["gloo", "gloo"]
    assert not any(p["peer"] for p in parts)
    y = np.concatenate([p["y"] for p in parts])
    assert y.tobytes() == sparse_ref.spmv(m, x).tobytes()
