"""Row-block partitioned SpMV and Krylov solves across the GPUs of one box.

SURVEY.md §8(e). One process per GPU (torch.distributed, NCCL over NVLink /
NVSwitch); the reference has no distributed code at all.

Partition: rank g owns the contiguous rows [row_lo_g, row_hi_g) (boundaries
multiples of 64, so SELL-P slices never straddle ranks). Its local matrix
keeps every row's entries in the GLOBAL column order, with columns renumbered
into the rank's extended vector x_ext = [owned (n_local) | halo (n_halo)]:
owned column c -> c - row_lo, non-owned column -> n_local + position in the
sorted list of needed remote columns. Because entries stay in global order,
the local fold is the global fold: the distributed SpMV is bitwise equal to
the single-GPU one.

Per SpMV: pack the entries of x the neighbours need (wk_gather_f64), one
grouped NCCL send/recv (torch.distributed.batch_isend_irecv) straight into
the halo segment of x_ext, then the local SpMV kernel. Dot products: the
local partial (written into a device state by the fused CG kernels) is
all-reduced in place (NCCL returns bit-identical sums on every rank, so the
device-side convergence decisions agree everywhere).

For CPU testing, `LocalOps` can be swapped (tests inject a numpy/oracle
implementation and run world-size-2 gloo groups); with the gloo backend,
CUDA tensors are staged through host memory.
"""

import ctypes
import os

import numpy as np
import torch

from . import _lib
from . import device as D
from .errors import BreakdownError, DimensionMismatch

ALIGN = 64


# ---- communication -------------------------------------------------------------------------


class Comm:
    """Thin wrapper over a torch.distributed process group."""

    def __init__(self, dist=None, group=None):
        import torch.distributed as tdist

        self.dist = dist if dist is not None else tdist
        self.group = group
        self.rank = self.dist.get_rank(group)
        self.world = self.dist.get_world_size(group)
        self.backend = str(self.dist.get_backend(group)).lower()
        self.peer = None  # PeerComm once an operator enables the peer-memory path

    def _staged(self, t):
        return self.backend == "gloo" and t.is_cuda

    def allreduce_(self, t):
        """In-place sum all-reduce (NCCL is called even for a single rank, so
        the graph-captured path is the same code at every world size); the
        peer-memory kernel once `DistOperator.enable_peer` ran."""
        if self.peer is not None:
            return self.peer.allreduce_(t)
        if self.world == 1 and self.backend != "nccl":
            return t
        if self._staged(t):
            h = t.cpu()
            self.dist.all_reduce(h, group=self.group)
            t.copy_(h)
        else:
            self.dist.all_reduce(t, group=self.group)
        return t

    def max_scalar(self, v):
        """Max of a host float over ranks (timing: max over ranks)."""
        if self.world == 1:
            return float(v)
        dev = "cpu" if self.backend == "gloo" else "cuda"
        t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def allgather_obj(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def exchange(self, sends, recvs):
        """sends: [(peer, tensor)], recvs: [(peer, tensor view)] — one
        grouped send/recv round (NCCL group / gloo P2P)."""
        if not sends and not recvs:
            return
        if self.backend == "gloo":
            ops, staged = [], []
            for peer, t in sends:
                ops.append(self.dist.P2POp(self.dist.isend, t.cpu() if t.is_cuda else t, peer, self.group))
            for peer, t in recvs:
                h = torch.empty(t.shape, dtype=t.dtype) if t.is_cuda else t
                staged.append((h, t))
                ops.append(self.dist.P2POp(self.dist.irecv, h, peer, self.group))
            for r in self.dist.batch_isend_irecv(ops):
                r.wait()
            for h, t in staged:
                if h is not t:
                    t.copy_(h)
            return
        ops = [self.dist.P2POp(self.dist.isend, t, peer, self.group) for peer, t in sends]
        ops += [self.dist.P2POp(self.dist.irecv, t, peer, self.group) for peer, t in recvs]
        for r in self.dist.batch_isend_irecv(ops):
            r.wait()

    def barrier(self):
        self.dist.barrier(group=self.group)


# ---- local compute backends -------------------------------------------------------------------


class DeviceOps:
    """Local kernels of libwk_sparse (the product path)."""

    def __init__(self, device=None):
        self.device = D._dev(device)
        self.ws = D.workspace(self.device)

    def stream(self):
        return D.stream_handle(self.device)

    def zeros(self, n):
        return torch.zeros(n, dtype=torch.float64, device=self.device)

    def index(self, arr):
        return torch.as_tensor(np.asarray(arr, dtype=np.int32), device=self.device)

    def gather(self, idx, src, dst):
        _lib.call("wk_gather_f64", idx.numel(), D._ptr(idx), D._ptr(src), D._ptr(dst), self.stream())

    def spmv(self, local, x_ext, y):
        _lib.call("wk_spmv", local.wk_ptr(), D._ptr(x_ext), D._ptr(y), self.stream())

    def spmv_masked(self, local, x_ext, y, state):
        done = ctypes.c_void_p(state.data_ptr() + _lib.WkCgState.done.offset)
        _lib.call("wk_spmv_masked", local.wk_ptr(), D._ptr(x_ext), D._ptr(y), done, self.stream())

    def spmv_dot(self, local, p_ext, q, state):
        """q = A p and state.pq = p.q (local part) in one fused pass."""
        _lib.call("wk_cg_spmv_dot", local.wk_ptr(), D._ptr(p_ext), D._ptr(q), D._ptr(state), D._ptr(self.ws.red),
                  self.stream())

    # CG building blocks (state = 80-byte wk_cg_state in a uint8 tensor)
    def new_state(self):
        return torch.zeros(ctypes.sizeof(_lib.WkCgState), dtype=torch.uint8, device=self.device)

    def cg(self, name, *args):
        conv = [D._ptr(a) if isinstance(a, torch.Tensor) else a for a in args]
        if name in ("wk_cg_init_local", "wk_cg_dot_pq", "wk_cg_update_xr", "wk_cg_replace_r", "wk_cg_update_xr_alpha",
                    "wk_cg_update_p_beta"):
            conv.append(D._ptr(self.ws.red))
        _lib.call(name, *conv, self.stream())

    def read_state(self, state, cls=None):
        return (cls or _lib.WkCgState).from_buffer_copy(state.cpu().numpy().tobytes())

    # generic step call: tensors -> device pointers, workspace appended on request
    def step(self, name, *args, ws=False):
        conv = [D._ptr(a) if isinstance(a, torch.Tensor) else a for a in args]
        if ws:
            conv.append(D._ptr(self.ws.red))
        _lib.call(name, *conv, self.stream())

    def new_struct(self, cls):
        return torch.zeros(ctypes.sizeof(cls), dtype=torch.uint8, device=self.device)

    def spmv_flag(self, local, x_ext, y, state, offset):
        """y = A x, skipped while the int32 flag at `state + offset` is set."""
        flag = ctypes.c_void_p(state.data_ptr() + offset)
        _lib.call("wk_spmv_masked", local.wk_ptr(), D._ptr(x_ext), D._ptr(y), flag, self.stream())

    def bicg_spmv_dots(self, local, x_ext, y, state, w, mode):
        """BiCGSTAB SpMV with its local dot(s) fused (mode 1: r-hat.v into rv,
        mode 2: t.t / t.s into tt / ts; wk_bicg_spmv_dots)."""
        _lib.call("wk_bicg_spmv_dots", local.wk_ptr(), D._ptr(x_ext), D._ptr(y), D._ptr(state),
                  D._ptr(w) if w is not None else None, mode, D._ptr(self.ws.red), self.stream())


# ---- partition plans ----------------------------------------------------------------------------


def row_blocks(nrows, world, align=ALIGN):
    """Contiguous row ranges, boundaries multiples of `align`."""
    units = (nrows + align - 1) // align
    bounds = [min(nrows, (units * g // world) * align) for g in range(world + 1)]
    bounds[-1] = nrows
    return bounds


class HaloPlan:
    """Which entries of x go to / come from which rank."""

    def __init__(self, n_local, halo_cols, send_idx, recv_ranges):
        self.n_local = n_local
        self.halo_cols = halo_cols          # sorted global ids of the halo (np.int64)
        self.n_halo = len(halo_cols)
        self.send_idx = send_idx            # {peer: local owned indices (np.int64)}
        self.recv_ranges = recv_ranges      # {peer: (offset into halo, count)}

    @property
    def bytes_per_exchange(self):
        return 8 * (sum(len(v) for v in self.send_idx.values()) + self.n_halo)


def _plan_from_needs(rank, bounds, needed_by_rank):
    """needed_by_rank[q] = sorted global columns rank q needs from others."""
    lo, hi = bounds[rank], bounds[rank + 1]
    mine = needed_by_rank[rank]
    recv = {}
    for q in range(len(bounds) - 1):
        if q == rank:
            continue
        a = np.searchsorted(mine, bounds[q])
        b = np.searchsorted(mine, bounds[q + 1])
        if b > a:
            recv[q] = (int(a), int(b - a))
    send = {}
    for q, need in enumerate(needed_by_rank):
        if q == rank:
            continue
        a = np.searchsorted(need, lo)
        b = np.searchsorted(need, hi)
        if b > a:
            send[q] = need[a:b] - lo
    return HaloPlan(hi - lo, mine, send, recv)


def localize_columns(cols, lo, hi, halo_cols):
    """Global -> extended-local column ids (owned first, then halo)."""
    cols = np.asarray(cols, dtype=np.int64)
    out = cols - lo
    remote = (cols < lo) | (cols >= hi)
    out[remote] = (hi - lo) + np.searchsorted(halo_cols, cols[remote])
    return out


class DistOperator:
    """Rank-local piece of a row-block partitioned matrix."""

    def __init__(self, comm, bounds, plan, local, local_nnz, ops=None, nrows_global=None):
        self.comm = comm
        self.bounds = bounds
        self.plan = plan
        self.local = local
        self.local_nnz = int(local_nnz)
        self.ops = ops if ops is not None else DeviceOps()
        self.n_local = plan.n_local
        self.n_halo = plan.n_halo
        self.nrows_global = nrows_global if nrows_global is not None else bounds[-1]
        self.row_lo = bounds[comm.rank]
        self._send_idx = {q: self.ops.index(v) for q, v in plan.send_idx.items()}
        self._send_buf = {q: self.ops.zeros(len(v)) for q, v in plan.send_idx.items()}
        self.launches_per_spmv = 1 + len(self._send_idx)
        self.peer = None
        self.n_ext_max = self.n_local + self.n_halo

    def enable_peer(self, vectors=40):
        """Switch halo exchange and all-reduces to the peer-memory kernels
        (peer.py / csrc/peer.cu): a symmetric arena per rank sized for
        `vectors` distributed vectors, IPC-opened by every rank. Collective
        over the group. Vectors made by `new_vector` afterwards live in the
        arena (same offsets on every rank)."""
        from . import peer as PE

        comm = self.comm
        info = comm.allgather_obj((self.n_local, self.n_local + self.n_halo,
                                   {q: off for q, (off, cnt) in self.plan.recv_ranges.items()}))
        self.n_ext_max = max(e for _, e, _ in info)
        if comm.peer is None:
            comm.peer = PE.PeerComm(comm, PE.arena_bytes_for(self.n_ext_max, vectors), self.ops.device)
        self.peer = comm.peer
        # where my data lands in each receiver's copy of a vector (element offset)
        self._peer_dst = {q: info[q][0] + info[q][2][comm.rank] for q in self._send_idx}
        self._peer_recv = sorted(self.plan.recv_ranges)
        self.launches_per_spmv = 2
        return self

    @property
    def stored(self):
        return getattr(self.local, "stored", self.local_nnz)

    def disable_peer(self):
        if self.peer is not None:
            self.peer.close()
        self.peer = None
        self.comm.peer = None
        self.n_ext_max = self.n_local + self.n_halo
        self.launches_per_spmv = 1 + len(self._send_idx)

    def new_vector(self):
        """Zeroed vector with halo room: [n_local | n_halo] (in the peer arena
        when the peer-memory path is enabled)."""
        if self.peer is not None:
            return self.peer.vector(self.n_local + self.n_halo, self.n_ext_max)
        return self.ops.zeros(self.n_local + self.n_halo)

    def peer_halo(self, vec):
        """Device `wk_peer_halo` for pushing `vec`'s boundary rows from the
        kernel that writes them, or None when a send set is not a contiguous
        row range (then the exchange kernel runs instead)."""
        if self.peer is None or len(self._send_idx) > 8 or len(self._peer_recv) > 8:
            return None
        off = self.peer.offset_of(vec)
        if off is None:
            return None
        h = _lib.WkPeerHalo()
        h.n = len(self._send_idx)
        for j, (q, idx_h) in enumerate(sorted(self.plan.send_idx.items())):
            idx_h = np.asarray(idx_h, dtype=np.int64)
            lo = int(idx_h[0]) if len(idx_h) else 0
            if len(idx_h) and not np.array_equal(idx_h, np.arange(lo, lo + len(idx_h))):
                return None
            h.peer[j], h.lo[j], h.hi[j] = q, lo, lo + len(idx_h)
            h.dst_off[j] = off + 8 * self._peer_dst[q]
        h.nrecv = len(self._peer_recv)
        for j, q in enumerate(self._peer_recv):
            h.recv_peer[j] = q
        h.int_lo, h.int_hi = self._interior_slices()
        t = torch.frombuffer(bytearray(bytes(h)), dtype=torch.uint8).to(self.ops.device)
        self._halo_keep = getattr(self, "_halo_keep", []) + [t]
        return t

    def _interior_slices(self):
        """Longest run [lo, hi) of local SELL-P slices with no halo column
        (entries with column >= n_local); (0, 0) when unknown or empty. The
        fused SpMV folds those before waiting for the halo."""
        L = self.local
        if getattr(L, "fmt", None) != "sellp" or L.nrows == 0:
            return 0, 0
        if getattr(self, "_int_range", None) is None:
            ss = int(L.slice_size)
            nsl = (L.nrows + ss - 1) // ss
            idx = torch.nonzero(L.col_idx >= self.n_local).flatten()
            if idx.numel() == 0:
                self._int_range = (0, nsl)
            else:
                starts = L.slice_sets.to(torch.int64) * ss
                sl = torch.searchsorted(starts, idx.to(torch.int64), right=True) - 1
                pts = np.concatenate(([-1], torch.unique(sl).cpu().numpy(), [nsl]))
                gaps = np.diff(pts) - 1
                g = int(np.argmax(gaps))
                self._int_range = (int(pts[g] + 1), int(pts[g + 1])) if gaps[g] > 0 else (0, 0)
        return self._int_range

    def arena_mark(self):
        """Allocation mark of the peer arena (None without the peer path)."""
        return None if self.peer is None else self.peer.mark()

    def arena_release(self, mark):
        """Free every arena vector allocated after `mark` (the same sequence on
        all ranks keeps the offsets in step)."""
        if mark is not None and self.peer is not None:
            self.peer.release(mark)

    def new_block(self, count, ld):
        """`count` vectors of leading dimension `ld` (>= n_ext_max on every
        rank when the peer path is on), zeroed, contiguous."""
        if self.peer is not None:
            return self.peer.vector(count * ld)
        return self.ops.zeros(count * ld)

    def exchange(self, x_ext):
        if self.peer is not None:
            off = self.peer.offset_of(x_ext)
            if off is None:
                raise ValueError("peer exchange needs a vector made by DistOperator.new_vector / new_block")
            sends = [(q, idx, off + 8 * self._peer_dst[q]) for q, idx in self._send_idx.items()]
            self.peer.exchange(x_ext, sends, self._peer_recv)
            return
        sends = []
        for q, idx in self._send_idx.items():
            buf = self._send_buf[q]
            self.ops.gather(idx, x_ext, buf)
            sends.append((q, buf))
        recvs = [(q, x_ext[self.n_local + off: self.n_local + off + cnt])
                 for q, (off, cnt) in self.plan.recv_ranges.items()]
        self.comm.exchange(sends, recvs)

    def spmv(self, x_ext, y):
        """y[:n_local] = (A x)[rows of this rank]; x_ext's owned part must be
        current, its halo part is refreshed here."""
        self.exchange(x_ext)
        self.ops.spmv(self.local, x_ext, y)
        return y

    def algorithmic_bytes(self):
        return self.local.algorithmic_bytes()

    def e2e(self, x, args, timed):
        """End-to-end SpMV through this API with host buffers (pinned host x
        slice in, host y out) — used by bench.py at N > 1."""
        xh = x[: self.n_local].cpu().pin_memory()
        yh = torch.empty(self.n_local, dtype=torch.float64, pin_memory=True)
        x_ext = self.new_vector()
        y = self.ops.zeros(self.n_local)

        def step():
            x_ext[: self.n_local].copy_(xh, non_blocking=True)
            self.spmv(x_ext, y)
            yh.copy_(y, non_blocking=True)
            torch.cuda.current_stream().synchronize()

        steps = max(3, args.steps // 2)
        ms, _ = timed(step, steps, 2, self.comm.dist)
        ms = self.comm.max_scalar(ms)
        return {"value": round(2.0 * self.local_nnz * self.comm.world * steps / (ms * 1e-3) / 1e9, 3),
                "unit": "GFLOP/s", "h2d_bytes_per_step": int(8 * self.n_local * self.comm.world),
                "d2h_bytes_per_step": int(8 * self.n_local * self.comm.world),
                "ms_per_step": round(ms / steps, 4), "api": "distributed.DistOperator.spmv (pinned host x/y)"}


def maybe_enable_peer(op, vectors=40):
    """The peer-memory path (NVLink stores into the other ranks' IPC-mapped
    arenas, no NCCL on the data path) unless WK_DIST_COMM=nccl; falls back to
    NCCL on every rank if any rank cannot set it up (collective decision).
    Returns "peer" or the process group's backend."""
    import warnings

    if os.environ.get("WK_DIST_COMM", "peer") != "peer" or op.comm.world == 1:
        return op.comm.backend
    try:
        op.enable_peer(vectors)
        return "peer"
    except Exception as exc:  # pragma: no cover - depends on the box
        warnings.warn(f"peer-memory path unavailable ({exc}); using {op.comm.backend}")
        op.peer = None
        op.comm.peer = None
        return op.comm.backend


def _check_peer(op):
    if op.peer is not None:
        op.peer.check()


def _convert_local(dcsr, fmt, slice_size):
    if fmt == "csr":
        return dcsr
    if fmt == "sellp":
        return D.csr_to_sellp(dcsr, slice_size)
    if fmt == "ell":
        return D.csr_to_ell(dcsr)
    if fmt == "hybrid":
        return D.csr_to_hybrid(dcsr)
    if fmt == "coo":
        return D.csr_to_coo(dcsr)
    raise ValueError(f"unknown format {fmt!r}")


def partition_csr(m, comm, fmt="sellp", slice_size=64, ops=None, bounds=None, upload=None):
    """Partition a global CSR (host object with row_ptrs/col_idx/values, the
    same on every rank) into row blocks. Returns this rank's DistOperator."""
    n = m.nrows
    if m.ncols != n:
        raise DimensionMismatch("row-block partitioning needs a square matrix")
    bounds = row_blocks(n, comm.world) if bounds is None else bounds
    ptrs = np.asarray(m.row_ptrs, dtype=np.int64)
    cols = np.asarray(m.col_idx, dtype=np.int64)
    vals = np.asarray(m.values, dtype=np.float64)
    needed = []
    for q in range(comm.world):
        lo, hi = bounds[q], bounds[q + 1]
        c = cols[ptrs[lo]:ptrs[hi]]
        needed.append(np.unique(c[(c < lo) | (c >= hi)]))
    plan = _plan_from_needs(comm.rank, bounds, needed)
    lo, hi = bounds[comm.rank], bounds[comm.rank + 1]
    lp = ptrs[lo:hi + 1] - ptrs[lo]
    lc = localize_columns(cols[ptrs[lo]:ptrs[hi]], lo, hi, plan.halo_cols)
    lv = vals[ptrs[lo]:ptrs[hi]]
    ncols_ext = (hi - lo) + plan.n_halo
    if upload is not None:
        local = upload(hi - lo, ncols_ext, lp, lc, lv)
    else:
        from types import SimpleNamespace

        dcsr = D.upload(SimpleNamespace(nrows=hi - lo, ncols=ncols_ext, row_ptrs=lp, col_idx=lc, values=lv),
                        (ops or DeviceOps()).device)
        local = _convert_local(dcsr, fmt, slice_size)
    return DistOperator(comm, bounds, plan, local, len(lv), ops, n)


class SlabLayout:
    """z-slab partition of an nx*ny*nzg stencil grid over P ranks (host index
    logic only, shared by the device operator and the CPU tests).

    weak=True: every rank owns nz_local planes of an nx*ny*(nz_local*P) grid;
    weak=False: the global grid has `nz` planes split as evenly as possible.
    Rank g owns planes [z0, z1) plus one halo plane on each side that exists
    (the stencils here reach +-1 plane); its extended slab is planes
    [e0, e1)."""

    def __init__(self, nx, ny, P, g, weak=True, nz_local=None, nz=None):
        self.plane = plane = nx * ny
        if weak:
            self.nzg = nz_local * P
            zb = [nz_local * q for q in range(P + 1)]
        else:
            self.nzg = nz
            zb = [nz * q // P for q in range(P + 1)]
        z0, z1 = zb[g], zb[g + 1]
        self.z0, self.z1 = z0, z1
        self.has_lo, self.has_hi = z0 > 0, z1 < self.nzg
        self.e0, self.e1 = z0 - int(self.has_lo), z1 + int(self.has_hi)
        self.n_local = (z1 - z0) * plane
        self.lo_rows = int(self.has_lo) * plane     # rows of the extended slab before the owned ones
        self.n_halo = (int(self.has_lo) + int(self.has_hi)) * plane
        self.bounds = [z * plane for z in zb]
        halo_cols, recv, send = [], {}, {}
        if self.has_lo:
            halo_cols.append(np.arange((z0 - 1) * plane, z0 * plane, dtype=np.int64))
            recv[g - 1] = (0, plane)
            send[g - 1] = np.arange(0, plane, dtype=np.int64)
        if self.has_hi:
            halo_cols.append(np.arange(z1 * plane, (z1 + 1) * plane, dtype=np.int64))
            recv[g + 1] = (int(self.has_lo) * plane, plane)
            send[g + 1] = np.arange(self.n_local - plane, self.n_local, dtype=np.int64)
        hc = np.concatenate(halo_cols) if halo_cols else np.zeros(0, np.int64)
        self.plan = HaloPlan(self.n_local, hc, send, recv)

    def localize(self, col):
        """Extended-slab column ids (torch int64, any device) -> [owned |
        halo lo plane | halo hi plane] local ids."""
        owned_lo, owned_hi, n_local = self.lo_rows, self.lo_rows + self.n_local, self.n_local
        lcol = col - owned_lo
        if self.has_lo:
            lcol = torch.where(col < owned_lo, n_local + col, lcol)
        if self.has_hi:
            lcol = torch.where(col >= owned_hi, n_local + self.lo_rows + (col - owned_hi), lcol)
        return lcol


def stencil_slab_operator(nx, ny, nz_local, points, dist=None, fmt="sellp", slice_size=64, weak=True, nz=None):
    """z-slab partition of a stencil matrix generated on the device (see
    SlabLayout): each rank generates only its planes plus one halo plane on
    each side."""
    from . import corpus

    comm = Comm(dist)
    lay = SlabLayout(nx, ny, comm.world, comm.rank, weak, nz_local, nz)
    ext = corpus.stencil(nx, ny, lay.e1 - lay.e0, points)          # device CSR of the extended slab
    n_local = lay.n_local
    ptrs = ext.row_ptrs[lay.lo_rows: lay.lo_rows + n_local + 1]
    base = int(ptrs[0].item())
    nnz = int(ptrs[-1].item()) - base
    col = ext.col_idx[base: base + nnz].to(torch.int64)
    val = ext.values[base: base + nnz]
    lcol = lay.localize(col)
    dcsr = D.DeviceCsr(n_local, n_local + lay.n_halo, (ptrs - base).contiguous(), lcol.to(torch.int32).contiguous(),
                       val.contiguous())
    del ext
    local = _convert_local(dcsr, fmt, slice_size)
    return DistOperator(comm, lay.bounds, lay.plan, local, nnz, DeviceOps(), lay.nzg * lay.plane)


# ---- distributed CG -------------------------------------------------------------------------------

_RHO, _PQ, _RR = 0, 1, 2  # float64 slots of wk_cg_state


REPLACE_EVERY = 50  # kernels.py:322, kReplaceEvery in krylov.cu


def cg_solve(op: DistOperator, b_local, tol, max_iters, graph=None, fused=True):
    """Row-block distributed CG with the reference's update order
    (kernels.py:283-331), all scalars on the device. Returns (x_local, hist)
    (device tensors). Iteration control is identical on all ranks because
    the all-reduced scalars are bit-identical.

    Per iteration: halo exchange of p, q = A p with p.q fused (local), one
    all-reduce, x/r update with the alpha step fused (local r.r), one
    all-reduce, p update with the beta step fused; every 50th iteration the
    true residual b - A x (exchange of x). With NCCL the 50-iteration period
    is captured once as a CUDA graph (kernels + NCCL ops; host reads the
    device `done` flag between replays); `graph=False` or WK_DIST_GRAPH=0
    keeps the eager loop (always eager for gloo).
    """
    ops, comm = op.ops, op.comm
    n = op.n_local
    if tol <= 0:
        raise ValueError("tol must be positive")
    mark = op.arena_mark()
    b = b_local
    x = op.new_vector()
    r = ops.zeros(n)
    p = op.new_vector()
    q = ops.zeros(n)
    hist = ops.zeros(int(max_iters) + 1)
    st = ops.new_state()
    f64 = st.view(torch.float64)
    ops.cg("wk_cg_init_local", n, b, x, r, p, st)
    comm.allreduce_(f64[_RHO:_RHO + 1])
    ops.cg("wk_cg_init_finish", st, float(tol), int(max_iters), hist)

    def period():
        """One residual-replacement period: iterations 50k+1 .. 50k+50."""
        for j in range(1, REPLACE_EVERY + 1):
            op.exchange(p)
            ops.spmv_dot(op.local, p, q, st)
            comm.allreduce_(f64[_PQ:_PQ + 1])
            ops.cg("wk_cg_update_xr_alpha", n, p, q, x, r, st)
            if j == REPLACE_EVERY:
                op.exchange(x)
                ops.spmv_masked(op.local, x, q, st)
                ops.cg("wk_cg_replace_r", n, b, q, r, st)
            comm.allreduce_(f64[_RR:_RR + 1])
            ops.cg("wk_cg_update_p_beta", n, r, p, x, st, hist)

    halo = op.peer_halo(p) if (op.peer is not None and fused) else None

    def period_fused():
        """The same period on the peer-memory path with both all-reduces fused
        into the kernels (producer epilogue push, consumer prologue wait) and,
        for contiguous boundary rows (slabs), the halo of p stored by the
        p-update kernel itself and awaited by the SpMV: one iteration is
        three kernels and no communication kernel."""
        pc = op.peer.ctx_dev
        for j in range(1, REPLACE_EVERY + 1):
            if halo is None:
                op.exchange(p)
            ops.step("wk_cg_spmv_dot_peer", op.local.wk_ptr(), p, q, st, ops.ws.red, pc, halo)
            ops.step("wk_cg_update_xr_alpha_peer", n, p, q, x, r, st, ops.ws.red, pc)
            if j == REPLACE_EVERY:
                op.exchange(x)
                ops.spmv_masked(op.local, x, q, st)
                ops.step("wk_cg_replace_r_peer", n, b, q, r, st, ops.ws.red, pc)
            ops.step("wk_cg_update_p_beta_peer", n, r, p, x, st, hist, ops.ws.red, pc, halo)

    if op.peer is not None and fused:
        period = period_fused  # noqa: F811
        if halo is not None:
            op.exchange(p)  # iteration 1's halo (later ones come from the p-update kernel)

    if graph is None:
        graph = (comm.backend == "nccl" or comm.peer is not None) and os.environ.get("WK_DIST_GRAPH", "1") != "0"
    g = None
    first = True
    while not ops.read_state(st).done:
        if g is None and graph and not first:
            g = _capture(period)
            if g is None:
                graph = False
        if g is not None:
            g.replay()
        else:
            period()
        first = False
    h = ops.read_state(st)
    _check_peer(op)
    x = x[:n].clone() if mark is not None else x[:n]
    del g, period
    op.arena_release(mark)
    if h.breakdown:
        raise BreakdownError(f"p.Ap <= 0 at iteration {h.iteration}; system is not SPD")
    return x, hist[: h.iteration + 1]


def _capture(fn):
    """Capture fn() (kernels + NCCL collectives) into a CUDA graph; None if the
    capture is refused (the caller then stays eager). The first period always
    runs eagerly, so communicators and caches exist before the capture."""
    try:
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, capture_error_mode="thread_local"):
            fn()
        torch.cuda.synchronize()
        return g
    except Exception as exc:  # pragma: no cover - depends on the NCCL build
        import warnings

        warnings.warn(f"CUDA graph capture of the distributed CG period failed ({exc}); running eagerly")
        torch.cuda.synchronize()
        return None


def _slot(cls, name):
    return getattr(cls, name).offset // 8


def _run_periods(ops, comm, st, cls, period, graph):
    """Replay `period` until the device `done` flag of state `st` is set;
    CUDA-graph captured after the first (eager) period when `graph`."""
    if graph is None:
        graph = (comm.backend == "nccl" or comm.peer is not None) and os.environ.get("WK_DIST_GRAPH", "1") != "0"
    g = None
    first = True
    while not ops.read_state(st, cls).done:
        if g is None and graph and not first:
            g = _capture(period)
            if g is None:
                graph = False
        if g is not None:
            g.replay()
        else:
            period()
        first = False
    return ops.read_state(st, cls)


def bicgstab_solve(op: DistOperator, b_local, tol, max_iters, graph=None, chunk=10):
    """Row-block distributed BiCGSTAB (oracle/krylov_ref.py order): four
    all-reduces per iteration (rh.v, s.s, {t.t, t.s}, {r.r, next rh.r}) and two
    halo exchanges (p before v = A p, s before t = A s); the dots are summed
    inside the SpMVs and the x/r update. Returns (x_local, hist)."""
    ops, comm = op.ops, op.comm
    n = op.n_local
    if tol <= 0:
        raise ValueError("tol must be positive")
    C = _lib.WkBicgState
    mark = op.arena_mark()
    x = ops.zeros(n)
    r, rh, v, t = ops.zeros(n), ops.zeros(n), ops.zeros(n), ops.zeros(n)
    p, sv = op.new_vector(), op.new_vector()
    hist = ops.zeros(int(max_iters) + 1)
    st = ops.new_struct(C)
    f = st.view(torch.float64)
    done = C.done.offset

    def red(*names):
        lo = _slot(C, names[0])
        comm.allreduce_(f[lo:lo + len(names)])

    ops.step("wk_bicg_init", n, b_local, x, r, rh, p, v, st, ws=True)
    red("rr")
    ops.step("wk_bicg_init_finish", st, float(tol), int(max_iters), hist)
    # the fused order of wk_bicgstab_solve: r-hat.v / t.t, t.s summed inside the
    # SpMVs, r-hat.r of the next iteration inside the x/r update (all-reduced
    # together with r.r): four all-reduces per iteration instead of five
    ops.step("wk_bicg_rho_first", n, rh, r, st, ws=True)
    red("rho_next")

    def period():
        for _ in range(chunk):
            ops.step("wk_bicg_take_rho", st)
            ops.step("wk_bicg_step_beta", st)
            ops.step("wk_bicg_update_p", n, r, v, p, st)
            op.exchange(p)
            ops.bicg_spmv_dots(op.local, p, v, st, rh, 1)
            red("rv")
            ops.step("wk_bicg_step_alpha", st)
            ops.step("wk_bicg_update_s", n, r, v, sv, st, ws=True)
            red("ss")
            ops.step("wk_bicg_step_s", st, hist)
            ops.step("wk_bicg_half_x", n, p, x, st, ws=True)
            op.exchange(sv)
            ops.bicg_spmv_dots(op.local, sv, t, st, None, 2)
            red("tt", "ts")
            ops.step("wk_bicg_step_omega", st)
            ops.step("wk_bicg_update_xr_rho", n, p, sv, t, rh, x, r, st, ws=True)
            red("rr", "rho_next")
            ops.step("wk_bicg_step_r", st, hist)

    h = _run_periods(ops, comm, st, C, period, graph)
    _check_peer(op)
    del period
    op.arena_release(mark)
    if h.breakdown:
        raise BreakdownError(f"BiCGSTAB breakdown at iteration {h.iteration}")
    return x, hist[: h.iteration + 1]


def gmres_solve(op: DistOperator, b_local, tol, max_iters, restart=30, graph=None):
    """Row-block distributed restarted GMRES(m) with classical Gram-Schmidt:
    per Arnoldi step one halo exchange, one all-reduce of the j+1 batched dots
    and one of ||w||^2; Givens rotations on one device thread (replicated on
    every rank); the basis is normalised lazily (per-vector scales, no
    rescaling pass). One cycle per CUDA-graph period. Returns (x_local, hist)."""
    ops, comm = op.ops, op.comm
    n, n_ext = op.n_local, op.n_local + op.n_halo
    m = int(restart)
    if tol <= 0:
        raise ValueError("tol must be positive")
    if not (1 <= m <= 31):
        raise ValueError("restart must be in [1, 31]")
    C = _lib.WkGmresState
    mark = op.arena_mark()
    ld = ((op.n_ext_max + 31) // 32) * 32  # the same on every rank (peer arena offsets)
    V = op.new_block(m + 1, ld)
    x = op.new_vector()
    w, r = ops.zeros(n), ops.zeros(n)
    H = ops.zeros((m + 1) * m)
    cs, sn, g, y = ops.zeros(m + 1), ops.zeros(m + 1), ops.zeros(m + 1), ops.zeros(m + 1)
    sig = ops.zeros(m + 1) + 1.0  # basis scales (deferred normalisation): v_i = sig[i] u_i, sig[0] = 1
    hist = ops.zeros(int(max_iters) + 1)
    st = ops.new_struct(C)
    f = st.view(torch.float64)
    sq = _slot(C, "sq")
    done, cdone = C.done.offset, C.cycle_done.offset

    ops.step("wk_gmres_init", n, b_local, x, r, st, ws=True)
    comm.allreduce_(f[sq:sq + 1])
    ops.step("wk_gmres_init_finish", st, float(tol), int(max_iters), m, hist)

    def period():
        # deferred normalisation (as wk_gmres_solve): A u_j lands in basis slot
        # j+1 and is orthogonalised there; the scales live in `sig`
        ops.step("wk_gmres_cycle_start", n, r, V[:n_ext], g, st)
        for j in range(m):
            Vj = V[j * ld: j * ld + n_ext]
            z = V[(j + 1) * ld: (j + 1) * ld + n]
            Hj = H[j * (m + 1): j * (m + 1) + m + 1]
            op.exchange(Vj)
            ops.spmv_flag(op.local, Vj, z, st, cdone)
            ops.step("wk_gmres_multidot", n, j, V, ld, z, Hj, st, ws=True)
            comm.allreduce_(Hj[: j + 1])
            ops.step("wk_gmres_orth_scaled", n, j, V, ld, z, Hj, sig, st, ws=True)
            comm.allreduce_(f[sq:sq + 1])
            ops.step("wk_gmres_givens_scaled", j, H, cs, sn, g, sig, st, hist)
        ops.step("wk_gmres_update_x_scaled", n, V, ld, H, g, y, x, sig, st)
        op.exchange(x)
        ops.spmv_flag(op.local, x, w, st, done)
        ops.step("wk_gmres_residual", n, b_local, w, r, st, ws=True)
        comm.allreduce_(f[sq:sq + 1])
        ops.step("wk_gmres_restart", st, hist)

    h = _run_periods(ops, comm, st, C, period, graph)
    _check_peer(op)
    x = x[:n].clone() if mark is not None else x[:n]
    del period
    op.arena_release(mark)
    return x, hist[: h.iteration + 1]


def bench_cg(grid, iters, dist, timed):
    """Strong-scaling CG on the 7-point Laplacian grid^3 (bench.py, N >= 1)."""
    from . import corpus

    op = stencil_slab_operator(grid, grid, None, corpus.points_7pt(), dist, fmt="sellp", weak=False, nz=grid)
    mode = maybe_enable_peer(op)
    b = op.ops.zeros(op.n_local) + 1.0
    cg_solve(op, b, 1e-30, 50)
    torch.cuda.synchronize()
    op.comm.barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    _, hist = cg_solve(op, b, 1e-30, iters)
    t1.record()
    torch.cuda.synchronize()
    ms = op.comm.max_scalar(t0.elapsed_time(t1))
    it = len(hist) - 1
    return {"workload": f"distributed CG, 7-point Laplacian {grid}^3 z-slab partitioned over {op.comm.world} GPUs, "
                        f"SELL-P(64), tol 1e-30, {iters} iterations", "iterations": it, "ms": round(ms, 2),
            "it_per_s": round(it / (ms * 1e-3), 1), "n_gpus": op.comm.world, "scaling": "strong",
            "halo_bytes_per_spmv": op.plan.bytes_per_exchange, "comm": mode}


def bench_nonsym(grid, iters, dist):
    """Strong-scaling BiCGSTAB and GMRES(30) on the 7-point convection-
    diffusion grid^3 (BASELINE config 5), fixed iteration counts."""
    from . import corpus

    op = stencil_slab_operator(grid, grid, None, corpus.points_7pt(6.0, corpus.CONV_DIFF_BETA), dist, fmt="sellp",
                               weak=False, nz=grid)
    mode = maybe_enable_peer(op)
    b = op.ops.zeros(op.n_local) + 1.0
    out = {"comm": mode, "workload": f"distributed BiCGSTAB / GMRES(30), 7-point convection-diffusion {grid}^3 z-slab partitioned "
                       f"over {op.comm.world} GPUs, SELL-P(64), tol 1e-30, fixed iteration counts",
           "n_gpus": op.comm.world, "scaling": "strong"}
    for kind, fn in (("bicgstab", lambda it: bicgstab_solve(op, b, 1e-30, it)),
                     ("gmres", lambda it: gmres_solve(op, b, 1e-30, it, restart=30))):
        fn(4)
        torch.cuda.synchronize()
        op.comm.barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        _, hist = fn(iters[kind])
        t1.record()
        torch.cuda.synchronize()
        ms = op.comm.max_scalar(t0.elapsed_time(t1))
        it = len(hist) - 1
        out[kind] = {"iterations": it, "ms": round(ms, 2), "it_per_s": round(it / (ms * 1e-3), 2)}
    return out
