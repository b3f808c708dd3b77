"""Host-side logic of the peer-memory distributed path, on CPU: the offsets a
rank stores its boundary entries at in the neighbours' arenas
(`DistOperator.enable_peer`, `exchange`, `peer_halo`), checked by applying
the stores to emulated arenas and comparing every rank's halo with the global
vector. The device protocol itself (flags, waits, fused kernels) is tested on
the GPU in tests/test_distributed_peer.py."""

from types import SimpleNamespace

import numpy as np
import torch

from oracle import corpus_ref
from paper_2006_14290_b200 import distributed as DI


class FakePeer:
    """An arena per rank as a CPU tensor; `exchange` records the stores."""

    def __init__(self, cap=1 << 16):
        self.arena = torch.zeros(cap, dtype=torch.float64)
        self._top = 64  # header (elements)
        self.sent = []

    def vector(self, n, n_max=None):
        n_max = n if n_max is None else n_max
        off = self._top
        self._top += -(-n_max // 32) * 32
        return self.arena[off: off + n]

    def offset_of(self, t):
        off = t.data_ptr() - self.arena.data_ptr()
        return off if 0 <= off < 8 * self.arena.numel() else None

    def exchange(self, x_ext, sends, recv_peers):
        self.sent.append([(q, idx.clone(), dst) for q, idx, dst in sends])


class StubComm:
    def __init__(self, rank, world, gathered):
        self.rank, self.world, self.backend = rank, world, "gloo"
        self._gathered = gathered
        self.peer = None

    def allgather_obj(self, obj):
        return self._gathered


class CpuOps:
    device = torch.device("cpu")

    def index(self, arr):
        return torch.as_tensor(np.asarray(arr, dtype=np.int64))

    def zeros(self, n):
        return torch.zeros(n, dtype=torch.float64)


def _operators(m, world):
    bounds = DI.row_blocks(m.nrows, world, align=1)
    ptrs, cols = np.asarray(m.row_ptrs), np.asarray(m.col_idx)
    needed = []
    for q in range(world):
        lo, hi = bounds[q], bounds[q + 1]
        c = cols[ptrs[lo]:ptrs[hi]]
        needed.append(np.unique(c[(c < lo) | (c >= hi)]))
    plans = [DI._plan_from_needs(g, bounds, needed) for g in range(world)]
    info = [(p.n_local, p.n_local + p.n_halo, {q: off for q, (off, cnt) in p.recv_ranges.items()}) for p in plans]
    ops = []
    for g in range(world):
        comm = StubComm(g, world, info)
        comm.peer = FakePeer()
        local = SimpleNamespace(nrows=plans[g].n_local)
        ops.append(DI.DistOperator(comm, bounds, plans[g], local, 0, CpuOps()).enable_peer())
    return bounds, plans, ops


def test_peer_exchange_offsets_fill_every_halo():
    m = corpus_ref.poisson2d(13)  # 169 rows, halos of up to 2 neighbours (3 ranks)
    world = 3
    bounds, plans, ops = _operators(m, world)
    xg = np.arange(m.nrows, dtype=np.float64) * 1.5 + 7.0
    vecs = []
    for g, op in enumerate(ops):
        v = op.new_vector()
        v[: op.n_local] = torch.from_numpy(xg[bounds[g]:bounds[g + 1]])
        vecs.append(v)
        op.exchange(v)
    # apply the recorded stores to the receivers' arenas
    for g, op in enumerate(ops):
        for q, idx, dst in op.peer.sent[-1]:
            arena_q = ops[q].peer.arena
            e0 = dst // 8
            arena_q[e0: e0 + len(idx)] = vecs[g][idx]
    for g, op in enumerate(ops):
        halo = vecs[g][op.n_local:].numpy()
        assert np.array_equal(halo, xg[plans[g].halo_cols])


def test_peer_halo_descriptor_matches_exchange():
    """Slab partitions: every send set is a contiguous row range, and the
    descriptor's destinations are the ones `exchange` uses."""
    m = corpus_ref.stencil(6, 5, 8, corpus_ref.points_7pt())
    world = 4
    bounds, plans, ops = _operators(m, world)
    for g, op in enumerate(ops):
        v = op.new_vector()
        op.exchange(v)
        sends = {q: (idx, dst) for q, idx, dst in op.peer.sent[-1]}
        h = op.peer_halo(v)
        assert h is not None
        hb = DI._lib.WkPeerHalo.from_buffer_copy(bytes(h.numpy()))
        assert hb.n == len(sends) and hb.nrecv == len(plans[g].recv_ranges)
        for j in range(hb.n):
            idx, dst = sends[hb.peer[j]]
            assert (hb.lo[j], hb.hi[j]) == (int(idx[0]), int(idx[-1]) + 1)
            assert hb.dst_off[j] == dst
        assert sorted(hb.recv_peer[j] for j in range(hb.nrecv)) == sorted(plans[g].recv_ranges)


def test_peer_halo_refuses_scattered_sends():
    m = corpus_ref.poisson2d(9)
    world = 2
    _, plans, ops = _operators(m, world)
    op = ops[0]
    # make the send set non-contiguous: the descriptor must refuse (exchange kernel instead)
    q = next(iter(op.plan.send_idx))
    op.plan.send_idx[q] = np.array([0, 2, 3], dtype=np.int64)
    assert op.peer_halo(op.new_vector()) is None
