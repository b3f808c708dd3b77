"""Peer-memory data path of the row-block distributed solvers (csrc/peer.cu).

Each rank cudaMallocs one arena, exports it with CUDA IPC and opens every
other rank's arena (handles exchanged once over the bootstrap process group);
with NVLink / NVSwitch peer access a kernel on rank g then stores straight
into rank q's memory. `PeerComm` provides

* `vector(n)`: a zeroed float64 tensor inside this rank's arena; the k-th
  vector sits at the same offset on every rank (offsets are allocated with
  the size agreed over the group), so a sender addresses the receiver's copy
  of "the same" vector without any per-call metadata;
* `allreduce_(t)`: in-place sum over ranks of up to 32 doubles, one kernel,
  the P contributions summed in rank order (bit-identical on all ranks);
* `exchange(...)`: halo exchange — gather the owned entries each neighbour
  needs and store them into the neighbour's vector halo segment, then flag.

Both are plain kernels, so the distributed solver periods (SpMV, fused
Krylov steps and communication) are captured into one CUDA graph with no NCCL
call inside. The bootstrap group (gloo or NCCL) is only used at set-up.
"""

import ctypes

import torch

from . import _lib


# ---- DLPack view over a raw device pointer (the arena is not a torch allocation)


class _DLDevice(ctypes.Structure):
    _fields_ = [("device_type", ctypes.c_int32), ("device_id", ctypes.c_int32)]


class _DLDataType(ctypes.Structure):
    _fields_ = [("code", ctypes.c_uint8), ("bits", ctypes.c_uint8), ("lanes", ctypes.c_uint16)]


class _DLTensor(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("device", _DLDevice), ("ndim", ctypes.c_int32),
                ("dtype", _DLDataType), ("shape", ctypes.POINTER(ctypes.c_int64)),
                ("strides", ctypes.POINTER(ctypes.c_int64)), ("byte_offset", ctypes.c_uint64)]


class _DLManagedTensor(ctypes.Structure):
    pass


_DELETER = ctypes.CFUNCTYPE(None, ctypes.POINTER(_DLManagedTensor))
_DLManagedTensor._fields_ = [("dl_tensor", _DLTensor), ("manager_ctx", ctypes.c_void_p), ("deleter", _DELETER)]
_NOOP = _DELETER(lambda _p: None)
_capsule_new = ctypes.pythonapi.PyCapsule_New
_capsule_new.restype = ctypes.py_object
_capsule_new.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_void_p]


def _device_tensor(ptr, n, device_index, keep):
    """float64[n] tensor aliasing device memory at `ptr` (owned elsewhere;
    the ctypes structs are appended to the list `keep` to outlive the tensor)."""
    shape = (ctypes.c_int64 * 1)(n)
    m = _DLManagedTensor()
    m.dl_tensor.data = ptr
    m.dl_tensor.device = _DLDevice(2, device_index)  # kDLCUDA
    m.dl_tensor.ndim = 1
    m.dl_tensor.dtype = _DLDataType(2, 64, 1)  # float64
    m.dl_tensor.shape = shape
    m.dl_tensor.strides = None
    m.dl_tensor.byte_offset = 0
    m.deleter = _NOOP
    keep.extend((shape, m))
    return torch.utils.dlpack.from_dlpack(_capsule_new(ctypes.addressof(m), b"dltensor", None))


class PeerComm:
    """Symmetric arenas + the peer all-reduce / halo exchange kernels."""

    def __init__(self, comm, arena_bytes, device=None):
        L = _lib.load()
        self.comm = comm
        self.rank, self.world = comm.rank, comm.world
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        self.header = int(L.wk_peer_arena_header_bytes())
        self.capacity = int(arena_bytes)
        # every step that can fail is followed by a collective agreement, so a
        # failure on one rank raises on all of them (nobody is left waiting)
        base = ctypes.c_void_p()
        handle = (ctypes.c_char * 64)()
        rc = L.wk_sym_alloc(self.capacity, ctypes.byref(base), handle)
        got = comm.allgather_obj((rc, bytes(handle)))
        if any(r != 0 for r, _ in got):
            if rc == 0:
                L.wk_sym_free(base)
            raise RuntimeError(f"peer arena allocation failed on a rank: {[r for r, _ in got]}")
        self._base = base.value
        self._opened = []
        arenas = []
        failed = None
        for q, (_, h) in enumerate(got):
            if q == self.rank:
                arenas.append(self._base)
                continue
            p = ctypes.c_void_p()
            if failed is None and L.wk_sym_open(ctypes.create_string_buffer(h, 64), ctypes.byref(p)) != 0:
                failed = _lib.last_error()
            arenas.append(p.value)
            if p.value:
                self._opened.append(p.value)
        oks = comm.allgather_obj(failed is None)
        if not all(oks):
            self.close()
            raise RuntimeError(f"peer arena mapping failed ({failed or 'on another rank'})")
        self.seq = torch.zeros(2, dtype=torch.int64, device=self.device)
        self.error = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.ticket = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.ctx = _lib.WkPeerCtx()
        self.ctx.rank, self.ctx.world = self.rank, self.world
        for q, a in enumerate(arenas):
            self.ctx.arena[q] = a
        self.ctx.seq = self.seq.data_ptr()
        self.ctx.error = self.error.data_ptr()
        # device copy of the context for the fused kernels (wk_cg_*_peer)
        self.ctx_dev = torch.frombuffer(bytearray(bytes(self.ctx)), dtype=torch.uint8).to(self.device)
        self._top = self.header
        self._keep = []

    # -- arena vectors -------------------------------------------------------------------------

    def vector(self, n, n_max=None):
        """Zeroed float64[n] in the arena; `n_max` (>= n, the same on every rank)
        reserves the slot so offsets agree across ranks."""
        n_max = n if n_max is None else n_max
        nbytes = ((8 * int(n_max) + 255) // 256) * 256
        if self._top + nbytes > self.capacity:
            raise MemoryError(f"peer arena full ({self.capacity} B); raise arena_bytes")
        off = self._top
        self._top += nbytes
        keep = []
        t = _device_tensor(self._base + off, int(n), self.device.index, keep)
        self._keep.append((off, keep))
        t.zero_()
        return t

    def mark(self):
        return self._top

    def release(self, mark):
        """Free the vectors allocated after `mark` (stack discipline; the
        caller keeps no tensor into that range)."""
        torch.cuda.current_stream(self.device).synchronize()
        self._top = int(mark)
        self._keep = [(o, k) for o, k in self._keep if o < self._top]

    def offset_of(self, t):
        """Byte offset of a tensor inside this rank's arena (None if outside)."""
        off = t.data_ptr() - self._base
        return off if 0 <= off < self.capacity else None

    # -- collectives ---------------------------------------------------------------------------

    def allreduce_(self, t):
        n = t.numel()
        st = ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        L = _lib.load()
        for lo in range(0, n, 32):
            k = min(32, n - lo)
            ptr = ctypes.c_void_p(t.data_ptr() + 8 * lo)
            _lib.check(L.wk_peer_allreduce(ctypes.byref(self.ctx), ptr, ptr, k, st), "peer all-reduce")
        return t

    def exchange(self, x_ext, sends, recv_peers):
        """sends: [(peer, device int32 index tensor, dst byte offset in the peer's arena)]."""
        L = _lib.load()
        ns = len(sends)
        peers = (ctypes.c_int32 * max(ns, 1))(*[s[0] for s in sends])
        idx = (ctypes.c_void_p * max(ns, 1))(*[s[1].data_ptr() for s in sends])
        cnt = (ctypes.c_int64 * max(ns, 1))(*[s[1].numel() for s in sends])
        dst = (ctypes.c_int64 * max(ns, 1))(*[s[2] for s in sends])
        rp = (ctypes.c_int32 * max(len(recv_peers), 1))(*recv_peers)
        st = ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        _lib.check(L.wk_peer_exchange(ctypes.byref(self.ctx), ctypes.c_void_p(x_ext.data_ptr()), ns, peers, idx, cnt,
                                      dst, len(recv_peers), rp, ctypes.c_void_p(self.ticket.data_ptr()), st),
                   "peer exchange")

    def check(self):
        """Raise if a peer wait timed out (reads one device word)."""
        e = int(self.error.item())
        if e:
            raise RuntimeError(f"peer {'all-reduce' if e == 1 else 'halo'} wait timed out on rank {self.rank}")

    def close(self):
        L = _lib.load()
        torch.cuda.synchronize(self.device)
        self.comm.barrier()  # no rank may still store into an arena that is going away
        for p in self._opened:
            L.wk_sym_close(ctypes.c_void_p(p))
        self._opened = []
        if self._base:
            L.wk_sym_free(ctypes.c_void_p(self._base))
            self._base = 0


def arena_bytes_for(n_ext_max, vectors=40):
    """Arena size for `vectors` distributed vectors of n_ext_max entries."""
    return int(_lib.load().wk_peer_arena_header_bytes()) + vectors * (((8 * int(n_ext_max) + 255) // 256) * 256)


def max_over_group(comm, v):
    return max(int(x) for x in comm.allgather_obj(int(v)))


__all__ = ["PeerComm", "arena_bytes_for", "max_over_group"]
