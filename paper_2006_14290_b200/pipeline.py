"""Host-to-host SpMV pipeline: y_host = A x_host with the PCIe transfers
overlapped with the kernels (the end-to-end path of the drop-in API).

A synchronous `spmv_sellp(A, x_host)` serialises copy-in (8 ncols bytes),
SpMV and copy-out (8 nrows bytes); on a B200 the two copies take ~3x the
SpMV. `SpmvPipeline` overlaps them on the GPU's independent copy engines:

* x is copied in `pieces` ordered chunks on an H2D stream (event per chunk);
* the rows are cut into `chunks` blocks of whole SELL-P slices; block c is
  launched (the same `wk_spmv_sellp_f64` entry point, on a slice sub-range:
  slice_sets / row_lengths / y offsets) as soon as the x chunks holding its
  largest column index have landed — found once per matrix from the stored
  column indices, so banded matrices (stencils) start computing after a
  fraction of x arrived and unstructured ones simply wait for all of x;
* each finished row block is copied out on a D2H stream;
* consecutive calls alternate between two device buffer sets, so step k+1's
  copy-in overlaps step k's compute / copy-out (`submit` is asynchronous;
  `synchronize` waits for everything submitted).

Results are bitwise those of the one-launch SpMV (same kernel, same per-row
fold; the sub-range launch only changes which CTA folds a slice).

Throughput is bound by the copy engines (measured on the box: 55 GB/s H2D,
57 GB/s D2H, 99.5 GB/s both at once, `tools/pcie_probe.py`); with the
cross-step overlap the SpMV already hides under the copies, so the default is
one piece / one row block (27-pt 200^3: 1.46 ms per step vs 1.81 ms with
8 blocks / 16 pieces and 2.76 ms for the synchronous call,
`tools/pipeline_probe.py`). More chunks lower the latency of the first
result rows, not the throughput.
"""

import ctypes

import numpy as np
import torch

from . import _lib
from . import device as D
from .errors import DimensionMismatch


class SpmvPipeline:
    def __init__(self, m, chunks=1, pieces=1, device=None):
        d = D.as_device(m, device)
        if d.fmt != "sellp":
            d = D.csr_to_sellp(d if d.fmt == "csr" else D.coo_to_csr(d) if d.fmt == "coo" else d, 64)
        self.A = d
        self.device = d.device
        n, nc, ss = d.nrows, d.ncols, d.slice_size
        nsl = d.nslices
        chunks = max(1, min(int(chunks), nsl))
        self.pieces = max(1, min(int(pieces), max(nc, 1)))
        sb = [nsl * c // chunks for c in range(chunks + 1)]
        self.blocks = []
        sets_h = d.slice_sets.cpu().numpy()
        piece_len = -(-max(nc, 1) // self.pieces)
        for c in range(chunks):
            s0, s1 = sb[c], sb[c + 1]
            if s1 <= s0:
                continue
            lo, hi = int(sets_h[s0]) * ss, int(sets_h[s1]) * ss
            maxcol = int(d.col_idx[lo:hi].max().item()) if hi > lo else 0
            need = min(self.pieces, maxcol // piece_len + 1)
            r0, r1 = s0 * ss, min(s1 * ss, n)
            self.blocks.append((s0, r0, r1, need))
        self.piece_bounds = [min(nc, p * piece_len) for p in range(self.pieces + 1)]
        self._sets_ptr = d.slice_sets.data_ptr()
        self._len_ptr = d.row_lengths_t.data_ptr()
        self._col_ptr, self._val_ptr = d.col_idx.data_ptr(), d.values.data_ptr()
        self.s_h2d = torch.cuda.Stream(self.device)
        self.s_cmp = torch.cuda.Stream(self.device)
        self.s_d2h = torch.cuda.Stream(self.device)
        self.bufs = [(torch.empty(nc, dtype=torch.float64, device=self.device),
                      torch.empty(n, dtype=torch.float64, device=self.device)) for _ in range(2)]
        # per buffer set: "copy-out of the previous use finished" / "compute of the previous use finished"
        self._d2h_done = [None, None]
        self._cmp_done = [None, None]
        self._k = 0
        self.launches_per_call = len(self.blocks)

    @property
    def h2d_bytes(self):
        return 8 * self.A.ncols

    @property
    def d2h_bytes(self):
        return 8 * self.A.nrows

    def submit(self, x_host: torch.Tensor, y_host: torch.Tensor):
        """Enqueue y_host = A x_host (both pinned CPU float64 tensors);
        returns immediately. The tensors must stay alive until `synchronize`."""
        A = self.A
        if x_host.numel() != A.ncols or y_host.numel() != A.nrows:
            raise DimensionMismatch(f"pipeline needs x of length {A.ncols} and y of length {A.nrows}")
        b = self._k & 1
        self._k += 1
        xd, yd = self.bufs[b]
        lib = _lib.load()
        # copy-in: may not overwrite x of buffer set b before its previous compute finished
        ev_in = []
        with torch.cuda.stream(self.s_h2d):
            if self._cmp_done[b] is not None:
                self.s_h2d.wait_event(self._cmp_done[b])
            for p in range(self.pieces):
                lo, hi = self.piece_bounds[p], self.piece_bounds[p + 1]
                if hi > lo:
                    xd[lo:hi].copy_(x_host[lo:hi], non_blocking=True)
                e = torch.cuda.Event()
                e.record(self.s_h2d)
                ev_in.append(e)
        ev_out = []
        st = ctypes.c_void_p(self.s_cmp.cuda_stream)
        if self._d2h_done[b] is not None:
            self.s_cmp.wait_event(self._d2h_done[b])  # y of buffer set b was copied out
        waited = -1
        for (s0, r0, r1, need) in self.blocks:
            if need - 1 > waited:
                self.s_cmp.wait_event(ev_in[need - 1])
                waited = need - 1
            rc = lib.wk_spmv_sellp_f64(r1 - r0, A.ncols, A.slice_size, ctypes.c_void_p(self._sets_ptr + 8 * s0),
                                       ctypes.c_void_p(self._col_ptr), ctypes.c_void_p(self._val_ptr),
                                       ctypes.c_void_p(self._len_ptr + 4 * r0), ctypes.c_void_p(xd.data_ptr()),
                                       ctypes.c_void_p(yd.data_ptr() + 8 * r0), st)
            _lib.check(rc, "SpmvPipeline")
            e = torch.cuda.Event()
            e.record(self.s_cmp)
            ev_out.append(e)
        done_c = torch.cuda.Event()
        done_c.record(self.s_cmp)
        self._cmp_done[b] = done_c
        with torch.cuda.stream(self.s_d2h):
            for (s0, r0, r1, need), e in zip(self.blocks, ev_out):
                self.s_d2h.wait_event(e)
                y_host[r0:r1].copy_(yd[r0:r1], non_blocking=True)
            done = torch.cuda.Event()
            done.record(self.s_d2h)
        self._d2h_done[b] = done
        return done

    def synchronize(self):
        for s in (self.s_h2d, self.s_cmp, self.s_d2h):
            s.synchronize()

    def __call__(self, x, out=None):
        """Synchronous convenience: host x (numpy or CPU tensor) -> host y."""
        as_np = not isinstance(x, torch.Tensor)
        xt = torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64)) if as_np else x.to(torch.float64)
        if not xt.is_pinned():
            xt = xt.pin_memory()
        y = out if out is not None else torch.empty(self.A.nrows, dtype=torch.float64, pin_memory=True)
        self.submit(xt, y)
        self.synchronize()
        return y.numpy() if as_np else y
