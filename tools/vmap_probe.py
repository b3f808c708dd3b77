"""CUDA-event timing of GMRES' basis scaling step (one-in / one-out vmap)
(development probe)."""
import ctypes
import sys

import torch

sys.path.insert(0, '.')
from paper_2006_14290_b200 import _lib  # noqa: E402
from paper_2006_14290_b200 import device as D  # noqa: E402

n = 1 << 27
w = torch.rand(n, dtype=torch.float64, device="cuda")
v = torch.empty_like(w)
h = _lib.WkGmresState()
h.hn = 3.0
st = torch.frombuffer(bytearray(bytes(h)), dtype=torch.uint8).to("cuda")
s = D.stream_handle()
for _ in range(3):
    _lib.call("wk_gmres_next_basis", n, D._ptr(w), D._ptr(v), D._ptr(st), s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    _lib.call("wk_gmres_next_basis", n, D._ptr(w), D._ptr(v), D._ptr(st), s)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"next_basis n=2^27: {ms:.3f} ms  {16 * n / ms / 1e6:.0f} GB/s", flush=True)
