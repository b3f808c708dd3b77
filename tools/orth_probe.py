"""CUDA-event timing of GMRES' classical Gram-Schmidt steps (multidot and the
orthogonalisation update) for several basis sizes (development probe)."""
import ctypes
import sys

import torch

sys.path.insert(0, '.')
from paper_2006_14290_b200 import _lib  # noqa: E402
from paper_2006_14290_b200 import device as D  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
K = 31
V = torch.rand(K * n, dtype=torch.float64, device="cuda")
w = torch.rand(n, dtype=torch.float64, device="cuda")
H = torch.rand(64, dtype=torch.float64, device="cuda") * 1e-3
st = torch.zeros(ctypes.sizeof(_lib.WkGmresState), dtype=torch.uint8, device="cuda")
L = _lib.load()
ws = torch.zeros(int(L.wk_gmres_workspace_bytes(n, 30)), dtype=torch.uint8, device="cuda")
s = D.stream_handle()
P = D._ptr


def t(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for j in (1, 7, 15, 23, 29):
    tm = t(lambda: _lib.call("wk_gmres_multidot", n, j, P(V), n, P(w), P(H), P(st), P(ws), s))
    to = t(lambda: _lib.call("wk_gmres_orth", n, j, P(V), n, P(w), P(H), P(st), P(ws), s))
    bm = (j + 2) * 8 * n
    bo = (j + 3) * 8 * n
    print(f"j={j:2d}: multidot {tm:.3f} ms {bm / tm / 1e6:.0f} GB/s   orth {to:.3f} ms {bo / to / 1e6:.0f} GB/s",
          flush=True)
