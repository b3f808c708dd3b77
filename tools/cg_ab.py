"""CG 7-point 256^3 (SELL-P 64) it/s for A/B library builds: 1000 iterations,
median of 3 (development probe; bench.py is the contract).
    WK_LIB_PATH=... python tools/cg_ab.py"""
import sys

import torch

sys.path.insert(0, '.')
import paper_2006_14290_b200 as wk  # noqa: E402
from paper_2006_14290_b200 import corpus  # noqa: E402
from paper_2006_14290_b200 import device as D  # noqa: E402

A = D.csr_to_sellp(corpus.stencil3d(256, 7), 64)
b = torch.ones(A.nrows, dtype=torch.float64, device="cuda")
ex = wk.make_executor("b200")
wk.cg_solve(A, b, 1e-30, 100, ex)
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    x, hist = wk.cg_solve(A, b, 1e-30, 1000, ex)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"cg 1000 it: median {ts[1]:.1f} ms ({1e6 / ts[1]:.1f} it/s), all {[round(t, 1) for t in ts]}, "
      f"last res {hist[-1].item():.6e}", flush=True)
