"""CUDA-event timing of the SELL-P(64) SpMV on the 7-point 256^3 and
27-point 200^3 operators, and of 1000 CG iterations on the 7-point one
(development probe; bench.py is the contract)."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2006_14290_b200 as wk  # noqa: E402
from paper_2006_14290_b200 import corpus  # noqa: E402
from paper_2006_14290_b200 import device as D  # noqa: E402
from paper_2006_14290_b200 import kernels as K  # noqa: E402


def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for pts, n in ((7, 256), (27, 200)):
    A = D.csr_to_sellp(corpus.stencil3d(n, pts), 64)
    x = torch.rand(A.ncols, dtype=torch.float64, device="cuda")
    y = torch.empty(A.nrows, dtype=torch.float64, device="cuda")
    ms = t(lambda: K.spmv_device(A, x, y))
    print(f"sellp {pts}-pt {n}^3: {ms:.4f} ms  {A.algorithmic_bytes() / ms / 1e6:.0f} GB/s", flush=True)
    if pts == 7:
        ex = wk.make_executor("b200")
        b = torch.ones(A.nrows, dtype=torch.float64, device="cuda")
        wk.cg_solve(A, b, 1e-30, 50, ex)
        for _ in range(2):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            xs, hist = wk.cg_solve(A, b, 1e-30, 1000, ex)
            e1.record()
            torch.cuda.synchronize()
            print(f"cg 1000 it: {e0.elapsed_time(e1):.1f} ms  {1000 / e0.elapsed_time(e1) * 1e3:.1f} it/s", flush=True)
    del A, x, y
    torch.cuda.empty_cache()
