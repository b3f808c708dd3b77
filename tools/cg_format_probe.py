"""CG (1000 iterations, 7-point 256^3, b = ones, tol 1e-30) on SELL-P(64) and
on ELL: the same iteration through wk_cg_solve, different SpMV kernels."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2006_14290_b200 as wk  # noqa: E402
from paper_2006_14290_b200 import corpus  # noqa: E402
from paper_2006_14290_b200 import device as D  # noqa: E402

A = corpus.stencil3d(256, 7)
ex = wk.make_executor("b200")
b = torch.ones(A.nrows, dtype=torch.float64, device="cuda")
hs = {}
for name, M in (("sellp", D.csr_to_sellp(A, 64)), ("ell", D.csr_to_ell(A))):
    wk.cg_solve(M, b, 1e-30, 60, ex)
    torch.cuda.synchronize()
    for _ in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        x, h = wk.cg_solve(M, b, 1e-30, 1000, ex)
        e1.record()
        torch.cuda.synchronize()
        print(f"cg {name}: {e0.elapsed_time(e1):.1f} ms -> {1000 / e0.elapsed_time(e1) * 1e3:.1f} it/s", flush=True)
    hs[name] = h
    x12, h12 = wk.cg_solve(M, b, 1e-12, 1000, ex)
    print(name, "iterations to 1e-12:", len(h12) - 1, flush=True)
    del M
