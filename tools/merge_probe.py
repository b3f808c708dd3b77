"""A CSR strategy (argv[1], default merge) on R-MAT 24 and the 27-point 200^3
operator, event-timed, checked against load_balance (development probe for
A/B builds)."""
import sys

import torch

sys.path.insert(0, '.')
from paper_2006_14290_b200 import corpus, kernels  # noqa: E402
from paper_2006_14290_b200 import device as D  # noqa: E402


def t(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


strat = sys.argv[1] if len(sys.argv) > 1 else "merge"
for name, A in (("rmat 24", D.coo_to_csr(corpus.rmat(24))), ("27pt 200^3", corpus.stencil3d(200, 27))):
    x = torch.rand(A.ncols, dtype=torch.float64, device="cuda")
    ref = kernels.spmv_device(A.with_strategy("load_balance"), x).clone()
    y = torch.empty_like(ref)
    A.with_strategy(strat)
    ms = t(lambda: kernels.spmv_device(A, x, y))
    lens = (A.row_ptrs[1:] - A.row_ptrs[:-1]).to(torch.float64).clamp(min=1)
    err = ((y - ref).abs() / (lens * ref.abs().clamp(min=1))).max().item()
    print(f"{name}: {strat} {ms:.3f} ms  err vs load_balance {err:.2e}", flush=True)
    del A, x, y, ref
    torch.cuda.empty_cache()
