"""CSR subwarp-per-row SpMV (the reference's CSR algorithm) on configs 1-3,
event-timed, with the max scaled error against the bitwise rowblock result
(development probe for A/B library builds; bench.py is the contract)."""
import sys

import torch

sys.path.insert(0, '.')
from paper_2006_14290_b200 import corpus, kernels  # noqa: E402
from paper_2006_14290_b200 import device as D  # noqa: E402


def t(fn, reps=20):
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


for name, A in (("27pt 200^3", corpus.stencil3d(200, 27)), ("poisson 1000^2", corpus.poisson2d_matrix(1000)),
                ("rmat 24", D.coo_to_csr(corpus.rmat(24)))):
    x = torch.rand(A.ncols, dtype=torch.float64, device="cuda")
    ref = kernels.spmv_device(A.with_strategy("rowblock"), x)
    y = torch.empty_like(ref)
    lens = (A.row_ptrs[1:] - A.row_ptrs[:-1]).to(torch.float64).clamp(min=1)
    for T in ([0, 4, 8, 16, 32] if "rmat" not in name else [0, 32]):
        A.with_strategy("subwarp", T)
        ms = t(lambda: kernels.spmv_device(A, x, y))
        err = ((y - ref).abs() / (lens * ref.abs().clamp(min=1))).max().item()
        gbs = A.algorithmic_bytes() / ms / 1e6
        print(f"{name}: subwarp T={T or 'auto'} {ms * 1e3:.1f} us  {gbs:.0f} GB/s  err {err:.2e}", flush=True)
    del A, x, ref, y
    torch.cuda.empty_cache()
