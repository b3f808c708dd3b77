"""CUDA-event timing of every CSR strategy on the 27-point 200^3 operator
(development probe)."""
import sys

import torch

sys.path.insert(0, '.')
from paper_2006_14290_b200 import corpus  # noqa: E402
from paper_2006_14290_b200 import kernels as K  # noqa: E402

A = corpus.stencil3d(200, 27)
x = torch.rand(A.ncols, dtype=torch.float64, device="cuda")
y = torch.empty(A.nrows, dtype=torch.float64, device="cuda")
for strat in sys.argv[1:] or ["subwarp", "rowblock"]:
    A.with_strategy(strat, 0)
    for _ in range(3):
        K.spmv_device(A, x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        K.spmv_device(A, x, y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"csr {strat}: {ms:.4f} ms  {A.algorithmic_bytes() / ms / 1e6:.0f} GB/s", flush=True)
