"""CUDA-event timing of the ELL kernels (ell_kernel 0..4) on the 27-point
200^3 stencil (development A/B; bench.py is the contract)."""
import sys

import torch

sys.path.insert(0, '.')
from paper_2006_14290_b200 import _lib, corpus, kernels  # noqa: E402
from paper_2006_14290_b200 import device as D  # noqa: E402


def t(d, x, n=20):
    y = torch.empty(d.nrows, dtype=torch.float64, device='cuda')
    for _ in range(3):
        kernels.spmv_device(d, x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        kernels.spmv_device(d, x, y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    return round(ms, 4), round(d.algorithmic_bytes() / ms / 1e6, 1), y


pts = int(sys.argv[1]) if len(sys.argv) > 1 else 27
grid = int(sys.argv[2]) if len(sys.argv) > 2 else 200
A = corpus.stencil3d(grid, pts)
x = torch.rand(A.ncols, dtype=torch.float64, device='cuda')
E = D.csr_to_ell(A)
S = D.csr_to_sellp(A, 64)
del A
print("sellp", t(S, x)[:2], flush=True)
del S
ref = None
for k in (0, 2, 3, 4):
    _lib.call("wk_config_set", b"ell_kernel", k)
    ms, gbs, y = t(E, x)
    if ref is None:
        ref = y.clone()
    print("ell kernel", k, ms, gbs, "bitwise==k0:", torch.equal(y, ref), flush=True)
