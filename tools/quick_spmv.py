"""Quick CUDA-event timing of the SpMV strategies on R-MAT scale 24 and the
27-point 200^3 stencil (development A/B; bench.py is the contract)."""
import sys

import torch

sys.path.insert(0, '.')
from paper_2006_14290_b200 import _lib, corpus, kernels  # noqa: E402
from paper_2006_14290_b200 import device as D  # noqa: E402


def t(d, x, n=10):
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
    return round(ms, 4), round(d.algorithmic_bytes() / ms / 1e6, 1)


R = corpus.rmat(24)
Rc = D.coo_to_csr(R)
x = torch.rand(Rc.ncols, dtype=torch.float64, device='cuda')
for s in ("load_balance", "merge", "stream"):
    Rc.with_strategy(s)
    print("rmat csr", s, t(Rc, x))
for c in (0, 1, 2, 3):
    _lib.call("wk_config_set", b"coo_kernel", c)
    print("rmat coo kernel", c, t(R, x))
del R, Rc
A = corpus.stencil3d(200, 27)
x = torch.rand(A.ncols, dtype=torch.float64, device='cuda')
for s in ("load_balance", "merge", "rowblock", "stream"):
    A.with_strategy(s)
    print("27pt csr", s, t(A, x))
