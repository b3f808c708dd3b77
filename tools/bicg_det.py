"""BiCGSTAB 128^3 convection-diffusion iteration counts: the GPU solve (run
three times: deterministic) against the C oracle at several thread counts (the
spread of a chaotic solver's count under rounding changes)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import paper_2006_14290_b200 as wk  # noqa: E402
from paper_2006_14290_b200 import device as D  # noqa: E402
from oracle import native  # noqa: E402
from test_gpu_solver_parity import _convdiff, _HostOp  # noqa: E402

C = _convdiff(128)
A = D.csr_to_sellp(C, 64)
b = torch.ones(A.nrows, dtype=torch.float64, device="cuda")
for i in range(3):
    x, h = wk.bicgstab_solve(A, b, 1e-8, 5000, wk.make_executor("b200"))
    h = h.cpu().numpy()
    print("gpu", len(h) - 1, h[5].hex(), float(x.sum()), flush=True)
P = native.Prepared(_HostOp(C))
for t in list(range(1, 17)) + [24, 32]:
    rx, rh = P.bicgstab(np.ones(A.nrows), 1e-8, 5000, nthreads=t)
    print("cpu threads", t, len(rh) - 1, flush=True)
print("nproc", os.cpu_count())
