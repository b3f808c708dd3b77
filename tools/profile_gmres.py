"""A few GMRES(30) cycles on the 7-point convection-diffusion 256^3 (for ncu
captures of the Gram-Schmidt kernels)."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2006_14290_b200 as wk  # noqa: E402
from paper_2006_14290_b200 import corpus  # noqa: E402
from paper_2006_14290_b200 import device as D  # noqa: E402

A = D.csr_to_sellp(corpus.convection_diffusion3d(256), 64)
b = torch.ones(A.nrows, dtype=torch.float64, device='cuda')
x, hist = wk.gmres_solve(A, b, 1e-30, 40, wk.make_executor('b200'), restart=30)
torch.cuda.synchronize()
print("iterations", len(hist) - 1)
