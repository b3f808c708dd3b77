"""A few BiCGSTAB / GMRES iterations on the 7-point convection-diffusion 256^3
(SELL-P(64)), for an ncu launch list: per-kernel duration and DRAM bytes."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2006_14290_b200 as wk  # noqa: E402
from paper_2006_14290_b200 import corpus  # noqa: E402
from paper_2006_14290_b200 import device as D  # noqa: E402

grid = int(sys.argv[2]) if len(sys.argv) > 2 else 256
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
A = D.csr_to_sellp(corpus.convection_diffusion3d(grid), 64)
b = torch.ones(A.nrows, dtype=torch.float64, device="cuda")
ex = wk.make_executor("b200")
which = sys.argv[1] if len(sys.argv) > 1 else "bicgstab"
if which == "bicgstab":
    wk.bicgstab_solve(A, b, 1e-30, iters, ex)
else:
    wk.gmres_solve(A, b, 1e-30, iters, ex, restart=30)
torch.cuda.synchronize()
print("ok")
