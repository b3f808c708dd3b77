"""CG on the 7-point 256^3 Laplacian (BASELINE config 4) for ncu launch lists."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2006_14290_b200 as wk
from paper_2006_14290_b200 import corpus
from paper_2006_14290_b200 import device as D

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
A = D.csr_to_sellp(corpus.stencil3d(n, 7), 64)
b = torch.ones(A.nrows, dtype=torch.float64, device='cuda')
ex = wk.make_executor('b200')
x, hist = wk.cg_solve(A, b, 1e-30, iters, ex)
torch.cuda.synchronize()
print("iterations", len(hist) - 1)
