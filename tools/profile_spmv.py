"""One format's SpMV a few times, for ncu: python tools/profile_spmv.py FMT [points] [n] [csr strategy]
FMT in csr, sellp, ell, coo(R-MAT scale n), hybrid(R-MAT), convert (CSR -> ELL and
CSR -> SELL-P(64) of the stencil, 5 times each)."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2006_14290_b200 import corpus, kernels
from paper_2006_14290_b200 import device as D

fmt = sys.argv[1]
pts = int(sys.argv[2]) if len(sys.argv) > 2 else 27
n = int(sys.argv[3]) if len(sys.argv) > 3 else 200
if fmt in ("coo", "hybrid", "csr_rmat"):
    R = corpus.rmat(n)
    A = R if fmt == "coo" else D.coo_to_csr(R)
    if fmt == "hybrid":
        A = D.csr_to_hybrid(A)
else:
    A = corpus.stencil3d(n, pts) if pts != 5 else corpus.poisson2d_matrix(n)
    if fmt == "sellp":
        A = D.csr_to_sellp(A, 64)
    elif fmt == "ell":
        A = D.csr_to_ell(A)
if fmt == "convert":
    for _ in range(5):
        E = D.csr_to_ell(A, width=27 if pts == 27 else None)
        del E
        S = D.csr_to_sellp(A, 64)
        del S
    torch.cuda.synchronize()
    print("ok convert", A.nrows)
    sys.exit(0)
strategy = sys.argv[4] if len(sys.argv) > 4 else None
if strategy and getattr(A, "fmt", None) == "csr":
    A.with_strategy(strategy)
x = torch.rand(A.ncols, dtype=torch.float64, device='cuda')
y = torch.empty(A.nrows, dtype=torch.float64, device='cuda')
for _ in range(5):
    kernels.spmv_device(A, x, y)
torch.cuda.synchronize()
print("ok", fmt, A.nrows)
