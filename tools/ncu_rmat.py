"""One launch each of the R-MAT COO / CSR load_balance SpMV with and without
the gather plan (for ncu --set full; not a timing tool). Order: COO plan off,
COO plan on, CSR plan off, CSR plan on."""
import sys

import torch

sys.path.insert(0, '.')
from paper_2006_14290_b200 import corpus  # noqa: E402
from paper_2006_14290_b200 import device as D  # noqa: E402
from paper_2006_14290_b200 import kernels as K  # noqa: E402

R = corpus.rmat(24)
x = torch.rand(R.ncols, dtype=torch.float64, device="cuda")
Rc = D.coo_to_csr(R).with_strategy("load_balance")
for m in (R, Rc):
    for pol in ("off", "on"):
        m.set_gather_plan(pol)
        m.gather_plan()
        torch.cuda.synchronize()
        K.spmv_device(m, x)
        torch.cuda.synchronize()
