"""CSR -> ELL / SELL-P conversions of the 27-point 200^3 matrix, event-timed
(development probe for A/B builds; bench.py is the contract)."""
import sys

import torch

sys.path.insert(0, '.')
from paper_2006_14290_b200 import corpus  # noqa: E402
from paper_2006_14290_b200 import device as D  # noqa: E402


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


A = corpus.stencil3d(200, 27)
ref_s = D.csr_to_sellp(A, 64)
ref_e = D.csr_to_ell(A)
print(f"csr_to_sellp {t(lambda: D.csr_to_sellp(A, 64)):.3f} ms  csr_to_ell {t(lambda: D.csr_to_ell(A)):.3f} ms",
      flush=True)
s2, e2 = D.csr_to_sellp(A, 64), D.csr_to_ell(A)
print("bitwise:", torch.equal(s2.values, ref_s.values) and torch.equal(s2.col_idx, ref_s.col_idx)
      and torch.equal(e2.values, ref_e.values) and torch.equal(e2.col_idx, ref_e.col_idx), flush=True)
