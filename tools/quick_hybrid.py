"""CUDA-event timing of CSR -> Hybrid(k) on R-MAT scale 24 (development probe;
bench.py is the contract) + a bitwise check of the COO remainder against a
torch restatement."""
import sys

import torch

sys.path.insert(0, '.')
from paper_2006_14290_b200 import corpus  # noqa: E402
from paper_2006_14290_b200 import device as D  # noqa: E402


def t(fn, n=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / n, 4)


scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
Rc = D.coo_to_csr(corpus.rmat(scale))
for k in (8, 4, 16):
    ms = t(lambda: D.csr_to_hybrid(Rc, width=k))
    H = D.csr_to_hybrid(Rc, width=k)
    # restatement: entries at position >= k of their row, row-major
    ptr = Rc.row_ptrs.long()
    lens = ptr[1:] - ptr[:-1]
    rows = torch.repeat_interleave(torch.arange(Rc.nrows, device='cuda'), lens)
    pos = torch.arange(Rc.nnz, device='cuda') - ptr[:-1][rows]
    keep = pos >= k
    ok = (torch.equal(H.coo.row_idx.long(), rows[keep]) and torch.equal(H.coo.col_idx, Rc.col_idx[keep])
          and torch.equal(H.coo.values, Rc.values[keep]))
    b = 12 * Rc.nnz + 4 * (Rc.nrows + 1) + 12 * k * Rc.nrows + 4 * Rc.nrows + 16 * H.coo.nnz + 8 * (Rc.nrows + 1)
    print(f"csr_to_hybrid k={k}: {ms} ms  {b / ms / 1e6:.1f} GB/s  coo_nnz {H.coo.nnz}  remainder equal: {ok}",
          flush=True)
    del H, rows, pos, keep
    torch.cuda.empty_cache()
