"""R-MAT 24 ingestion pieces, event-timed (development probe): the duplicate
fold after the sort (wk_coo_dedup_count + wk_coo_dedup_scatter through
coo_from_keys on pre-sorted keys) and COO -> CSR row pointers."""
import sys

import torch

sys.path.insert(0, '.')
from paper_2006_14290_b200 import _lib, corpus  # noqa: E402
from paper_2006_14290_b200 import device as D  # noqa: E402


def t(fn, setup=None, n=5):
    if setup:
        setup()
    fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(n):
        if setup:
            setup()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / n


k0, v0 = corpus.rmat_edge_keys(24)
sk, sv = D.sort_pairs(k0, v0, 48, inplace=True)
n = 1 << 24
m = sk.numel()
L = _lib.load()
st = D.stream_handle(sk.device)
nt = int(L.wk_coo_dedup_tiles(m))
work = torch.empty(nt + 1, dtype=torch.int64, device="cuda")
_lib.call("wk_coo_dedup_count", m, D._ptr(sk), D._ptr(work), st)
nu = int(work[nt].item())
row = torch.empty(nu, dtype=torch.int32, device="cuda")
col = torch.empty(nu, dtype=torch.int32, device="cuda")
val = torch.empty(nu, dtype=torch.float64, device="cuda")
print("unique", nu, flush=True)
print("dedup count:", round(t(lambda: _lib.call("wk_coo_dedup_count", m, D._ptr(sk), D._ptr(work), st)), 3), "ms")
print("dedup scatter:", round(t(lambda: _lib.call("wk_coo_dedup_scatter", m, n, D._ptr(sk), D._ptr(sv), D._ptr(work),
                                                  D._ptr(row), D._ptr(col), D._ptr(val), st)), 3), "ms", flush=True)
R = D.DeviceCoo(n, n, row, col, val)
print("coo_to_csr:", round(t(lambda: D.coo_to_csr(R)), 3), "ms", flush=True)
print("checksum", float(val.sum()), int(row.to(torch.int64).sum()), int(col.to(torch.int64).sum()), flush=True)
