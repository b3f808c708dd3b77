"""CUDA-event timing of CSR -> SELL-P(64) / ELL on the 27-point 200^3 stencil,
per fill kernel (development A/B; bench.py is the contract)."""
import sys

import torch

sys.path.insert(0, '.')
from paper_2006_14290_b200 import _lib, corpus  # noqa: E402
from paper_2006_14290_b200 import device as D  # noqa: E402

A = corpus.stencil3d(200, 27)


def t(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / n, 4)


ref = None
for k in (0, 1, 0, 1):
    _lib.call("wk_config_set", b"fill_kernel", k)
    ms = t(lambda: D.csr_to_sellp(A, 64))
    S = D.csr_to_sellp(A, 64)
    if ref is None:
        ref = (S.col_idx.clone(), S.values.clone())
    same = torch.equal(S.col_idx, ref[0]) and torch.equal(S.values, ref[1])
    print("csr_to_sellp fill_kernel", k, ms, "ms", round(5206259564 / ms / 1e6, 1), "GB/s", "same:", same, flush=True)
    del S
# the fill kernel alone (outputs preallocated)
S = D.csr_to_sellp(A, 64)
st = D.stream_handle(A.device)
P = lambda t: t.data_ptr()  # noqa: E731
for k in (0, 1, 0, 1):
    _lib.call("wk_config_set", b"fill_kernel", k)
    ms = t(lambda: _lib.call("wk_csr_to_sellp_fill", A.nrows, 64, P(A.row_ptrs), P(A.col_idx), P(A.values),
                             P(S.slice_sets), P(S.col_idx), P(S.values), st))
    print("sellp fill only, kernel", k, ms, "ms", round(5206259564 / ms / 1e6, 1), "GB/s", flush=True)
ws = D.workspace(A.device)
lens = torch.empty(A.nrows, dtype=torch.int32, device='cuda')
sets = torch.empty_like(S.slice_sets)
ms = t(lambda: _lib.call("wk_csr_to_sellp_sets", A.nrows, 64, P(A.row_ptrs), P(sets), P(lens),
                         P(ws.scan_ws(sets.numel() - 1)), st))
print("sellp sets only", ms, "ms; equal:", torch.equal(sets, S.slice_sets), flush=True)
E = D.csr_to_ell(A, width=27)
for k in (0, 1, 0, 1):
    _lib.call("wk_config_set", b"fill_kernel", k)
    ms = t(lambda: _lib.call("wk_csr_to_ell_fill", A.nrows, 27, A.nrows, P(A.row_ptrs), P(A.col_idx), P(A.values),
                             P(E.col_idx), P(E.values), P(E.row_lengths_t), st))
    print("ell fill only, kernel", k, ms, "ms", round(5222166308 / ms / 1e6, 1), "GB/s", flush=True)
print("csr_to_ell", t(lambda: D.csr_to_ell(A, width=27)), "ms")
