"""CUDA-event timing of the SELL-P(64) SpMV and of CG's fused SpMV + p.q on
the 7-point 256^3 operator, narrow and wide configurations (development
probe; the wide configuration is forced by overstating the stored-slot count
in the operand, the dispatch key)."""
import ctypes
import sys

import torch

sys.path.insert(0, '.')
from paper_2006_14290_b200 import _lib, corpus  # noqa: E402
from paper_2006_14290_b200 import device as D  # noqa: E402

A = D.csr_to_sellp(corpus.stencil3d(256, 7), 64)
n = A.nrows
L = _lib.load()
st = D.stream_handle()
p = torch.rand(n, dtype=torch.float64, device="cuda")
q = torch.empty_like(p)
state = torch.zeros(256, dtype=torch.uint8, device="cuda")
ws = torch.zeros(int(L.wk_reduce_workspace_bytes()), dtype=torch.uint8, device="cuda")
P = D._ptr
narrow = A.wk()
wide = _lib.WkMatrix.from_buffer_copy(narrow)
wide.nnz = A.stored * 100


def t(fn, reps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for rep in range(2):
    for name, m in (("narrow", narrow), ("wide", wide)):
        a = t(lambda: _lib.call("wk_spmv", ctypes.byref(m), P(p), P(q), st))
        b = t(lambda: _lib.call("wk_cg_spmv_dot", ctypes.byref(m), P(p), P(q), P(state), P(ws), st))
        print(f"{name}: spmv {a:.1f} us  spmv+dot {b:.1f} us", flush=True)
