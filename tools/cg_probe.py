"""Where does a CG iteration go? (7-point 256^3, SELL-P(64)).
1. wk.cg_solve, 1000 iterations (the bench number);
2. each building-block kernel of one iteration timed alone (100 reps, events);
3. the three kernels back to back eagerly (no graph)."""
import ctypes
import sys

import torch

sys.path.insert(0, '.')
import paper_2006_14290_b200 as wk  # noqa: E402
from paper_2006_14290_b200 import _lib, corpus  # noqa: E402
from paper_2006_14290_b200 import device as D  # noqa: E402

A = D.csr_to_sellp(corpus.stencil3d(256, 7), 64)
n = A.nrows
ex = wk.make_executor("b200")
b = torch.ones(n, dtype=torch.float64, device="cuda")


def ev_time(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for _ in range(2):
    x, hist = wk.cg_solve(A, b, 1e-30, 50, ex)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x, hist = wk.cg_solve(A, b, 1e-30, 1000, ex)
    e1.record()
    torch.cuda.synchronize()
    print(f"cg_solve 1000 it: {e0.elapsed_time(e1):.1f} ms -> it/s {1000 / e0.elapsed_time(e1) * 1e3:.1f}", flush=True)

L = _lib.load()
st = D.stream_handle()
state = torch.zeros(ctypes.sizeof(_lib.WkCgState), dtype=torch.uint8, device="cuda")
ws = torch.zeros(int(L.wk_reduce_workspace_bytes()), dtype=torch.uint8, device="cuda")
p = torch.rand(n, dtype=torch.float64, device="cuda")
q = torch.empty_like(p)
xx = torch.zeros_like(p)
r = torch.rand(n, dtype=torch.float64, device="cuda")
P = D._ptr
# a state that never finishes and never replaces: iteration 1 (not a multiple of 50)
h = _lib.WkCgState()
h.rho, h.pq, h.rr, h.threshold, h.alpha, h.beta = 1.0, 1.0, 1.0, 0.0, 1e-9, 0.5
h.iteration, h.max_iters, h.done, h.breakdown = 1, 1 << 40, 0, 0
state.copy_(torch.frombuffer(bytearray(bytes(h)), dtype=torch.uint8).to("cuda"))
t_spmv = ev_time(lambda: _lib.call("wk_cg_spmv_dot", A.wk_ptr(), P(p), P(q), P(state), P(ws), st), 100)
t_spmv_plain = ev_time(lambda: _lib.call("wk_spmv", A.wk_ptr(), P(p), P(q), st), 100)
t_xr = ev_time(lambda: _lib.call("wk_cg_update_xr", n, P(p), P(q), P(xx), P(r), P(state), P(ws), st), 100)
t_p = ev_time(lambda: _lib.call("wk_cg_update_p", n, P(r), P(p), P(state), st), 100)


def it():
    _lib.call("wk_cg_spmv_dot", A.wk_ptr(), P(p), P(q), P(state), P(ws), st)
    _lib.call("wk_cg_update_xr", n, P(p), P(q), P(xx), P(r), P(state), P(ws), st)
    _lib.call("wk_cg_update_p", n, P(r), P(p), P(state), st)


t_it = ev_time(it, 50)
print(f"spmv+dot {t_spmv * 1e3:.1f} us (plain spmv {t_spmv_plain * 1e3:.1f}), update_xr {t_xr * 1e3:.1f} us, "
      f"update_p {t_p * 1e3:.1f} us, sum {1e3 * (t_spmv + t_xr + t_p):.1f} us; back-to-back iteration {t_it * 1e3:.1f} us")
