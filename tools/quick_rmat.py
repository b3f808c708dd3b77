"""CUDA-event timing of the R-MAT (BASELINE config 3) SpMV kernels with and
without the hot-column gather plan (development probe; bench.py is the
contract)."""
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_2006_14290_b200 import corpus  # noqa: E402
from paper_2006_14290_b200 import device as D  # noqa: E402
from paper_2006_14290_b200 import kernels as K  # noqa: E402


def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
R = corpus.rmat(scale)
x = torch.rand(R.ncols, dtype=torch.float64, device="cuda")
Rc = D.coo_to_csr(R).with_strategy("load_balance")
H = D.csr_to_hybrid(Rc, width=8)
for name, m in (("coo", R), ("csr_load_balance", Rc), ("hybrid_k8", H.coo)):
    for mc in (0,):
        g = m if name != "hybrid_k8" else H.coo
        g.set_gather_plan("on", mc)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plan = g.gather_plan()
        torch.cuda.synchronize()
        build_ms = (time.perf_counter() - t0) * 1e3
        op = H if name == "hybrid_k8" else m
        op._wk = None
        y_on = K.spmv_device(op, x)
        ms_on = t(lambda: K.spmv_device(op, x))
        g.set_gather_plan("off")
        op._wk = None
        y_off = K.spmv_device(op, x)
        ms_off = t(lambda: K.spmv_device(op, x))
        b = op.algorithmic_bytes()
        d = float(((y_on - y_off).abs() / y_off.abs().clamp(min=1)).max())
        print(f"{name}: off {ms_off:.4f} ms ({b / ms_off / 1e6:.0f} GB/s)  on {ms_on:.4f} ms ({b / ms_on / 1e6:.0f} GB/s)"
              f"  nhot {plan.nhot} thr {plan.threshold} covered {plan.covered / m.nnz:.3f}  build {build_ms:.1f} ms"
              f"  bitwise {torch.equal(y_on, y_off)} maxrel {d:.2e}", flush=True)
