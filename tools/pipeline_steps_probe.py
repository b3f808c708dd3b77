"""SpmvPipeline per-step time vs the number of steps (fill/drain amortisation)."""
import sys, torch
sys.path.insert(0, '.')
import paper_2006_14290_b200 as wk
from paper_2006_14290_b200 import corpus
from paper_2006_14290_b200 import device as D
A = D.csr_to_sellp(corpus.stencil3d(200, 27), 64)
xh = torch.rand(A.ncols, dtype=torch.float64).pin_memory()
yhs = [torch.empty(A.nrows, dtype=torch.float64, pin_memory=True) for _ in range(2)]
pipe = wk.SpmvPipeline(A)
for k in range(3): pipe.submit(xh, yhs[k % 2])
pipe.synchronize(); torch.cuda.synchronize()
for steps in (5, 20, 80):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(pipe.s_h2d)
    for k in range(steps): pipe.submit(xh, yhs[k % 2])
    e1.record(pipe.s_d2h); torch.cuda.synchronize()
    print(steps, round(e0.elapsed_time(e1) / steps, 4), flush=True)
