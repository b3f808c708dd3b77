"""SpmvPipeline A/B: chunk / piece counts, host submit cost (27-pt 200^3)."""
import sys
import time

import torch

sys.path.insert(0, '.')
import paper_2006_14290_b200 as wk  # noqa: E402
from paper_2006_14290_b200 import corpus  # noqa: E402
from paper_2006_14290_b200 import device as D  # noqa: E402

A = D.csr_to_sellp(corpus.stencil3d(200, 27), 64)
xh = torch.rand(A.ncols, dtype=torch.float64).pin_memory()
yhs = [torch.empty(A.nrows, dtype=torch.float64, pin_memory=True) for _ in range(2)]
for chunks, pieces in ((1, 1), (4, 4), (8, 16), (16, 32), (32, 64)):
    pipe = wk.SpmvPipeline(A, chunks=chunks, pieces=pieces)
    for k in range(3):
        pipe.submit(xh, yhs[k % 2])
    pipe.synchronize()
    torch.cuda.synchronize()
    steps = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(pipe.s_h2d)
    t0 = time.perf_counter()
    for k in range(steps):
        pipe.submit(xh, yhs[k % 2])
    host = (time.perf_counter() - t0) / steps * 1e3
    e1.record(pipe.s_d2h)
    torch.cuda.synchronize()
    print(f"chunks {chunks:2d} pieces {pieces:2d}: {e0.elapsed_time(e1) / steps:.3f} ms/step, host submit {host:.3f} ms",
          flush=True)
