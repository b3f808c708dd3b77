"""Config 1 (CSR 5-point Poisson 1000^2) with the bench's L2 flush before
every launch: per-strategy CUDA-event times (development A/B)."""
import statistics
import sys

import torch

sys.path.insert(0, '.')
import bench  # noqa: E402
from paper_2006_14290_b200 import corpus, kernels  # noqa: E402

A = corpus.poisson2d_matrix(1000)
x = torch.rand(A.ncols, dtype=torch.float64, device='cuda')
y = torch.empty(A.nrows, dtype=torch.float64, device='cuda')
buf = torch.ones(512 * 1024 * 1024 // 8, dtype=torch.float64, device='cuda')
flush = lambda: buf.sum()  # noqa: E731
for s in ("rowblock", "subwarp", "stream", "rowblock"):
    A.with_strategy(s)
    _, per = bench.timed(lambda: kernels.spmv_device(A, x, y), 30, 5, None, flush)
    ms = statistics.mean(per)
    print(s, round(ms * 1e3, 2), "us", round(A.algorithmic_bytes() / ms / 1e6, 1), "GB/s", flush=True)

# floor: a plain 80 MB streaming read (torch sum) and a 80 MB copy, same flush
z = torch.rand(10_000_000, dtype=torch.float64, device='cuda')
z2 = torch.empty_like(z)
for name, fn in (("torch sum 80MB", lambda: z.sum()), ("torch copy 80MB->80MB", lambda: z2.copy_(z))):
    _, per = bench.timed(fn, 30, 5, None, flush)
    print(name, round(statistics.mean(per) * 1e3, 2), "us", flush=True)
