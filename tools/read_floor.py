"""Read-only streaming floor on this B200: torch sum over 2.7 GB (the headline
SpMV's byte count) and over 1.7 GB (the 7-point CG SpMV), CUDA events."""
import torch

for gb in (2.704, 1.677):
    n = int(gb * 1e9 / 8)
    z = torch.rand(n, dtype=torch.float64, device='cuda')
    for _ in range(3):
        z.sum()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        z.sum()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"sum {gb} GB: {ms:.4f} ms -> {gb / ms * 1e3:.1f} GB/s", flush=True)
    del z
