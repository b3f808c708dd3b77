"""Distributed-CG iteration rate on the 7-point n^3 Laplacian, eager vs CUDA
graph (run under torchrun; at world size 1 it still goes through NCCL)."""
import os
import sys

sys.path.insert(0, '.')
import torch
import torch.distributed as dist

from paper_2006_14290_b200 import corpus
from paper_2006_14290_b200 import distributed as DI

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 500
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
op = DI.stencil_slab_operator(n, n, None, corpus.points_7pt(), dist, fmt="sellp", weak=False, nz=n)
b = op.ops.zeros(op.n_local) + 1.0
for graph in (False, True):
    DI.cg_solve(op, b, 1e-30, 100, graph=graph)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    _, hist = DI.cg_solve(op, b, 1e-30, iters, graph=graph)
    t1.record()
    torch.cuda.synchronize()
    ms = op.comm.max_scalar(t0.elapsed_time(t1))
    if dist.get_rank() == 0:
        print(f"graph={graph} world={dist.get_world_size()} n={n} iterations={len(hist) - 1} "
              f"ms={ms:.1f} it/s={(len(hist) - 1) / ms * 1e3:.1f}", flush=True)
dist.destroy_process_group()
