"""A/B sweep of the SELL-P(64) kernel configurations (wk_config_set
"sellp_kernel"): python tools/sweep_sellp.py [points=27] [n=200]."""
import json
import statistics
import sys

sys.path.insert(0, '.')
import torch

from paper_2006_14290_b200 import _lib, corpus, kernels
from paper_2006_14290_b200 import device as D
import bench

pts = int(sys.argv[1]) if len(sys.argv) > 1 else 27
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
A = D.csr_to_sellp(corpus.stencil3d(n, pts), 64)
x = torch.rand(A.ncols, dtype=torch.float64, device='cuda')
y = torch.empty(A.nrows, dtype=torch.float64, device='cuda')
ref = None
for choice in range(11):
    _lib.call('wk_config_set', b'sellp_kernel', choice)
    tot, per = bench.timed(lambda: kernels.spmv_device(A, x, y), 20, 5)
    ms = statistics.mean(per)
    if ref is None:
        ref = y.clone()
    print(json.dumps({"matrix": f"{pts}pt_{n}", "choice": choice, "ms": round(ms, 4),
                      "GB/s": round(A.algorithmic_bytes() / ms / 1e6, 1), "bitwise_same": bool(torch.equal(ref, y))}))
