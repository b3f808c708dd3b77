import sys, json, statistics
sys.path.insert(0, '.')
import torch
import paper_2006_14290_b200 as wk
from paper_2006_14290_b200 import corpus, _lib, kernels
from paper_2006_14290_b200 import device as D
import bench
A = D.csr_to_sellp(corpus.stencil3d(200, 27), 64)
x = torch.rand(A.ncols, dtype=torch.float64, device='cuda')
y = torch.empty(A.nrows, dtype=torch.float64, device='cuda')
ref = None
for choice in range(9):
    _lib.call('wk_config_set', b'sellp_kernel', choice)
    tot, per = bench.timed(lambda: kernels.spmv_device(A, x, y), 20, 5)
    ms = statistics.mean(per)
    if ref is None: ref = y.clone()
    same = bool(torch.equal(ref, y))
    print(json.dumps({"choice": choice, "ms": round(ms,4), "GB/s": round(A.algorithmic_bytes()/ms/1e6,1), "bitwise_same": same}))
