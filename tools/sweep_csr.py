"""A/B of the CSR stream kernels (wk_config_set "csr_kernel": 0 = CTA per
chunk, 1 = persistent TMA pipeline) and the subwarp kernel."""
import json
import statistics
import sys

sys.path.insert(0, '.')
import torch

from paper_2006_14290_b200 import _lib, corpus, kernels
from paper_2006_14290_b200 import device as D
import bench

flush_buf = torch.ones(512 * 1024 * 1024 // 8, dtype=torch.float64, device='cuda')


def flush():
    # read (not write) 512 MB: evicts L2 without leaving dirty lines behind
    flush_buf.sum()


cases = [("poisson2d_1000", corpus.poisson2d_matrix(1000), True), ("27pt_200", corpus.stencil3d(200, 27), False),
         ("7pt_256", corpus.stencil3d(256, 7), False)]
if len(sys.argv) > 1 and sys.argv[1] == "rmat":
    cases.append(("rmat20", D.coo_to_csr(corpus.rmat(20)), False))
for name, A, fl in cases:
    x = torch.rand(A.ncols, dtype=torch.float64, device='cuda')
    y = torch.empty(A.nrows, dtype=torch.float64, device='cuda')
    ref = None
    for label, strat, choice in (("stream_cta", "stream", 0), ("stream_tma", "stream", 1), ("rb_8x2x1024", "stream", 2),
                                 ("rb_16x1x1024", "stream", 3), ("rb_16x2x512", "stream", 4), ("rb_20x1x768", "stream", 5),
                                 ("rb_24x1x640", "stream", 6), ("rb_12x2x768", "stream", 7), ("subwarp", "subwarp", 1)):
        _lib.call('wk_config_set', b'csr_kernel', choice)
        A.with_strategy(strat, 0)
        _, per = bench.timed(lambda: kernels.spmv_device(A, x, y), 20, 5, None, flush if fl else None)
        ms = statistics.mean(per)
        if ref is None:
            ref = y.clone()
        print(json.dumps({"matrix": name, "kernel": label, "ms": round(ms, 4),
                          "GB/s": round(A.algorithmic_bytes() / ms / 1e6, 1), "same_as_first": bool(torch.equal(ref, y))}))
    A.with_strategy("stream", 0)
