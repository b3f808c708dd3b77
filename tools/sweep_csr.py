"""A/B of every CSR strategy / kernel configuration (wk_config_set "csr_kernel":
stream 0 = CTA per chunk, 1 = persistent TMA pipeline; rowblock 2..7 = fixed
configurations, 1 = by mean row length), L2 flushed before each launch for
the small config-1 matrix."""
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
    runs = [("rowblock_auto", "rowblock", 1, 0)] + [(f"rowblock_cfg{c}", "rowblock", c, 0) for c in range(2, 8)]
    runs += [("stream_cta", "stream", 0, 0), ("stream_tma", "stream", 1, 0), ("load_balance", "load_balance", 1, 0),
             ("merge", "merge", 1, 0)] + [(f"subwarp{t}", "subwarp", 1, t) for t in (1, 2, 4, 8)]
    for label, strat, choice, sw in runs:
        _lib.call('wk_config_set', b'csr_kernel', choice)
        A.with_strategy(strat, sw)
        _, per = bench.timed(lambda: kernels.spmv_device(A, x, y), 20, 5, None, flush if fl else None)
        ms = statistics.mean(per)
        if ref is None:
            ref = y.clone()
        print(json.dumps({"matrix": name, "kernel": label, "ms": round(ms, 4), "min_ms": round(min(per), 4),
                          "GB/s": round(A.algorithmic_bytes() / ms / 1e6, 1),
                          "max_abs_diff_vs_first": float((ref - y).abs().max())}), flush=True)
    _lib.call('wk_config_set', b'csr_kernel', 1)
    A.with_strategy("auto", 0)
