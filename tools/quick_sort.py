"""CUDA-event timing of the device ingestion of R-MAT scale 24 (development
probe; bench.py is the contract): the stable radix sort alone, torch.sort +
gather for comparison, and the whole coo_from_keys."""
import sys

import torch

sys.path.insert(0, '.')
from paper_2006_14290_b200 import corpus  # noqa: E402
from paper_2006_14290_b200 import device as D  # noqa: E402


def t(fn, setup, n=3):
    setup()
    fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(n):
        setup()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / n


scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
k0, v0 = corpus.rmat_edge_keys(scale)
kb, vb = torch.empty_like(k0), torch.empty_like(v0)


def setup():
    kb.copy_(k0)
    vb.copy_(v0)


bits = 2 * scale
print("entries", k0.numel(), "key bits", bits, flush=True)
print("sort_pairs (ours, in place):", round(t(lambda: D.sort_pairs(kb, vb, bits, inplace=True), setup), 3), "ms", flush=True)
sk, sv = D.sort_pairs(kb.clone(), vb.clone(), bits, inplace=True)


def torch_sort():
    s, p = torch.sort(kb, stable=True)
    return s, vb[p]


print("torch.sort + gather:", round(t(torch_sort, setup), 3), "ms", flush=True)
ts, tv = torch_sort()
print("equal to torch stable sort:", torch.equal(ts, sk) and torch.equal(tv, sv), flush=True)
n = 1 << scale
print("coo_from_keys (ours):", round(t(lambda: D.coo_from_keys(n, n, kb, vb, owned=True), setup), 3), "ms", flush=True)
