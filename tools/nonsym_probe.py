"""BiCGSTAB / GMRES(30) on the 7-point convection-diffusion 512^3 (BASELINE
config 5) exactly as bench.py times them (development A/B)."""
import json
import sys
import types

sys.path.insert(0, '.')
import bench  # noqa: E402
import paper_2006_14290_b200 as wk  # noqa: E402
from paper_2006_14290_b200 import corpus  # noqa: E402
from paper_2006_14290_b200 import device as D  # noqa: E402

print(json.dumps(bench.bench_nonsym(types.SimpleNamespace(), wk, corpus, D)))
