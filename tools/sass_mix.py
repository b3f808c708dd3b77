"""Warp-instruction mix of one ncu report (SASS source page), by opcode:
python tools/sass_mix.py REPORT.ncu-rep"""
import collections
import csv
import io
import re
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
start = next(i for i, r in enumerate(rows) if "Source" in r and "Address" in r)
hdr, data = rows[start], rows[start + 1:]
cand = [h for h in hdr if h.startswith("Instructions Executed")] or [h for h in hdr if "Instructions" in h]
iI, iS = hdr.index(cand[0]), hdr.index("Source")
agg, tot = collections.Counter(), 0.0
for r in data:
    try:
        n = float(r[iI])
    except (ValueError, IndexError):
        continue
    op = re.sub(r"^@!?U?P\w+\s+", "", r[iS].strip()).split(" ")[0].split(".")[0]
    agg[op] += n
    tot += n
print(f"{sys.argv[1]}: {tot:.4g} warp instructions")
print("  " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in agg.most_common(16)))
