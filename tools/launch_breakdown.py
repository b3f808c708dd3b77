"""Aggregate an `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv` launch list per kernel name: launches, total
time, share, DRAM GB/s. python tools/launch_breakdown.py LIST.csv [skip-regex]"""
import collections
import csv
import re
import sys

SCALE = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'nsecond': 1, 'usecond': 1e3, 'msecond': 1e6}


def main():
    path = sys.argv[1]
    skip = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
    rows = list(csv.reader(line for line in open(path) if not line.startswith('==')))
    hdr, data = rows[0], rows[1:]
    iK, iM, iV, iU, iID = (hdr.index(c) for c in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'))
    per, names = collections.defaultdict(dict), {}
    for r in data:
        if not r[iID].isdigit():
            continue
        k = int(r[iID])
        names[k] = r[iK]
        per[k][r[iM]] = float(r[iV].replace(',', '')) * SCALE.get(r[iU], 1)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for k, m in per.items():
        name = names[k].split('(')[0]
        if skip and skip.search(name):
            continue
        a = agg[name]
        a[0] += 1
        a[1] += m.get('gpu__time_duration.sum', 0.0)
        a[2] += m.get('dram__bytes_read.sum', 0.0) + m.get('dram__bytes_write.sum', 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':70s} {'launches':>8s} {'time_us':>10s} {'share':>6s} {'DRAM GB/s':>9s}")
    for name, a in sorted(agg.items(), key=lambda t: -t[1][1]):
        print(f"{name[:70]:70s} {a[0]:8d} {a[1] / 1e3:10.1f} {100 * a[1] / tot:5.1f}% {a[2] / a[1] if a[1] else 0:9.1f}")


if __name__ == "__main__":
    main()
