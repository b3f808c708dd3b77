"""Summarise `ncu --set full` captures (tools/ncu_capture.sh) into
profiles/ncu_summary.json: per kernel, the launch's duration, DRAM bytes
read/written (the `traffic` of bench.py's roofline object), DRAM throughput,
L1/L2 sector efficiency, registers, occupancy and the top warp stall reasons.

    python tools/ncu_summarize.py gpurun_out/ncu r01b [profiles/ncu_summary.json]
"""

import csv
import io
import json
import os
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_bytes_read",
    "dram__bytes_write.sum": "dram_bytes_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "lts__t_sectors_srcunit_tex_op_read.sum": "l2_read_sectors",
    "lts__t_sector_hit_rate.pct": "l2_hit_rate_pct",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum": "l1_global_ld_sectors",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum": "l1_global_ld_requests",
    "launch__registers_per_thread": "registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__shared_mem_per_block_dynamic": "dyn_smem",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6,
              "msecond": 1e6, "nsecond": 1}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, units, data


def num(v, unit):
    v = v.replace(",", "")
    try:
        f = float(v)
    except ValueError:
        return None
    return f * UNIT_SCALE.get(unit, 1)


def summarize(rep):
    hdr, units, data = raw(rep)
    col = {h: i for i, h in enumerate(hdr)}
    out = []
    for row in data:
        k = {"kernel": row[col["Kernel Name"]][:160]}
        for m, name in METRICS.items():
            if m in col:
                k[name] = num(row[col[m]], units[col[m]])
        stalls = []
        for h, i in col.items():
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                v = num(row[i], units[i])
                name = h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]
                if v and name not in ("selected", "not_selected"):
                    stalls.append((name, v))
        stalls.sort(key=lambda t: -t[1])
        # warps stalled per issued instruction, by reason (the ncu "warp state" view)
        k["top_stalls_per_issue"] = {a: round(b, 2) for a, b in stalls[:5]}
        iss = "smsp__issue_active.avg.pct_of_peak_sustained_active"
        if iss in col:
            k["issue_active_pct"] = num(row[col[iss]], units[col[iss]])
        if k.get("l1_global_ld_requests"):
            k["sectors_per_request"] = round(k["l1_global_ld_sectors"] / k["l1_global_ld_requests"], 2)
        if k.get("dram_bytes_read") is not None and k.get("duration_ns"):
            tot = k["dram_bytes_read"] + (k.get("dram_bytes_write") or 0)
            k["dram_gbs"] = round(tot / k["duration_ns"], 1)
        out.append(k)
    return out


def main():
    d, tag = sys.argv[1], sys.argv[2]
    dst = sys.argv[3] if len(sys.argv) > 3 else os.path.join("profiles", "ncu_summary.json")
    try:
        with open(dst) as fh:
            summary = json.load(fh)
    except FileNotFoundError:
        summary = {"kernels": {}}
    summary["source"] = f"ncu --set full --clock-control none captures ({tag}), tools/ncu_capture.sh"
    for f in sorted(os.listdir(d)):
        if not (f.startswith(tag + "_") and f.endswith(".ncu-rep")):
            continue
        name = f[len(tag) + 1:-len(".ncu-rep")]
        ks = summarize(os.path.join(d, f))
        if not ks:
            continue
        # the dominant launch (longest) represents the capture
        main_k = max(ks, key=lambda k: k.get("duration_ns") or 0)
        main_k["launches_captured"] = len(ks)
        main_k["capture"] = tag
        summary["kernels"][name] = main_k
        print(name, json.dumps(main_k)[:300])
    os.makedirs(os.path.dirname(dst), exist_ok=True)
    with open(dst, "w") as fh:
        json.dump(summary, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
