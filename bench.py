#!/usr/bin/env python
"""Benchmark of the B200 sparse fp64 hot path (driver contract: one JSON line).

Headline (N=1): BASELINE config 2 — fp64 SELL-P(64) SpMV on the 3-D 27-point
stencil 200^3 (8M rows, 213.8M nonzeros), matrix and vectors resident in HBM.
A step is one SpMV y = A x. `value` is GFLOP/s (2 * true nnz per SpMV). The
operands (2.7 GB per SpMV) are 21x the 126 MB L2, so consecutive steps cannot
hit in L2 (no flush needed; stated in `config`).

N > 1 (torchrun): row-block (z-slab) partitioned SpMV, weak scaling — rank g
owns a 200x200x200 slab of a 200x200x(200N) grid, halo planes exchanged over
NCCL inside every step (see paper_2006_14290_b200/distributed.py).

Extra keys (N=1): `formats` (CSR cfg1 with L2 flush, ELL cfg2, CSR->ELL and
CSR->SELL-P conversions, COO and Hybrid on R-MAT scale 24), `cg` (cfg4: 1000
CG iterations on the 7-point 256^3 Laplacian, SELL-P) and, for every N, the
distributed CG iteration rate.

--impl reference: the reference's algorithm on the host cores (the CPU
restatement in oracle/, C + OpenMP, all threads) on the same workload,
bounded samples; rank 0 only.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 SpMV GFLOP/s & HBM GB/s per format; CG iterations/sec at 1/2/4/8 B200"
GRID = 200          # config 2: 27-point stencil on GRID^3
SLICE = 64
CG_GRID = 256       # config 4
CG_ITERS = 1000
RMAT_SCALE = 24     # config 3


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---- clocks ------------------------------------------------------------------------------


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index=0):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-f", self.path], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if self.path is None or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as fh:
            for line in fh:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    smax.append(float(parts[2]))
                except ValueError:
                    continue
                for nm, v in zip(names, parts[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "samples": len(sm),
                "reasons": sorted(reasons)}


# ---- timing --------------------------------------------------------------------------------


def barrier(dist):
    if dist is not None:
        dist.barrier()


def timed(fn, steps, warmup, dist=None, flush=None):
    """W untimed warm-up calls, then K timed calls bracketed by barrier +
    synchronize; per-call CUDA events on the launching (current) stream.
    Returns (total_ms over the K calls, per-call ms list). With `flush`, an
    L2-flushing write runs before every call, outside the per-call events
    (total_ms then sums the per-call times)."""
    import torch

    for _ in range(warmup):
        if flush is not None:
            flush()
        fn()
    torch.cuda.synchronize()
    barrier(dist)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for a, b in ev:
        if flush is not None:
            flush()
        a.record(stream)
        fn()
        b.record(stream)
    t1.record(stream)
    torch.cuda.synchronize()
    barrier(dist)
    per = [a.elapsed_time(b) for a, b in ev]
    total = sum(per) if flush is not None else t0.elapsed_time(t1)
    return total, per


def max_over_ranks(v, dist):
    if dist is None:
        return v
    import torch

    dev = "cpu" if str(dist.get_backend()).lower() == "gloo" else "cuda"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sellp_bytes(d):
    return d.algorithmic_bytes()


def load_traffic(name):
    """DRAM bytes per launch of `name` from the committed ncu --set full
    summary (a STATIC capture, not measured in this run: ncu replays a kernel
    ~40 times and cannot run inside the timed region). Returns (bytes,
    source description) or (None, reason)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as fh:
            s = json.load(fh)
        k = s["kernels"][name]
        return (int(k["dram_bytes_read"] + k["dram_bytes_write"]),
                f"static: profiles/ncu_summary.json [{name}], {s.get('source', '')}")
    except Exception as exc:  # noqa: BLE001
        return None, f"unavailable ({exc.__class__.__name__})"


# ---- CPU baseline (oracle C port, all host threads) ---------------------------------------------


def workload_config(rows, nnz, stored, nbytes, world=1):
    """`config` of the N=1 headline, shared verbatim by the reference arm."""
    return {"workload": f"SELL-P({SLICE}) SpMV, 27-point stencil {GRID}^3 per GPU (BASELINE config 2)",
            "rows_per_gpu": int(rows), "nnz_per_gpu": int(nnz), "stored_per_gpu": int(stored),
            "bytes_per_spmv": int(nbytes),
            "l2": "operands 2.7 GB/step >> 126 MB L2: no flush needed between steps",
            "parallelism": f"rowblock{world}"}


def cpu_matrix():
    """The whole config-2 matrix (27-point 200^3, SELL-P(64)) built on the
    host by the oracle's C builders (oracle.native.stencil_csr /
    csr_to_sellp, equal to the numpy restatements, tests/test_oracle_golden.py)."""
    from oracle import corpus_ref, native

    m = native.stencil_csr(GRID, GRID, GRID, corpus_ref.points_27pt())
    sp = native.csr_to_sellp(m, SLICE)
    nnz = int(m.row_ptrs[-1])
    del m
    return sp, nnz


def cpu_sample(budget_s=10.0, steps=None, matrix=None):
    """The reference fold (oracle/csrc/oracle.c or_spmv_sellp: per row
    acc = 0.0; acc += v * x[c], sparse.py:397-417) of the WHOLE config-2
    matrix on every host thread; x = default_rng(42).random(n) as the
    reference's bench (bench.py:233-234)."""
    from oracle import native

    sp, nnz = matrix if matrix is not None else cpu_matrix()
    prep = native.Prepared(sp)
    x = np.random.default_rng(42).random(sp.ncols)
    threads = native.max_threads()
    y = prep.spmv(x, nthreads=threads)  # warm-up
    times = []
    t_start = time.perf_counter()
    while True:
        t = time.perf_counter()
        prep.spmv(x, y, nthreads=threads)
        times.append(time.perf_counter() - t)
        if steps is not None and len(times) >= steps:
            break
        if steps is None and time.perf_counter() - t_start > budget_s:
            break
    mean = sum(times) / len(times)
    stored = len(sp.values)
    nbytes = 12 * stored + 8 * (len(sp.slice_sets)) + 8 * sp.ncols + 8 * sp.nrows
    sample = (f"the whole config-2 matrix ({sp.nrows} rows, {nnz} nnz, {stored} stored), SELL-P({SLICE}), "
              f"{len(times)} reps")
    return {"value": round(2 * nnz / mean / 1e9, 4), "unit": "GFLOP/s", "cores": threads, "kind": "port",
            "sample": sample, "ms_per_rep": round(mean * 1e3, 3), "impl": "oracle/csrc/oracle.c or_spmv_sellp",
            "nnz": nnz, "stored": stored, "bytes_per_spmv": nbytes, "rows": sp.nrows, "host": host_info()}, times


def host_info():
    """CPU model and logical CPU count of the host the CPU baseline ran on."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def cpu_per_config(wk, corpus, D, reps=10):
    """The reference algorithm on the host cores for the other BASELINE
    configs (oracle/csrc/oracle.c, all threads, sequential per-row fold): the
    CPU side of each GPU number in `formats` / `cg`. Bounded samples."""
    import torch

    from oracle import corpus_ref, native

    threads = native.max_threads()
    res = {}

    def spmv_rate(prep, x, nnz, label, sample):
        y = prep.spmv(x, nthreads=threads)
        t0 = time.perf_counter()
        for _ in range(reps):
            prep.spmv(x, y, nthreads=threads)
        ms = (time.perf_counter() - t0) / reps * 1e3
        res[label] = {"GFLOP/s": round(2 * nnz / (ms * 1e-3) / 1e9, 3), "ms": round(ms, 3), "cores": threads,
                      "kind": "port", "sample": sample}

    # config 1: CSR 5-point Poisson 1000^2, the whole matrix
    m = corpus_ref.poisson2d(1000)
    spmv_rate(native.Prepared(m), np.random.default_rng(42).random(m.ncols), int(m.row_ptrs[-1]),
              "cfg1_csr_poisson2d_1000", "whole matrix, or_spmv_csr")
    # config 1 with the reference AS SHIPPED (warpkit's pure-Python sequential
    # oracle, one core) on the first 100k rows, when the offline install of the
    # reference (baseline/_ref) is present
    ref = _shipped_reference()
    if ref is not None:
        rows = 100_000
        e = int(m.row_ptrs[rows])
        sub = ref.sparse.CsrMatrix(rows, m.ncols, np.asarray(m.row_ptrs[: rows + 1], np.int64),
                                   np.asarray(m.col_idx[:e], np.int64), np.asarray(m.values[:e], np.float64))
        x1 = np.random.default_rng(42).random(m.ncols)
        t0 = time.perf_counter()
        ref.sparse.dense_spmv_reference(sub, x1)
        sec = time.perf_counter() - t0
        res["cfg1_reference_as_shipped"] = {
            "GFLOP/s": round(2 * e / sec / 1e9, 5), "ms": round(sec * 1e3, 1), "cores": 1, "kind": "reference",
            "sample": f"warpkit.sparse.dense_spmv_reference on the first {rows} rows ({e} nnz) of the "
                      f"5-point Poisson 1000^2 matrix (pure Python, sparse.py:367-430)"}
    # config 3: COO R-MAT scale 24, the first 32M sorted entries (the dense rows)
    R = corpus.rmat(RMAT_SCALE)
    k = min(R.nnz, 32 << 20)
    from types import SimpleNamespace

    nrows_s = int(R.row_idx[k - 1].item()) + 1
    coo = SimpleNamespace(nrows=nrows_s, ncols=R.ncols, row_idx=R.row_idx[:k].cpu().numpy(),
                          col_idx=R.col_idx[:k].cpu().numpy(), values=R.values[:k].cpu().numpy())
    del R
    spmv_rate(native.Prepared(coo), np.random.default_rng(42).random(coo.ncols), k, "cfg3_coo_rmat24_sample",
              f"first {k} sorted entries (rows 0..{nrows_s - 1}), or_spmv_coo")
    del coo
    torch.cuda.empty_cache()
    # config 4: CG on the 7-point 256^3 Laplacian, SELL-P(64), 20 iterations
    A = D.csr_to_sellp(corpus.stencil3d(CG_GRID, 7), SLICE)
    prep = native.Prepared(A.to_host())
    del A
    torch.cuda.empty_cache()
    b = np.ones(prep.nrows)
    its = 20
    t0 = time.perf_counter()
    _, hist = prep.cg(b, 1e-30, its, nthreads=threads)
    sec = time.perf_counter() - t0
    res["cfg4_cg_256"] = {"it_per_s": round((len(hist) - 1) / sec, 2), "iterations": len(hist) - 1,
                          "ms": round(sec * 1e3, 1), "cores": threads, "kind": "port",
                          "sample": f"{its} iterations of the whole system, or_cg_sellp"}
    return res


def _shipped_reference():
    """warpkit from the offline install baseline/_ref (None if absent)."""
    root = os.path.join(os.path.dirname(os.path.abspath(__file__)), "baseline", "_ref")
    if not os.path.isdir(os.path.join(root, "warpkit")):
        return None
    if root not in sys.path:
        sys.path.append(root)
    try:
        import warpkit
        import warpkit.sparse  # noqa: F401
    except Exception:
        return None
    return warpkit


def run_reference(args, rank):
    if rank != 0:
        return
    from oracle import native

    native.lib()
    base, times = cpu_sample(steps=args.steps + args.warmup)
    times = times[args.warmup:] or times
    ms = 1e3 * sum(times) / len(times)
    base["value"] = round(2 * base["nnz"] / (ms * 1e-3) / 1e9, 4)
    line = {
        "impl": "reference", "metric": METRIC, "value": base["value"], "unit": "GFLOP/s", "n_gpus": args.gpus,
        "steps": len(times), "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(base["rows"], base["nnz"], base["stored"], base["bytes_per_spmv"]),
        "cpu_baseline": base,
        "e2e": {"value": base["value"], "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---- GPU arm ---------------------------------------------------------------------------------


def run_gpu(args, rank, world, dist):
    import torch

    import paper_2006_14290_b200 as wk
    from paper_2006_14290_b200 import corpus
    from paper_2006_14290_b200 import device as D

    dev = torch.device("cuda", torch.cuda.current_device())
    ex = wk.make_executor("b200", device=dev.index)
    peak, peak_src = peaks()
    out = {}

    comm_mode = None
    if world == 1:
        A_csr = corpus.stencil3d(GRID, 27)
        A = D.csr_to_sellp(A_csr, SLICE)
        nnz = A_csr.nnz
    else:
        from paper_2006_14290_b200 import distributed as DI

        part = DI.stencil_slab_operator(GRID, GRID, GRID, corpus.points_27pt(), dist, fmt="sellp",
                                        slice_size=SLICE)
        comm_mode = DI.maybe_enable_peer(part)
        A = part.local
        nnz = part.local_nnz
    n_local = A.nrows
    x = torch.rand(A.ncols, dtype=torch.float64, device=dev, generator=torch.Generator(device=dev).manual_seed(42))
    if world > 1:
        xe = part.new_vector()  # in the peer arena when the peer path is on
        xe.copy_(x)
        x = xe
    y = torch.empty(n_local, dtype=torch.float64, device=dev)
    if world == 1:
        step = lambda: wk.kernels.spmv_device(A, x, y)  # noqa: E731
    else:
        step = lambda: part.spmv(x, y)  # noqa: E731

    with ClockSampler(dev.index) as clk:
        total_ms, per = timed(step, args.steps, args.warmup, dist)
    clocks = clk.summary()
    total_ms = max_over_ranks(total_ms, dist)
    flops_all = 2.0 * nnz * args.steps * world
    value = flops_all / (total_ms * 1e-3) / 1e9
    # roofline of the dominant kernel (the SELL-P SpMV launch): per-launch events
    if world == 1:
        kernel_ms = statistics.mean(per)
    else:
        _, kper = timed(lambda: wk.kernels.spmv_device(A, x, y), args.steps, args.warmup, dist)
        kernel_ms = statistics.mean(kper)
    bytes_launch = sellp_bytes(A)
    achieved = bytes_launch / (kernel_ms * 1e-3) / 1e9

    # end to end through the public API: pinned host x in, pinned host y out
    e2e = None
    if True:
        xh = x[: A.ncols].cpu().pin_memory() if world == 1 else None
        if world == 1:
            # the host-to-host pipeline of the public API (paper_2006_14290_b200.SpmvPipeline):
            # copy-in, SpMV row blocks and copy-out overlapped on three streams,
            # consecutive steps in flight on two buffer sets
            pipe = wk.SpmvPipeline(A)
            yhs = [torch.empty(n_local, dtype=torch.float64, pin_memory=True) for _ in range(2)]
            # a streaming pipeline: the first copy-in and the last SpMV +
            # copy-out (~1.5 ms) are not overlapped; 40+ steps keep that
            # fill / drain under 3% of the timed region
            e_steps = max(40, args.steps)
            for k in range(3):
                pipe.submit(xh, yhs[k % 2])
            pipe.synchronize()
            torch.cuda.synchronize()
            barrier(dist)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(pipe.s_h2d)
            for k in range(e_steps):
                pipe.submit(xh, yhs[k % 2])
            e1.record(pipe.s_d2h)
            torch.cuda.synchronize()
            e_ms = e0.elapsed_time(e1)
            # the synchronous single-call API, for reference
            s_ms, _ = timed(lambda: wk.spmv_sellp(A, xh, ex), e_steps, 2, dist)
            e2e = {"value": round(2.0 * nnz * e_steps / (e_ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
                   "h2d_bytes_per_step": int(pipe.h2d_bytes), "d2h_bytes_per_step": int(pipe.d2h_bytes),
                   "ms_per_step": round(e_ms / e_steps, 4), "steps": e_steps,
                   "api": "paper_2006_14290_b200.SpmvPipeline(A).submit(pinned x, pinned y)",
                   "sync_api_ms_per_step": round(s_ms / e_steps, 4),
                   "sync_api": "paper_2006_14290_b200.spmv_sellp(A, pinned x)"}
        else:
            e2e = part.e2e(x, args, timed)

    if world > 1:
        comm_how = 'NVLink peer stores' if comm_mode == 'peer' else comm_mode.upper()
        part_desc = f", z-slab partitioned {GRID}x{GRID}x{GRID * world}, halo over {comm_how}"
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(n_local, nnz, A.stored, bytes_launch, world),
        "hbm_gbs": round(bytes_launch * args.steps * world / (total_ms * 1e-3) / 1e9, 1),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "frac_of_8tbs": round(achieved / 8000.0, 4),
                     "peak_source": peak_src, "traffic": load_traffic("sellp_spmv")[0],
                     "traffic_source": load_traffic("sellp_spmv")[1],
                     "kernel": "sellp64_tma_kernel<J=4,S=3,W=16> (SELL-P(64), TMA bulk-copy ring, 2 rows/lane)",
                     "kernel_ms": round(kernel_ms, 4), "algorithmic_bytes": int(bytes_launch)},
        "e2e": e2e,
        "gpu_launches": args.steps * (1 if world == 1 else part.launches_per_spmv),
        **({"partition": part_desc.lstrip(", ")} if world > 1 else {}),
        "clocks": clocks,
        "comm": {"nranks": world, "backend": str(dist.get_backend()).lower() if dist is not None else None,
                 "data_path": comm_mode if world > 1 else "none (1 GPU)",
                 "halo_bytes_per_spmv": int(part.plan.bytes_per_exchange) if world > 1 else 0},
    }
    # extra sections
    if world == 1 and not args.quick:
        out["formats"] = bench_formats(args, wk, corpus, D, A_csr, A, x, peak)
        del A_csr
        torch.cuda.empty_cache()
        out["cg"] = _safe(lambda: bench_cg(args, wk, corpus, D))
        torch.cuda.empty_cache()
        out["nonsymmetric"] = _safe(lambda: bench_nonsym(args, wk, corpus, D))
        torch.cuda.empty_cache()
        line["cpu_baseline"] = cpu_sample(budget_s=args.cpu_budget)[0] if not args.no_cpu else None
        if not args.no_cpu:
            out["cpu_baselines"] = _safe(lambda: cpu_per_config(wk, corpus, D))
    elif world > 1 and not args.quick:
        # strong scaling of CG 256^3 (north_star: >= 6x at 8 GPUs): the same
        # solve on rank 0's GPU alone first (the other ranks wait), then
        # partitioned over all ranks
        single = None
        if rank == 0:
            single = _safe(lambda: bench_cg(args, wk, corpus, D))
            torch.cuda.empty_cache()
        barrier(dist)
        out["cg"] = _safe(lambda: part_cg(args, dist, world))
        if rank == 0 and "it_per_s" in out["cg"] and single and "it_per_s" in single:
            out["cg"]["single_gpu_it_per_s"] = single["it_per_s"]
            out["cg"]["speedup_vs_1gpu"] = round(out["cg"]["it_per_s"] / single["it_per_s"], 3)
            line["cg_strong_it_per_s"] = out["cg"]["it_per_s"]
            line["cg_strong_speedup_vs_1gpu"] = out["cg"]["speedup_vs_1gpu"]
        torch.cuda.empty_cache()
        out["nonsymmetric"] = _safe(lambda: part_nonsym(args, dist, world))
    line.update(out)
    if rank == 0:
        print(json.dumps(line), flush=True)


def bench_formats(args, wk, corpus, D, A_csr, A_sellp, x, peak):
    import torch

    res = {}
    K, W = max(5, args.steps // 2), 3
    flush_buf = torch.ones(512 * 1024 * 1024 // 8, dtype=torch.float64, device=x.device)

    def flush():
        # read (not write) 512 MB: evicts the L2 without leaving dirty lines
        # whose write-back would be charged to the timed kernel
        flush_buf.sum()

    def rec(name, d, xx, flush_l2=False, nnz=None):
        yy = torch.empty(d.nrows, dtype=torch.float64, device=x.device)
        _, per = timed(lambda: wk.kernels.spmv_device(d, xx, yy), K, W, None, flush if flush_l2 else None)
        ms = statistics.mean(per)
        b = d.algorithmic_bytes()
        nz = d.nnz if nnz is None else nnz
        res[name] = {"ms": round(ms, 4), "min_ms": round(min(per), 4), "GFLOP/s": round(2 * nz / (ms * 1e-3) / 1e9, 2),
                     "GB/s": round(b / (ms * 1e-3) / 1e9, 1), "frac_hbm": round(b / (ms * 1e-3) / 1e9 / peak, 4),
                     "bytes": int(b), "nnz": int(nz)}
        if flush_l2:
            res[name]["l2"] = "flushed (512 MB read) before every launch"
        return yy

    rec("sellp_27pt_200", A_sellp, x)
    for strat in ("rowblock", "load_balance", "merge", "stream", "subwarp"):
        A_csr.with_strategy(strat, 0)
        rec(f"csr_{strat}_27pt_200", A_csr, x)
    A_csr.with_strategy("auto", 0)
    ell = D.csr_to_ell(A_csr)
    rec("ell_27pt_200", ell, x)
    del ell
    torch.cuda.empty_cache()
    # conversions (read CSR, write ELL / SELL-P)
    for name, fn in (("csr_to_ell", lambda: D.csr_to_ell(A_csr, width=27)),
                     ("csr_to_sellp", lambda: D.csr_to_sellp(A_csr, SLICE))):
        _, per = timed(fn, 3, 1, None)
        ms = statistics.mean(per)
        if name == "csr_to_ell":
            b = A_csr.nnz * 12 + 4 * (A_csr.nrows + 1) + 27 * A_csr.nrows * 12 + 4 * A_csr.nrows
        else:
            b = A_csr.nnz * 12 + 4 * (A_csr.nrows + 1) + A_sellp.stored * 12 + 8 * (A_sellp.nslices + 1) + 4 * A_csr.nrows
        res[name] = {"ms": round(ms, 3), "GB/s": round(b / (ms * 1e-3) / 1e9, 1), "bytes": int(b),
                     "note": "includes the host sync reading the total storage size"}
        torch.cuda.empty_cache()
    # config 1: CSR on the 2-D Poisson 1000^2 (80 MB: flush L2 before every launch)
    P = corpus.poisson2d_matrix(1000)
    xp = torch.rand(P.ncols, dtype=torch.float64, device=x.device)
    for strat in ("rowblock", "load_balance", "merge", "stream"):
        P.with_strategy(strat, 0)
        rec(f"csr_{strat}_poisson2d_1000", P, xp, flush_l2=True)
    del P
    # config 3: COO and Hybrid on R-MAT scale 24
    R = corpus.rmat(RMAT_SCALE)
    xr = torch.rand(R.ncols, dtype=torch.float64, device=x.device)
    rec("coo_rmat24", R, xr)
    Rc = D.coo_to_csr(R)
    for strat in ("load_balance", "merge", "stream"):
        Rc.with_strategy(strat, 0)
        rec(f"csr_{strat}_rmat24", Rc, xr)
    # Hybrid: Ginkgo's minimal-storage width (0 on R-MAT: 56% of the rows are
    # empty, any ELL slot costs more than the COO entry it replaces) and a
    # real split, ELL width k = 8 (12kn + 16 rem + 16n)
    H = D.csr_to_hybrid(Rc)
    rec("hybrid_rmat24", H, xr, nnz=R.nnz)
    res["hybrid_rmat24"].update(ell_width=H.ell.width, coo_nnz=H.coo.nnz, strategy="minimal_storage")
    del H
    torch.cuda.empty_cache()
    _, per = timed(lambda: D.csr_to_hybrid(Rc, width=8), 3, 1, None)
    H = D.csr_to_hybrid(Rc, width=8)
    ms = statistics.mean(per)
    b = 12 * Rc.nnz + 4 * (Rc.nrows + 1) + 12 * 8 * Rc.nrows + 4 * Rc.nrows + 16 * H.coo.nnz + 8 * (Rc.nrows + 1)
    res["csr_to_hybrid_k8_rmat24"] = {"ms": round(ms, 3), "GB/s": round(b / (ms * 1e-3) / 1e9, 1), "bytes": int(b),
                                      "note": "read CSR, write ELL(8) + lengths, COO offsets + remainder; "
                                              "includes the host sync reading the remainder size"}
    rec("hybrid_k8_rmat24", H, xr, nnz=R.nnz)
    res["hybrid_k8_rmat24"].update(ell_width=H.ell.width, ell_real_nnz=int(H.ell.nnz), coo_nnz=H.coo.nnz)
    del R, Rc, H, flush_buf
    torch.cuda.empty_cache()
    # device ingestion of the raw R-MAT edge list (from_entries, sparse.py:63-80):
    # stable radix sort of (row * 2^24 + col, value) over 48 key bits (6 passes
    # of 8), duplicate offsets (scan) and the in-order duplicate fold
    keys0, vals0 = corpus.rmat_edge_keys(RMAT_SCALE)
    kb, vb = torch.empty_like(keys0), torch.empty_like(vals0)
    n_r = 1 << RMAT_SCALE
    m = keys0.numel()

    def setup():
        kb.copy_(keys0)
        vb.copy_(vals0)

    out = {}

    def ingest():
        out["coo"] = D.coo_from_keys(n_r, n_r, kb, vb, sum_duplicates=True, owned=True)

    _, per = timed(ingest, 3, 1, None, flush=setup)
    ms = statistics.mean(per)
    nu = out["coo"].nnz
    passes = (2 * RMAT_SCALE + 7) // 8
    # sort: per pass 8 B (histogram read) + 16 B read + 16 B write per pair;
    # duplicate fold: keys read twice, values once, 16 B per unique entry out
    moved = m * (passes * 40 + 24) + nu * 16
    res["from_entries_rmat24"] = {
        "ms": round(ms, 3), "entries": int(m), "unique": int(nu), "Gentries/s": round(m / (ms * 1e-3) / 1e9, 2),
        "GB/s": round(moved / (ms * 1e-3) / 1e9, 1), "bytes_moved": int(moved),
        "note": "stable LSD radix sort (csrc/sort.cu: per pass 8 B upsweep read + 16 B read + 16 B write per "
                "entry) + tiled duplicate count / fold; includes one D2H read of the unique count"}
    del keys0, vals0, kb, vb, out
    torch.cuda.empty_cache()
    return res


def bench_cg(args, wk, corpus, D):
    import torch

    A = D.csr_to_sellp(corpus.stencil3d(CG_GRID, 7), SLICE)
    b = torch.ones(A.nrows, dtype=torch.float64, device="cuda")
    ex = wk.make_executor("b200")
    wk.cg_solve(A, b, 1e-30, 60, ex)  # warm-up (graph capture path, caches)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    x, hist = wk.cg_solve(A, b, 1e-30, CG_ITERS, ex)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    it = len(hist) - 1
    spmv_b = A.algorithmic_bytes()
    # SpMV + vector passes per 50-iteration period: iterations 0..47 in pairs
    # (r, q -> r twice; p, r -> p'; x, p_prev, p, r -> x, p'': 15 vectors per
    # pair), iteration 48 with 8 (r, q -> r; x, p, r -> x, p), the
    # residual-replacement iteration with 9 (x/r then p) plus SpMV(x) and
    # r = b - q
    per_it = spmv_b + (24 * 120 + 64 + 72) * A.nrows / 50 + (spmv_b + 24 * A.nrows) / 50
    # the CG operator's plain SpMV (narrow SELL-P configuration: 7-wide slices)
    xs = torch.rand(A.ncols, dtype=torch.float64, device="cuda")
    ys = torch.empty(A.nrows, dtype=torch.float64, device="cuda")
    _, per = timed(lambda: wk.kernels.spmv_device(A, xs, ys), 20, 3, None)
    sp_ms = statistics.mean(per)
    return {"workload": f"CG, 7-point Laplacian {CG_GRID}^3, SELL-P({SLICE}), b = ones, tol 1e-30, {CG_ITERS} iterations",
            "iterations": it, "ms": round(ms, 2), "it_per_s": round(it / (ms * 1e-3), 1),
            "GB/s_effective": round(per_it * it / (ms * 1e-3) / 1e9, 1), "bytes_per_iteration": int(per_it),
            "n_gpus": 1,
            "operator_spmv": {"ms": round(sp_ms, 4), "GB/s": round(spmv_b / (sp_ms * 1e-3) / 1e9, 1),
                              "bytes": int(spmv_b), "GFLOP/s": round(2 * A.nnz / (sp_ms * 1e-3) / 1e9, 1),
                              "kernel": "sellp64_tma_kernel<J=2,S=5,W=24> (narrow: slices <= 12 wide)"}}


def _safe(fn):
    """Extra sections must never take the headline line down with them."""
    try:
        return fn()
    except Exception as exc:  # pragma: no cover - reported in the JSON line
        return {"error": f"{type(exc).__name__}: {exc}"}


NONSYM_GRID = 512   # config 5: 7-point convection-diffusion 512^3
NONSYM_ITERS = {"bicgstab": 50, "gmres": 60}


def _nonsym_bytes(n, spmv_b, kind, iters, restart=30):
    """Algorithmic bytes per iteration: BiCGSTAB = 2 SpMV + 15 vector passes
    (p update 4, s update 3, x/r update + rh.r 7, rh read by the fused r-hat.v
    of the first SpMV 1; t.t / t.s fused into the second SpMV);
    GMRES(m) inner step j = SpMV + (2j + 4) vector passes (CGS dots, update
    with the norm; the new direction is not rescaled: deferred normalisation),
    averaged over the iterations run, + one SpMV and 4 passes per restart."""
    if kind == "bicgstab":
        return 2 * spmv_b + 15 * 8 * n
    steps = [(i % restart) for i in range(iters)]
    cyc = max(1, -(-iters // restart))
    tot = sum(spmv_b + (2 * j + 4) * 8 * n for j in steps) + cyc * (spmv_b + 4 * 8 * n)
    return tot / max(iters, 1)


def bench_nonsym(args, wk, corpus, D):
    import torch

    A = D.csr_to_sellp(corpus.convection_diffusion3d(NONSYM_GRID), SLICE)
    torch.cuda.empty_cache()
    b = torch.ones(A.nrows, dtype=torch.float64, device="cuda")
    ex = wk.make_executor("b200")
    out = {"workload": f"7-point convection-diffusion {NONSYM_GRID}^3 (beta = (1, 0.5, 0.25)), SELL-P({SLICE}), "
                       f"b = ones, tol 1e-30, fixed iteration counts", "n_gpus": 1}
    for kind, fn in (("bicgstab", lambda it: wk.bicgstab_solve(A, b, 1e-30, it, ex)),
                     ("gmres", lambda it: wk.gmres_solve(A, b, 1e-30, it, ex, restart=30))):
        iters = NONSYM_ITERS[kind]
        fn(4)
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        x, hist = fn(iters)
        t1.record()
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1)
        it = len(hist) - 1
        per_it = _nonsym_bytes(A.nrows, A.algorithmic_bytes(), kind, it)
        out[kind] = {"iterations": it, "ms": round(ms, 2), "it_per_s": round(it / (ms * 1e-3), 2),
                     "GB/s_effective": round(per_it * it / (ms * 1e-3) / 1e9, 1), "bytes_per_iteration": int(per_it)}
    return out


def part_nonsym(args, dist, world):
    from paper_2006_14290_b200 import distributed as DI

    return DI.bench_nonsym(NONSYM_GRID, NONSYM_ITERS, dist)


def part_cg(args, dist, world):
    from paper_2006_14290_b200 import distributed as DI

    return DI.bench_cg(CG_GRID, CG_ITERS, dist, timed)


def _free_port():
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def spawn_ranks(args):
    """`python bench.py --gpus N` without a torchrun environment: relaunch
    this script under torch.distributed.run with N ranks (one per GPU,
    rendezvous on 127.0.0.1) and return its exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--quick", action="store_true", help="headline only")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        # host-only arm: rank 0 times the CPU restatement, other ranks exit
        run_reference(args, rank)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if world != args.gpus and os.environ.get("WK_DIST_BACKEND", "nccl") == "nccl":
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started {world} ranks")
    import torch

    local = int(os.environ.get("LOCAL_RANK", "0"))
    # WK_DIST_BACKEND=gloo lets the N>1 path run with several ranks on one
    # GPU (host-staged exchange) to test it; the driver's runs use NCCL.
    backend = os.environ.get("WK_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend == "gloo" else local
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as tdist

        if backend == "nccl":
            # communicator init lines (rank / nRanks) for the launcher's rank check
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            tdist.init_process_group(backend)
        dist = tdist
    run_gpu(args, rank, world, dist)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
