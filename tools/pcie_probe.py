"""PCIe copy-engine probe: pinned H2D, D2H and both at once (64 MB each)."""
import torch

n = 8_000_000
h_in = torch.rand(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_in = torch.empty(n, dtype=torch.float64, device="cuda")
d_out = torch.rand(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    ev = torch.cuda.Event()
    ev.record()
    s1.wait_event(ev)
    s2.wait_event(ev)
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    e1, e2 = torch.cuda.Event(), torch.cuda.Event()
    e1.record(s1)
    e2.record(s2)
    torch.cuda.current_stream().wait_event(e1)
    torch.cuda.current_stream().wait_event(e2)


h2d = t(lambda: d_in.copy_(h_in, non_blocking=True))
d2h = t(lambda: h_out.copy_(d_out, non_blocking=True))
bo = t(both)
gb = n * 8 / 1e9
print(f"H2D {h2d:.3f} ms ({gb / h2d * 1e3:.1f} GB/s)  D2H {d2h:.3f} ms ({gb / d2h * 1e3:.1f} GB/s)  "
      f"both {bo:.3f} ms ({2 * gb / bo * 1e3:.1f} GB/s aggregate)")
