"""PCIe copy ceiling for the e2e leg: 64 MB pinned H2D alone, D2H alone, and both at once on two
streams (GB/s per direction, CUDA events; median of 10)."""
import json, sys
import numpy as np
import torch
n = 16 * 1024 * 1024
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_in = torch.empty(n, device="cuda")
d_out = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=10):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def h2d():
    s1.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


b = 4 * n
r = {k: round(b / timed(f) / 1e6, 1) for k, f in (("h2d_GBps", h2d), ("d2h_GBps", d2h))}
r["both_per_direction_GBps"] = round(b / timed(both) / 1e6, 1)
print(json.dumps(r))
