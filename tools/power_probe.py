"""Clocks and power while (a) the C3 step (tile kernel with the x-reuse plan) and (b) the plan-aware
stream+gather probe run back to back for ~3 s each (nvidia-smi sampled every 100 ms)."""
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import lbgen
import paper_2212_08964_b200 as lb
from bench import ClockSampler

A = lbgen.make_config("c3", "float", device="cuda")
x = lbgen.x_for_config("c3", A.cols, "float", device="cuda")
M = lb.CsrMatrix.from_csr(A)
M.plan_hot_x(0, -1)
y = torch.empty(A.rows, device="cuda")
for name, fn in (("tile_step", lambda: M.spmv(x, y, "merge_path", repartition=True)),
                 ("probe", lambda: M.probe_stream_gather(x, reps=50))):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    s = ClockSampler(0)
    s.__enter__()
    t0, n = time.perf_counter(), 0
    while time.perf_counter() - t0 < 3.0:
        fn()
        n += 1
    torch.cuda.synchronize()
    s.__exit__()
    print(json.dumps({"kernel": name, "calls": n, "clocks": s.summary()}), flush=True)
