"""A/B of the x-reuse plan's warm modes on one B200: none (0), auto (-1) and compact (-2, every
referenced non-hot column in the dense x_warm, gathered by the plain TIER-1 tile kernel).
usage: python tools/compact_ab.py CFG [pairs]   -- prints one JSON line per measurement."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
import lbgen
import paper_2212_08964_b200 as lb

cfg = sys.argv[1]
pairs = int(sys.argv[2]) if len(sys.argv) > 2 else 3
modes = [int(m) for m in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0, -2]
A = lbgen.make_config(cfg, "float", device="cuda")
x = lbgen.x_for_config(cfg, A.cols, "float", device="cuda")
M = lb.CsrMatrix.from_csr(A)
y = torch.empty(A.rows, device="cuda")
ref = None


def timeit(n=50):
    for _ in range(5):
        M.spmv(x, y, "merge_path", repartition=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n):
        M.spmv(x, y, "merge_path", repartition=True)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for p in range(pairs):
    for mode in modes:
        M.plan_hot_x(16384, mode)
        info = M.plan_info()
        ms = timeit()
        ph = [sum(v) / 10 for v in zip(*[M.phase_times(x, y) for _ in range(10)])]
        pr = M.probe_stream_gather(x, 10)
        M.spmv(x, y, "merge_path", repartition=True)
        torch.cuda.synchronize()
        if ref is None:
            ref = y.clone()
        print(json.dumps({"config": cfg, "warm_mode": mode, "warm_cols": info["warm_cols"],
                          "kernel": M.kernel_name("merge_path"), "ms_step": round(ms, 4),
                          "GNZ/s": round(A.nnz / ms / 1e6, 1), "phase_ms": [round(v, 4) for v in ph],
                          "probe_GNZ/s": round(A.nnz / pr / 1e6, 1), "bitwise_equal_first": bool(torch.equal(y, ref))}),
              flush=True)
