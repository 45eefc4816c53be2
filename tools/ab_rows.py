"""Short-row tile kernel at L = 2040 vs thread-mapped: median of 50 CUDA-graph replays of
lb_spmv_ex(REPARTITION) per config, with per-phase times.  Round 2 ran it once per candidate kernel
(selected by diagnostic environment switches that were removed with the losing candidates; the
results are in profiles/r02_ab_short_rows_*.jsonl)."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import lbgen
import paper_2212_08964_b200 as lb
from bench import graph_median

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c2"]
for cfg in cfgs:
    A = lbgen.make_config(cfg, "float", device="cuda")
    x = lbgen.x_for_config(cfg, A.cols, "float", device="cuda")
    M = lb.CsrMatrix.from_csr(A)
    y = torch.empty(A.rows, device="cuda")
    M.set_items_per_tile(2040)
    out = {"config": cfg, "kernel": M.kernel_name("merge_path")}
    for sched in ("merge_path", "thread_mapped"):
        med, lo, hi = graph_median(lambda: M.spmv(x, y, sched, repartition=True), 50)
        ph = np.mean(np.array([M.phase_times(x, y, sched) for _ in range(20)]), axis=0)
        out[sched] = {"ms": round(med, 5), "GNZ/s": round(A.nnz / med / 1e6, 1),
                      "phases_ms": [round(float(v), 5) for v in ph]}
    print(json.dumps(out), flush=True)
    del M, A, x, y
    torch.cuda.empty_cache()
