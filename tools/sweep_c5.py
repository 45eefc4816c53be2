"""C5 (x = 256 MB > L2): hot slots x warm-tier budget sweep of the merge-path step (graph-replayed median
of 20), to re-check the plan's defaults with the round-2 kernels."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
import lbgen
import paper_2212_08964_b200 as lb
from bench import graph_median

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
A = lbgen.make_config(cfg, "float", device="cuda")
x = lbgen.x_for_config(cfg, A.cols, "float", device="cuda")
M = lb.CsrMatrix.from_csr(A)
y = torch.empty(A.rows, device="cuda")
for slots in (4096, 8192, 16384):
    for warm_mb in (32, 48, 64):
        n, hn = M.plan_hot_x(slots, warm_mb * (1 << 20) // 4)
        info = M.plan_info()
        med, lo, hi = graph_median(lambda: M.spmv(x, y, "merge_path", repartition=True), 20)
        print(json.dumps({"config": cfg, "slots": n, "hot_frac": round(hn / A.nnz, 4), "warm_MB": warm_mb,
                          "warm_frac": round(info["warm_nnz"] / A.nnz, 4), "ms": round(med, 4),
                          "GNZ/s": round(A.nnz / med / 1e6, 1), "kernel": M.kernel_name()}), flush=True)
