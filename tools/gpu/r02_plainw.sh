cat > /tmp/plainw.py <<'PY'
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch, lbgen
import paper_2212_08964_b200 as lb
from bench import graph_median
for cfg in ("c3", "c4", "c5"):
    A = lbgen.make_config(cfg, "float", device="cuda"); x = lbgen.x_for_config(cfg, A.cols, "float", device="cuda")
    M = lb.CsrMatrix.from_csr(A); y = torch.empty(A.rows, device="cuda"); M.set_items_per_tile(1016)
    med, lo, hi = graph_median(lambda: M.spmv(x, y, "merge_path", repartition=True), 20)
    print(json.dumps({"cfg": cfg, "W": os.environ.get("LB_PLAIN_W", "8"), "GNZ/s": round(A.nnz / med / 1e6, 1)}), flush=True)
    del M, A, x, y; torch.cuda.empty_cache()
PY
for w in 0 16 12 0 16 12; do LB_PLAIN_W=$w timeout 600 python /tmp/plainw.py; done 2>&1 | tee gpurun_out/r02w_plainw.txt
