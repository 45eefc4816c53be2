"""Dev sweep: correctness + C3 throughput of every pipelined tile-kernel variant (LB_PIPE_VARIANT)."""
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import lbgen, oracle
import paper_2212_08964_b200 as lb

VARIANTS = [(0, 1016), (13, 1016), (10, 1016), (3, 504), (11, 2040)]
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
# correctness on a small int matrix
As = lbgen.rmat(13, 16, 5, "int"); xs = lbgen.make_x(As.cols, "int", 3)
yref, _ = oracle.spmv(As.row_offsets, As.col_idx, As.values, xs)
Ms = lb.CsrMatrix.from_csr(As)
A = lbgen.make_config(cfg, "float", device="cuda")
x = lbgen.x_for_config(cfg, A.cols, "float", device="cuda")
M = lb.CsrMatrix.from_csr(A)
y = torch.empty(A.rows, device="cuda")
for v, L in VARIANTS:
    os.environ["LB_PIPE_VARIANT"] = str(v)
    Ms.set_items_per_tile(L)
    ok = np.array_equal(Ms.spmv(xs.cuda(), repartition=True).double().cpu().numpy(), yref)
    M.set_items_per_tile(L)
    for _ in range(5):
        M.spmv(x, y, repartition=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    n = 100
    e0.record()
    for _ in range(n):
        M.spmv(x, y, repartition=True)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    ph = np.mean([M.phase_times(x, y) for _ in range(10)], axis=0)
    print(json.dumps({"variant": v, "L": L, "ok": bool(ok), "ms": round(ms, 4), "GNZ/s": round(A.nnz / ms / 1e6, 1),
                      "main_ms": round(float(ph[1]), 4), "part_ms": round(float(ph[0]), 4)}), flush=True)
