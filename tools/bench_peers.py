"""Cost of the fused multi-GPU epilogue on one GPU: merge-path step (plan as bench.py) with 0, 1, 3 and 7
peer buffers on the same GPU (lb_spmv_peers).  On a node the peer stores leave over NVLink instead of
landing in local HBM, so this bounds the kernel-side overhead (instructions + store issue)."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
import lbgen
import paper_2212_08964_b200 as lb

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
A = lbgen.make_config(cfg, "float", device="cuda")
x = lbgen.x_for_config(cfg, A.cols, "float", device="cuda")
M = lb.CsrMatrix.from_csr(A)
M.plan_hot_x(0, -1)
y = torch.empty(A.rows, device="cuda")
bufs = [torch.empty(A.rows, device="cuda") for _ in range(7)]
for npeers in (0, 1, 3, 7):
    f = (lambda: M.spmv(x, y, "merge_path", repartition=True)) if npeers == 0 else \
        (lambda: M.spmv_peers(x, y, bufs[:npeers], repartition=True))
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(json.dumps({"config": cfg, "peers_on_same_gpu": npeers, "ms": round(ms, 4),
                      "GNZ/s": round(A.nnz / ms / 1e6, 1), "extra_y_bytes": 4 * A.rows * npeers}), flush=True)
