import json, sys, os
sys.path.insert(0, os.getcwd())
import torch, lbgen, paper_2212_08964_b200 as lb
for cfg in sys.argv[1].split(","):
    A = lbgen.make_config(cfg, "float", device="cuda"); x = lbgen.x_for_config(cfg, A.cols, "float", device="cuda")
    M = lb.CsrMatrix.from_csr(A); y = torch.empty(A.rows, device="cuda")
    for sched in sys.argv[2].split(","):
        for _ in range(3): M.spmv(x, y, sched)
        torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True); e0.record()
        n = max(10, int(4e9 / A.nnz))
        for _ in range(n): M.spmv(x, y, sched)
        e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1) / n
        print(cfg, sched, round(A.nnz / ms / 1e6, 1), flush=True)
    del M, A, x, y; torch.cuda.empty_cache()
