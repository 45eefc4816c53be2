"""SpMM rates on one B200: both tile processors (lanes over columns: default; lanes over nonzeros:
LB_SPMM=lanes) for n in N, per config.  usage: python tools/bench_spmm.py c3,c4 8,16,32"""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
import lbgen
import paper_2212_08964_b200 as lb

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c3"]
ns = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [8, 16, 32]
for cfg in cfgs:
    A = lbgen.make_config(cfg, "float", device="cuda")
    M = lb.CsrMatrix.from_csr(A)
    for n in ns:
        X = torch.randn(A.cols, n, device="cuda")
        Y = torch.empty(A.rows, n, device="cuda")
        for mode in ("cols", "lanes"):
            if mode == "lanes":
                os.environ["LB_SPMM"] = "lanes"
            else:
                os.environ.pop("LB_SPMM", None)
            for _ in range(2):
                M.spmm(X, Y)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            reps = 5
            e0.record()
            for _ in range(reps):
                M.spmm(X, Y)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            print(json.dumps({"config": cfg, "op": "spmm", "kernel": mode, "n": n, "ms": round(ms, 4),
                              "Gnnz_cols_per_s": round(A.nnz * n / ms / 1e6, 1)}), flush=True)
        del X, Y
        torch.cuda.empty_cache()
    os.environ.pop("LB_SPMM", None)
    del M, A
    torch.cuda.empty_cache()
