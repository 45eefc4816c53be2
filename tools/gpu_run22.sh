timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "spmm" > gpurun_out/pt22.log 2>&1; echo "spmm tests rc=$?"; tail -3 gpurun_out/pt22.log
cat > /tmp/spmm_t.py <<'PY'
import json, sys, os
sys.path.insert(0, os.getcwd())
import torch, lbgen, paper_2212_08964_b200 as lb
for cfg in ("c2", "c3", "c4", "c5"):
    A = lbgen.make_config(cfg, "float", device="cuda"); M = lb.CsrMatrix.from_csr(A)
    for n in (4, 8, 16):
        X = lbgen.make_x(A.cols * n, "float", 5, device="cuda").reshape(A.cols, n); Y = torch.empty(A.rows, n, device="cuda")
        for _ in range(2): M.spmm(X, Y)
        torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True); e0.record()
        for _ in range(5): M.spmm(X, Y)
        e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1) / 5
        print(json.dumps({"config": cfg, "op": "spmm", "n": n, "ms": round(ms, 4), "Gnnz_cols_per_s": round(A.nnz * n / ms / 1e6, 1)}), flush=True)
        del X, Y
    del M, A; torch.cuda.empty_cache()
PY
timeout 600 python /tmp/spmm_t.py
