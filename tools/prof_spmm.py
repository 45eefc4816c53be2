"""ncu driver: SpMM Y = A X (X dense cols x n, row-major) `reps` times.  usage: python tools/prof_spmm.py CFG N REPS"""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import lbgen
import paper_2212_08964_b200 as lb

cfg, n, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
A = lbgen.make_config(cfg, "float", device="cuda")
M = lb.CsrMatrix.from_csr(A)
X = torch.randn(A.cols, n, device="cuda")
Y = torch.empty(A.rows, n, device="cuda")
for _ in range(reps):
    M.spmm(X, Y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(10):
    M.spmm(X, Y)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"{cfg} n={n}: {ms:.3f} ms, {A.nnz * n / ms / 1e6:.1f} G nnz-cols/s")
