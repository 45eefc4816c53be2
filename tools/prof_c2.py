"""One C2 merge-path step (L = 2040) for ncu: partition + the short-row tile kernel."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import lbgen
import paper_2212_08964_b200 as lb
A = lbgen.make_config("c2", "float", device="cuda")
x = lbgen.x_for_config("c2", A.cols, "float", device="cuda")
M = lb.CsrMatrix.from_csr(A)
M.set_items_per_tile(2040)
y = torch.empty(A.rows, device="cuda")
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    M.spmv(x, y, "merge_path", repartition=True)
torch.cuda.synchronize()
