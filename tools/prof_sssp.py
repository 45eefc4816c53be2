"""ncu driver: one merge-path SSSP solve on C3 (weights |value|, source = max-degree vertex), after a warm-up."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch, lbgen, paper_2212_08964_b200 as lb
sched = sys.argv[1] if len(sys.argv) > 1 else "merge_path"
A = lbgen.make_config("c3", "float", device="cuda")
M = lb.CsrMatrix(A.rows, A.cols, A.row_offsets, A.col_idx, A.values.abs())
src = int(torch.argmax(A.row_offsets[1:] - A.row_offsets[:-1]).item())
d, r = M.sssp(src, sched)
torch.cuda.synchronize()
d, r = M.sssp(src, sched)
torch.cuda.synchronize()
print("rounds", r, "reached", int(torch.isfinite(d).sum()))
