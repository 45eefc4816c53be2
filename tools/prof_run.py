"""Driver for ncu captures: build config, optional hot-column plan, run merge-path SpMV `reps` times.
usage: python tools/prof_run.py CFG SLOTS(-1 = no plan) REPS [L]   (LB_HOT_W / LB_PIPE_VARIANT from env)"""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import lbgen
import paper_2212_08964_b200 as lb

cfg, slots, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
L = int(sys.argv[4]) if len(sys.argv) > 4 else 0
A = lbgen.make_config(cfg, "float", device="cuda")
x = lbgen.x_for_config(cfg, A.cols, "float", device="cuda")
M = lb.CsrMatrix.from_csr(A)
if L:
    M.set_items_per_tile(L)
if slots >= 0:
    print("plan", M.plan_hot_x(slots))
y = torch.empty(A.rows, device="cuda")
for _ in range(reps):
    M.spmv(x, y, "merge_path", repartition=True)
torch.cuda.synchronize()
print("kernel", M.kernel_name())
