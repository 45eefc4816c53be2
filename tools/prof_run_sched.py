"""ncu driver: run one schedule `reps` times on a config.  usage: python tools/prof_run_sched.py CFG SCHED REPS"""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import lbgen
import paper_2212_08964_b200 as lb

cfg, sched, reps = sys.argv[1], sys.argv[2], int(sys.argv[3])
A = lbgen.make_config(cfg, "float", device="cuda")
x = lbgen.x_for_config(cfg, A.cols, "float", device="cuda")
M = lb.CsrMatrix.from_csr(A)
y = torch.empty(A.rows, device="cuda")
for _ in range(reps):
    M.spmv(x, y, sched, repartition=True)
torch.cuda.synchronize()
print("kernel", M.kernel_name(sched))
