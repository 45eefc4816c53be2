"""DSMEM hot-tier experiment: stream+gather probe on C3 with the hot columns staged in
one SM (tier-1 probe) or spread over a cluster of C SMs (LB_PROBE_CLUSTER = C), for several slot
budgets.  GNZ/s of the probe (median of 3 x 20 passes)."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import lbgen
import paper_2212_08964_b200 as lb

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
A = lbgen.make_config(cfg, "float", device="cuda")
x = lbgen.x_for_config(cfg, A.cols, "float", device="cuda")
M = lb.CsrMatrix.from_csr(A)
M.set_items_per_tile(1016)
cases = [(0, 16384), (1, 16384), (2, 16384), (2, 32768), (4, 16384), (4, 32768), (4, 45056), (8, 45056),
         (0, 8192), (0, 24576), (0, 32768), (0, 45056)]
for C, slots in cases:
    n, hn = M.plan_hot_x(slots, 0)
    if C:
        os.environ["LB_PROBE_CLUSTER"] = str(C)
    else:
        os.environ.pop("LB_PROBE_CLUSTER", None)
    try:
        ms = float(np.median([M.probe_stream_gather(x, reps=20) for _ in range(3)]))
        r = {"C": C, "slots": n, "hot_frac": round(hn / A.nnz, 4), "ms": round(ms, 4), "GNZ/s": round(A.nnz / ms / 1e6, 1)}
    except Exception as e:
        r = {"C": C, "slots": slots, "error": str(e)[:200]}
    print(json.dumps(r), flush=True)
os.environ.pop("LB_PROBE_CLUSTER", None)
