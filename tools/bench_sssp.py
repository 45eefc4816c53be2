"""SSSP (NEXT-4) on R-MAT graphs (C3 structure at scale 24, weights |value|): time per solve (CUDA events
around lb_sssp, which syncs once per round), rounds, and edges/s = nnz / time (every edge of the
reachable part is relaxed at least once).  One JSON line per (scale, schedule)."""
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import lbgen
import paper_2212_08964_b200 as lb

SCALES = [int(s) for s in sys.argv[1].split(",")] if len(sys.argv) > 1 else [20, 22, 24]
SCHEDS = sys.argv[2].split(",") if len(sys.argv) > 2 else ["merge_path", "group_mapped", "thread_mapped"]
for sc in SCALES:
    A = lbgen.make_config("c3", "float", device="cuda") if sc == 24 else lbgen.rmat(sc, 16, 3, "float", device="cuda")
    w = A.values.abs()
    M = lb.CsrMatrix(A.rows, A.cols, A.row_offsets, A.col_idx, w)
    src = int(torch.argmax(A.row_offsets[1:] - A.row_offsets[:-1]).item())
    for sched in SCHEDS:
        d, rounds = M.sssp(src, sched)  # warm-up (workspace allocation)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            d, rounds = M.sssp(src, sched)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        t = sorted(ts)[1]
        reach = int(torch.isfinite(d).sum())
        print(json.dumps({"scale": sc, "schedule": sched, "vertices": A.rows, "edges": A.nnz, "reached": reach,
                          "rounds": rounds, "ms": round(t * 1e3, 2), "G_edges_per_s": round(A.nnz / t / 1e9, 2)}),
              flush=True)
    del M, A, w
    torch.cuda.empty_cache()
