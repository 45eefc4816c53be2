"""Landscape: every BASELINE config x every schedule on one B200 (GNZ/s, algorithmic GB/s).
Prints one JSON line per (config, schedule); used for profiles/ and DESIGN.md section 9."""
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import lbgen
import paper_2212_08964_b200 as lb

CFGS = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c1", "c2", "c3", "c4", "c5"]
SCHEDS = ["merge_path", "nonzero_split", "thread_mapped", "group_mapped", "block_mapped", "warp_mapped", "binning", "auto"]


def timeit(fn, n):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for cfg in CFGS:
    A = lbgen.make_config(cfg, "float", device="cuda")
    x = lbgen.x_for_config(cfg, A.cols, "float", device="cuda")
    M = lb.CsrMatrix.from_csr(A)
    y = torch.empty(A.rows, device="cuda")
    alg = 8 * A.nnz + 4 * (A.rows + 1) + 4 * A.rows + 4 * A.cols
    for sched in SCHEDS + ["merge_path+plan"]:
        plan = None
        if sched == "merge_path+plan":
            sched = "merge_path"
            M.set_items_per_tile(1016)
            M.plan_hot_x(0, -1)
            plan = M.plan_info()
        n = 20 if sched in ("merge_path",) else 5
        if cfg == "c1":
            n = 200
        ms_step = timeit(lambda: M.spmv(x, y, sched, repartition=True), n)
        ms_cached = timeit(lambda: M.spmv(x, y, sched), n)
        # the same step captured once in a CUDA graph and replayed (no per-call host launch cost)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            M.spmv(x, y, sched, repartition=True)
        ms_graph = timeit(g.replay, n)
        del g
        print(json.dumps({"config": cfg, "rows": A.rows, "nnz": A.nnz, "schedule": sched, "plan": plan,
                          "kernel": M.kernel_name(sched), "L": M.items_per_tile if sched == "merge_path" else None,
                          "ms_step": round(ms_step, 4), "GNZ/s_step": round(A.nnz / ms_step / 1e6, 2),
                          "ms_cached_partition": round(ms_cached, 4),
                          "GNZ/s_cached": round(A.nnz / ms_cached / 1e6, 2),
                          "ms_graph": round(ms_graph, 4), "GNZ/s_graph": round(A.nnz / ms_graph / 1e6, 2),
                          "alg_GB/s_cached": round(alg / ms_cached / 1e6, 1)}), flush=True)
    del M, A, x, y
    torch.cuda.empty_cache()

# SpMM panels (n = 4, 8, 16) on the same merge-path tiles
for cfg in CFGS:
    if cfg == "c1":
        continue
    A = lbgen.make_config(cfg, "float", device="cuda")
    M = lb.CsrMatrix.from_csr(A)
    for n in (4, 8, 16):
        X = lbgen.make_x(A.cols * n, "float", 5, device="cuda").reshape(A.cols, n)
        Y = torch.empty(A.rows, n, device="cuda")
        ms = timeit(lambda: M.spmm(X, Y), 10)
        alg = (n + 3) // 4 * 8 * A.nnz + 4 * (A.rows + 1) + 4 * n * (A.rows + A.cols)
        print(json.dumps({"config": cfg, "op": "spmm", "n": n, "ms": round(ms, 4),
                          "Gnnz_cols_per_s": round(A.nnz * n / ms / 1e6, 1),
                          "alg_GB/s": round(alg / ms / 1e6, 1)}), flush=True)
        del X, Y
    del M, A
    torch.cuda.empty_cache()
