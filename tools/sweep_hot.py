"""Sweep of the hot-column plan on one B200: slot budget x warps per CTA x tile length, per config.
Prints one JSON line per point (GNZ/s of lb_spmv_ex(REPARTITION) and of the cached-partition call)."""
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import lbgen
import paper_2212_08964_b200 as lb

CFGS = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c3"]
SLOTS = [int(s) for s in sys.argv[2].split(",")] if len(sys.argv) > 2 else [8192, 16384, 24576, 32768, 40960, 45056]
WS = sys.argv[3].split(",") if len(sys.argv) > 3 else ["8", "16", "20"]
LS = [int(s) for s in sys.argv[4].split(",")] if len(sys.argv) > 4 else [1016, 504]
WARMS = [int(s) for s in sys.argv[5].split(",")] if len(sys.argv) > 5 else [0]


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
    n = 10 if A.nnz > 5e8 else 30
    for L in LS:
        M.set_items_per_tile(L)
        M.plan_hot_x(-1)
        ms0 = timeit(lambda: M.spmv(x, y, "merge_path", repartition=True), n)
        print(json.dumps({"config": cfg, "L": L, "plan": None, "kernel": M.kernel_name(), "ms_step": round(ms0, 4),
                          "GNZ/s": round(A.nnz / ms0 / 1e6, 1)}), flush=True)
        for slots in SLOTS:
          for warm in WARMS:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            hn, hnnz = M.plan_hot_x(slots, warm)
            torch.cuda.synchronize()
            tplan = time.perf_counter() - t0
            info = M.plan_info()
            for W in WS:
                os.environ["LB_HOT_W"] = W
                ms = timeit(lambda: M.spmv(x, y, "merge_path", repartition=True), n)
                msc = timeit(lambda: M.spmv(x, y, "merge_path"), n)
                print(json.dumps({"config": cfg, "L": L, "slots": slots, "warm_req": warm, "W": int(W), "hot_cols": hn,
                                  "hot_frac": round(hnnz / A.nnz, 4), "warm_cols": info["warm_cols"],
                                  "warm_frac": round(info["warm_nnz"] / A.nnz, 4), "plan_ms": round(tplan * 1e3, 1),
                                  "kernel": M.kernel_name(), "ms_step": round(ms, 4),
                                  "GNZ/s": round(A.nnz / ms / 1e6, 1), "GNZ/s_cached": round(A.nnz / msc / 1e6, 1)}),
                      flush=True)
        os.environ.pop("LB_HOT_W", None)
    del M, A, x, y
    torch.cuda.empty_cache()
