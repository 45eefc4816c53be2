"""Small workload that touches every kernel of liblb.so once, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck).  Prints "sanitize driver ok" at the end.
usage: compute-sanitizer --tool memcheck python tools/sanitize_driver.py"""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import lbgen
import paper_2212_08964_b200 as lb

SCHEDS = ["merge_path", "thread_mapped", "group_mapped", "block_mapped", "warp_mapped", "binning",
          "nonzero_split", "auto"]
mats = {
    "rmat10": lbgen.rmat(10, 16, 3, "float"),
    "stencil40": lbgen.stencil(40, 2, "float"),
    "skewed": lbgen.skewed(1 << 10, 2, 3000, 5000, 4, "float"),
    "c1": lbgen.make_config("c1", "float"),
}
for name, A in mats.items():
    x = lbgen.make_x(A.cols, "float", 1).cuda()
    M = lb.CsrMatrix.from_csr(A)
    y = torch.empty(A.rows, device="cuda")
    for L in (504, 1016, 2040):
        M.set_items_per_tile(L)
        M.partition()
        M.spmv(x, y, "merge_path", repartition=True)
    M.set_items_per_tile(0)
    for s in SCHEDS:
        M.spmv(x, y, s, repartition=True)
    M.partition_nz(1016)
    M.bins()
    M.plan_hot_x(64, 200)  # hot + warm tiers
    M.spmv(x, y, "merge_path", repartition=True)
    M.plan_hot_x(-1)
    M.set_items_per_tile(1016)
    M.spmv_peers(x, y, [torch.empty(A.rows, device="cuda") for _ in range(2)], repartition=True)
    M.set_items_per_tile(0)
    for n in (1, 4, 8, 16, 32):
        X = torch.randn(A.cols, n, device="cuda")
        M.spmm(X)
    if A.rows == A.cols:
        W = lb.CsrMatrix(A.rows, A.cols, A.row_offsets.cuda(), A.col_idx.cuda(), A.values.abs().cuda())
        for s in ("merge_path", "group_mapped", "thread_mapped"):
            W.sssp(0, s)
    torch.cuda.synchronize()
    print(name, "ok", flush=True)
os.environ["LB_SPMM"] = "lanes"
A = mats["rmat10"]
lb.CsrMatrix.from_csr(A).spmm(torch.randn(A.cols, 16, device="cuda"))
os.environ.pop("LB_SPMM")
torch.cuda.synchronize()
print("sanitize driver ok")
