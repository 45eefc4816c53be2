cat > /tmp/r4088.py <<'PY'
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch, lbgen
import paper_2212_08964_b200 as lb
from bench import graph_median
A = lbgen.make_config("c2", "float", device="cuda"); x = lbgen.x_for_config("c2", A.cols, "float", device="cuda")
M = lb.CsrMatrix.from_csr(A); y = torch.empty(A.rows, device="cuda")
for L in (2040, 4088):
    M.set_items_per_tile(L)
    med, lo, hi = graph_median(lambda: M.spmv(x, y, "merge_path", repartition=True), 50)
    print(json.dumps({"L": L, "v": os.environ.get("LB_ROWS4088", "0"), "kernel": M.kernel_name("merge_path"), "GNZ/s": round(A.nnz / med / 1e6, 1)}), flush=True)
PY
LB_ROWS4088=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "tile_lengths or every_tile or full_size or edge" > gpurun_out/r02aa_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02aa_tests.log
for v in 0 1 0 1; do LB_ROWS4088=$v timeout 300 python /tmp/r4088.py; done 2>&1 | tee gpurun_out/r02aa_r4088.txt
