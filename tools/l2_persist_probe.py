"""Experiment: pin x in a persisting L2 window (cudaStreamAttributeAccessPolicyWindow) while the C3 step
streams col/val -- does the DRAM re-fetch of x go away, and does the step get faster (less DRAM traffic,
less power)?  Prints ms per step with and without the window, and the device's persisting-L2 limits."""
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from cuda.bindings import runtime as rt
import lbgen
import paper_2212_08964_b200 as lb

A = lbgen.make_config("c3", "float", device="cuda")
x = lbgen.x_for_config("c3", A.cols, "float", device="cuda")
M = lb.CsrMatrix.from_csr(A)
M.plan_hot_x(0, -1)
y = torch.empty(A.rows, device="cuda")
err, maxp = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, 0)
err, maxw = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxAccessPolicyWindowSize, 0)
print(json.dumps({"max_persisting_l2": maxp, "max_window": maxw}), flush=True)
s = torch.cuda.current_stream()


def timeit(n=300):
    for _ in range(10):
        M.spmv(x, y, "merge_path", repartition=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n):
        M.spmv(x, y, "merge_path", repartition=True)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


mode = sys.argv[1] if len(sys.argv) > 1 else "both"
if mode in ("off", "both"):
    print(json.dumps({"window": None, "ms": round(timeit(), 4)}), flush=True)
if mode in ("on", "both"):
    rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize, maxp)
    for nbytes, ratio in ((min(maxw, 4 * A.cols), 1.0), (min(maxw, 4 * A.cols), 0.6)):
        attr = rt.cudaStreamAttrValue()
        attr.accessPolicyWindow.base_ptr = x.data_ptr()
        attr.accessPolicyWindow.num_bytes = nbytes
        attr.accessPolicyWindow.hitRatio = ratio
        attr.accessPolicyWindow.hitProp = rt.cudaAccessProperty.cudaAccessPropertyPersisting
        attr.accessPolicyWindow.missProp = rt.cudaAccessProperty.cudaAccessPropertyStreaming
        e = rt.cudaStreamSetAttribute(s.cuda_stream, rt.cudaStreamAttrID.cudaLaunchAttributeAccessPolicyWindow, attr)
        print(json.dumps({"window_bytes": nbytes, "hit_ratio": ratio, "set": str(e[0]), "ms": round(timeit(), 4)}), flush=True)
