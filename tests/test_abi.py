"""C-ABI checks that need no GPU: the library builds/loads, exports every symbol include/lb.h
declares, and its host-only entry point (lb_shard_bounds) matches the oracle."""
import ctypes
import subprocess

import numpy as np
import pytest
import torch

import lbgen
import oracle
import paper_2212_08964_b200 as lb
from paper_2212_08964_b200 import build


def test_library_builds_and_loads():
    path = build.build()
    assert path.endswith("liblb.so")
    L = lb.lib()
    assert lb.version().startswith("liblb")
    assert isinstance(lb.launch_count(), int)


def test_exports_every_declared_symbol():
    names = lb.declared_functions()
    assert len(names) >= 19
    for required in ("lb_csr_create", "lb_partition", "lb_spmv", "lb_spmv_multi", "lb_shard_bounds"):
        assert required in names
    out = subprocess.run(["nm", "-D", "--defined-only", lb.LIB_PATH], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    missing = [n for n in names if n not in exported]
    assert not missing, missing


def test_kernels_are_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", lb.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_shard_bounds_matches_oracle(G):
    for A in (lbgen.rmat(12, 8, 1, "ones"), lbgen.skewed(1 << 11, 3, 4000, 9000, 2, "ones"),
              lbgen.stencil(40, 2, "stencil"), lbgen.make_config("c1", "ones")):
        assert lb.shard_bounds(A.row_offsets, G).tolist() == oracle.shard_bounds(A.row_offsets, G).tolist()


def test_shard_bounds_rejects_bad_args():
    with pytest.raises(lb.LbError):
        lb.shard_bounds(np.array([0, 1], np.int32), 0)


def test_shard_csr_rebases_offsets():
    A = lbgen.rmat(9, 8, 2, "int")
    b = lb.shard_bounds(A.row_offsets, 3)
    parts = [lb.shard_csr(A.row_offsets, A.col_idx, A.values, b, r) for r in range(3)]
    assert sum(p[0].numel() - 1 for p in parts) == A.rows
    assert torch.equal(torch.cat([p[1] for p in parts]), A.col_idx)
    for off, col, _ in parts:
        assert int(off[0]) == 0 and int(off[-1]) == col.numel()


def test_compute_without_gpu_fails_loudly():
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    L = lb.lib()
    h = ctypes.c_void_p()
    st = L.lb_csr_create(1, 1, 0, ctypes.c_void_p(16), None, None, 0, None, ctypes.byref(h))
    assert st == lb.lb.LB_ERR_CUDA
    assert lb.last_error()


def test_shape_limits_checked_before_any_access():
    """Size errors come back as LB_ERR_INVALID_ARG before the library touches the arrays or the device:
    rows + nnz above 2^31 - 2^16 - 1 (lbgen.MAX_MERGE_ITEMS), cols >= 2^31 - 1, negative sizes."""
    L = lb.lib()
    fake = ctypes.c_void_p(256)  # never dereferenced
    cases = [(lbgen.MAX_MERGE_ITEMS - (1 << 30) + 1, 1 << 20, 1 << 30), (1, (1 << 31) - 1, 1), (-1, 1, 0), (1, 1, -2)]
    for rows, cols, nnz in cases:
        h = ctypes.c_void_p()
        st = L.lb_csr_create(rows, cols, nnz, fake, fake, fake, 0, None, ctypes.byref(h))
        assert st == lb.lb.LB_ERR_INVALID_ARG and not h, (rows, cols, nnz)
        assert "2^31" in lb.last_error() or "negative" in lb.last_error()
