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


# ---------------------------------------------------------------- host logic, property-based (no GPU)
from hypothesis import given, settings, strategies as st  # noqa: E402


@st.composite
def _offsets(draw):
    """Row offsets of a CSR with 0..300 rows of lengths 0..60 (many empty rows allowed)."""
    lens = draw(st.lists(st.one_of(st.just(0), st.integers(0, 60)), min_size=0, max_size=300))
    off = np.zeros(len(lens) + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    return off.astype(np.int32)


@settings(max_examples=150, deadline=None)
@given(_offsets(), st.integers(1, 12))
def test_shard_bounds_property(off, G):
    """lb_shard_bounds equals the oracle's linear scan (b_g = min{r : off[r] >= ceil(g nnz / G)}) for any
    offsets and rank count, including G > rows and nnz = 0; bounds are monotone from 0 to rows."""
    got = lb.shard_bounds(off, G)
    assert got.tolist() == oracle.shard_bounds(off, G).tolist()
    assert got[0] == 0 and got[-1] == off.size - 1 and np.all(np.diff(got) >= 0)


@settings(max_examples=150, deadline=None)
@given(_offsets(), st.integers(1, 8), st.integers(1, 8), st.randoms(use_true_random=False))
def test_exchange_schedule_property(off, G, K, rnd):
    """lb_exchange_schedule over random bounds and random cut tables: the (chunk, root) broadcast ranges
    tile [0, rows) exactly once, each inside its root's shard, in cut order; lb_padded_rows is the
    largest shard."""
    b = lb.shard_bounds(off, G)
    rows = off.size - 1
    cuts = np.zeros((G, K + 1), np.int64)
    for k in range(G):
        n = int(b[k + 1] - b[k])
        inner = sorted(rnd.randint(0, n) for _ in range(K - 1))
        cuts[k] = [0, *inner, n]
    o, c = lb.exchange_schedule(b, cuts)
    cover = np.zeros(rows, np.int64)
    for ch in range(K):
        for k in range(G):
            s0, n = int(o[ch, k]), int(c[ch, k])
            assert b[k] <= s0 and s0 + n <= b[k + 1]
            assert s0 == b[k] + cuts[k, ch] and n == cuts[k, ch + 1] - cuts[k, ch]
            cover[s0:s0 + n] += 1
    assert np.all(cover == 1)
    assert lb.padded_rows(b) == int(np.max(np.diff(b))) if G > 0 else 0
