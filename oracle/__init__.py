"""CPU oracle for the SpMV hot path of arXiv 2212.08964 (ctypes wrapper over oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs are the only callers.  It shares no code with the CUDA product
(paper_2212_08964_b200/) and the product never imports it.

Every function follows the plain definition of what the method computes (see oracle.c
for the PAPER.md citations); pins live in tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (no fast-math, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                               "-shared", "-o", _LIB, _SRC])
    return _LIB


_lib = None
_timing = None


def timing_lib():
    """The same oracle.c built for TIMING on this host (bench.py's cpu_baseline / reference arm only):
    -O3 -march=native -fopenmp, still -ffp-contract=off and no fast-math (the summation order and
    rounding are the definition's).  Built fresh per process into a temporary directory, so a library
    compiled for another host's ISA is never loaded."""
    global _timing
    if _timing is None:
        import tempfile
        d = tempfile.mkdtemp(prefix="oracle_native_")
        out = os.path.join(d, "liboracle_native.so")
        subprocess.check_call(["gcc", "-O3", "-march=native", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-o", out, _SRC])
        L = ctypes.CDLL(out)
        i64, p = ctypes.c_int64, ctypes.c_void_p
        L.oracle_spmv.argtypes = [i64, p, p, p, p, p, p]
        L.oracle_spmv_omp.argtypes = [i64, p, p, p, p, p, p]
        L.oracle_partition.argtypes = [i64, i64, p, i64, p]
        L.oracle_partition.restype = i64
        L.oracle_num_threads.restype = ctypes.c_int
        _timing = L
    return _timing


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i64, p = ctypes.c_int64, ctypes.c_void_p
        L.oracle_spmv.argtypes = [i64, p, p, p, p, p, p]
        L.oracle_spmv_omp.argtypes = [i64, p, p, p, p, p, p]
        L.oracle_spmv_packed.argtypes = [i64, p, p, p, p, p, p]
        L.oracle_spmm.argtypes = [i64, p, p, p, i64, p, i64, p, i64, p]
        L.oracle_partition.argtypes = [i64, i64, p, i64, p]
        L.oracle_partition.restype = i64
        L.oracle_partition_nz.argtypes = [i64, i64, p, i64, p]
        L.oracle_partition_nz.restype = i64
        L.oracle_shard_bounds.argtypes = [i64, p, ctypes.c_int32, p]
        L.oracle_bins.argtypes = [i64, p, i64, i64, p, p]
        L.oracle_x_plan.argtypes = [i64, i64, p, ctypes.c_int32, i64, p, p, p, p, p, p, p, p]
        L.oracle_x_plan.restype = i64
        L.oracle_sssp.argtypes = [i64, p, p, p, i64, p, p]
        L.oracle_sssp.restype = i64
        L.oracle_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _np(a, dtype):
    """torch tensor / list / ndarray -> contiguous host ndarray of dtype."""
    if hasattr(a, "detach"):
        a = a.detach().cpu().numpy()
    a = np.ascontiguousarray(np.asarray(a), dtype=dtype)
    return a


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def spmv(row_offsets, col_idx, values, x, threads: bool = False, timing: bool = False):
    """y = A x in double, plus s_i = sum_k |a_ik x_k|.  Returns (y, s) as float64 arrays.
    timing: run the -O3 -march=native build (timing_lib; same arithmetic)."""
    off = _np(row_offsets, np.int32)
    col = _np(col_idx, np.int32)
    val = _np(values, np.float32)
    xx = _np(x, np.float32)
    rows = off.size - 1
    y = np.empty(rows, np.float64)
    s = np.empty(rows, np.float64)
    L = timing_lib() if timing else lib()
    f = L.oracle_spmv_omp if threads else L.oracle_spmv
    f(rows, _ptr(off), _ptr(col), _ptr(val), _ptr(xx), _ptr(y), _ptr(s))
    return y, s


def spmm(row_offsets, col_idx, values, X):
    """Y = A X in double (X: [cols, n] row-major), plus S = sum |a_ik X_kj|.  Returns (Y, S)."""
    off = _np(row_offsets, np.int32)
    col = _np(col_idx, np.int32)
    val = _np(values, np.float32)
    XX = _np(X, np.float32)
    rows = off.size - 1
    n = XX.shape[1] if XX.ndim == 2 else 1
    Y = np.empty((rows, n), np.float64)
    S = np.empty((rows, n), np.float64)
    lib().oracle_spmm(rows, _ptr(off), _ptr(col), _ptr(val), n, _ptr(XX), n, _ptr(Y), n, _ptr(S))
    return Y, S


def spmv_packed(sel_offsets, sel_cols, sel_vals, x):
    """Definition of y on a packed subset of rows (for sampled parity at full size)."""
    so = _np(sel_offsets, np.int64)
    sc = _np(sel_cols, np.int32)
    sv = _np(sel_vals, np.float32)
    xx = _np(x, np.float32)
    n = so.size - 1
    y = np.empty(n, np.float64)
    s = np.empty(n, np.float64)
    lib().oracle_spmv_packed(n, _ptr(so), _ptr(sc), _ptr(sv), _ptr(xx), _ptr(y), _ptr(s))
    return y, s


def partition(row_offsets, L: int, timing: bool = False) -> np.ndarray:
    """Brute-force merge-path tile coordinates: int32 array [T+1, 2] of (row, nz)."""
    off = _np(row_offsets, np.int32)
    rows = off.size - 1
    nnz = int(off[-1]) if rows > 0 else 0
    T = (rows + nnz + L - 1) // L
    out = np.empty((T + 1, 2), np.int32)
    got = (timing_lib() if timing else lib()).oracle_partition(rows, nnz, _ptr(off), L, _ptr(out))
    if got != T:
        raise ValueError("bad partition arguments")
    return out


def partition_nz(row_offsets, L: int) -> np.ndarray:
    """Nonzero-splitting tile coordinates (brute force): int32 [T+1, 2] of (row, nz)."""
    off = _np(row_offsets, np.int32)
    rows = off.size - 1
    nnz = int(off[-1]) if rows > 0 else 0
    T = max(1, (nnz + L - 1) // L)
    out = np.empty((T + 1, 2), np.int32)
    if lib().oracle_partition_nz(rows, nnz, _ptr(off), L, _ptr(out)) != T:
        raise ValueError("bad partition arguments")
    return out


def shard_bounds(row_offsets, G: int) -> np.ndarray:
    off = _np(row_offsets, np.int32)
    out = np.empty(G + 1, np.int64)
    lib().oracle_shard_bounds(off.size - 1, _ptr(off), G, _ptr(out))
    return out


def bins(row_offsets, block_size: int = 256, warp_size: int = 32):
    """Alg.4 three-bin classification (oracle_bins): (cta_rows, warp_rows, thread_rows), ascending int32."""
    off = _np(row_offsets, np.int32)
    rows = off.size - 1
    ids = np.zeros(max(rows, 1), np.int32)
    sizes = np.zeros(3, np.int64)
    lib().oracle_bins(rows, _ptr(off), block_size, warp_size, _ptr(ids), _ptr(sizes))
    n0, n1 = int(sizes[0]), int(sizes[1])
    return ids[:n0].copy(), ids[n0:n0 + n1].copy(), ids[n0 + n1:rows].copy()


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def x_plan(col_idx, cols: int, slots: int, warm: int = 0):
    """x-reuse plan by definition (oracle_x_plan): (hot slot -> column int32[n], warm index -> column
    int32[m], remapped col_idx int32[nnz], stored entries in hot columns, in warm columns)."""
    col = _np(col_idx, np.int32)
    nnz = col.size
    deg = np.zeros(max(cols, 1), np.int64)
    tier = np.zeros(max(cols, 1), np.int32)
    slot_cols = np.zeros(max(slots, 1), np.int32)
    warm_cols = np.zeros(max(cols, 1), np.int32)
    remapped = np.zeros(max(nnz, 1), np.int32)
    nw, hn, wn = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    n = lib().oracle_x_plan(cols, nnz, _ptr(col), slots, warm, _ptr(deg), _ptr(tier), _ptr(slot_cols),
                            _ptr(warm_cols), _ptr(remapped), ctypes.byref(nw), ctypes.byref(hn), ctypes.byref(wn))
    return (slot_cols[:n].copy(), warm_cols[:nw.value].copy(), remapped[:nnz].copy(), int(hn.value),
            int(wn.value))


def hot_columns(col_idx, cols: int, slots: int):
    """Hot tier only: (slot -> column, remapped col_idx, stored entries in hot columns)."""
    sc, _, rm, hn, _ = x_plan(col_idx, cols, slots, 0)
    return sc, rm, hn


def sssp(row_offsets, col_idx, weights, source: int) -> np.ndarray:
    """Dijkstra distances (fp32, +inf if unreachable) by oracle_sssp; ValueError on a negative weight."""
    off = _np(row_offsets, np.int32)
    col = _np(col_idx, np.int32)
    w = _np(weights, np.float32)
    n = off.size - 1
    dist = np.zeros(max(n, 1), np.float32)
    settled = np.zeros(max(n, 1), np.uint8)
    r = lib().oracle_sssp(n, _ptr(off), _ptr(col), _ptr(w), int(source), _ptr(dist), _ptr(settled))
    if r < 0:
        raise ValueError("negative edge weight")
    return dist[:n].copy()
