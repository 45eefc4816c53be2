"""Thin ctypes binding over liblb.so (include/lb.h).  Argument marshalling only: every step of
the SpMV path runs in the library's CUDA kernels; there is no Python or CPU fallback, and a
missing/unloadable library raises immediately.

PyTorch is used for device memory and streams only.
"""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_PKG)
LIB_PATH = os.environ.get("LB_LIB_PATH") or os.path.join(_PKG, "liblb.so")
HEADER = os.path.join(_ROOT, "include", "lb.h")

LB_OK, LB_ERR_INVALID_ARG, LB_ERR_INVALID_CSR, LB_ERR_UNSUPPORTED, LB_ERR_OOM, LB_ERR_CUDA, LB_ERR_NCCL = range(7)
SCHEDULES = {"thread_mapped": 0, "group_mapped": 1, "merge_path": 2, "block_mapped": 3, "auto": 4,
             "nonzero_split": 5, "warp_mapped": 6, "binning": 7}
SCHEDULE_NAMES = {v: k for k, v in SCHEDULES.items()}
LB_SPMV_REPARTITION = 1
LB_SPMV_CHUNKED = 2
LB_SPMV_PADDED = 4
CHUNKS_MAX = 8
DEFAULT_ITEMS_PER_TILE = 1016
TILE_LENGTHS = (504, 1016, 2040, 3064, 4088)


class LbError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"liblb status {status}: {msg}")
        self.status = status


class InvalidCsr(LbError, ValueError):
    pass


_lib = None


def declared_functions() -> list[str]:
    """Names of every function include/lb.h declares."""
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(lb_[a-z_0-9]+)\s*\(", src, flags=re.M)))


def lib() -> ctypes.CDLL:
    """Load liblb.so (fails loudly if it is missing; build it with paper_2212_08964_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2212_08964_b200.build` "
                           "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    i32, i64, u32, p, sz = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_size_t
    st = ctypes.c_int
    sig = {
        "lb_csr_create": ([i64, i64, i64, p, p, p, i32, p, ctypes.POINTER(p)], st),
        "lb_csr_destroy": ([p], st),
        "lb_csr_set_items_per_tile": ([p, i32], st),
        "lb_partition_size": ([p, i32, ctypes.POINTER(i64)], st),
        "lb_partition": ([p, i32, p, p], st),
        "lb_partition_nz": ([p, i32, p, p], st),
        "lb_spmv": ([p, ctypes.c_int, p, p, p], st),
        "lb_spmv_ex": ([p, ctypes.c_int, p, p, u32, p], st),
        "lb_spmm": ([p, i64, p, i64, p, i64, p], st),
        "lb_csr_plan_hot_x": ([p, i32, i64, p, ctypes.POINTER(i32), ctypes.POINTER(i64)], st),
        "lb_csr_hot_plan": ([p, ctypes.POINTER(i32), ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64),
                             p, p, p, p], st),
        "lb_sssp": ([p, i64, ctypes.c_int, p, p, ctypes.POINTER(i32)], st),
        "lb_bins": ([p, p, ctypes.POINTER(i64), p], st),
        "lb_spmv_host_workspace_size": ([i64, i64, i64], sz),
        "lb_spmv_host": ([i64, i64, i64, p, p, p, p, p, ctypes.c_int, p, sz, p], st),
        "lb_spmv_phase_times": ([p, ctypes.c_int, p, p, p, ctypes.POINTER(ctypes.c_float)], st),
        "lb_probe_stream_gather": ([p, p, i32, p, ctypes.POINTER(ctypes.c_float)], st),
        "lb_probe_stream": ([p, i32, p, ctypes.POINTER(ctypes.c_float)], st),
        "lb_csr_trace_phases": ([p, i32], st),
        "lb_csr_trace_read": ([p, ctypes.POINTER(i32), ctypes.POINTER(ctypes.c_float)], st),
        "lb_spmv_host_x": ([p, i32, p, p, ctypes.c_uint32, p], st),
        "lb_spmv_host_x_async": ([p, i32, p, p, ctypes.c_uint32, p], st),
        "lb_spmv_host_x_wait": ([p], st),
        "lb_shard_bounds": ([p, i64, i32, p], st),
        "lb_comm_unique_id": ([p], st),
        "lb_comm_init": ([p, i32, i32, i32, ctypes.POINTER(p)], st),
        "lb_comm_destroy": ([p], st),
        "lb_spmv_multi": ([p, p, ctypes.c_int, p, p, p, p], st),
        "lb_spmv_multi_ex": ([p, p, ctypes.c_int, p, p, p, u32, p], st),
        "lb_allgather_rows": ([p, p, p, p], st),
        "lb_exchange_schedule": ([i32, p, i32, p, p, p], st),
        "lb_csr_chunk_rows": ([p, i32, p, p], st),
        "lb_padded_rows": ([i32, p], i64),
        "lb_remap_cols_padded": ([i32, p, p, i64, p, p], st),
        "lb_allgather_padded": ([p, i64, p, p], st),
        "lb_y_checksum": ([p, i64, p, ctypes.POINTER(ctypes.c_uint64)], st),
        "lb_comm_check_replicas": ([p, p, i64, p, ctypes.POINTER(i32), ctypes.POINTER(ctypes.c_uint64)], st),
        "lb_peer_create": ([p, p, i64, p, ctypes.POINTER(p)], st),
        "lb_peer_destroy": ([p], st),
        "lb_spmv_multi_fused": ([p, p, ctypes.c_int, p, p, u32, p], st),
        "lb_spmv_peers": ([p, p, p, p, i32, u32, p], st),
        "lb_kernel_name": ([p, ctypes.c_int], ctypes.c_char_p),
        "lb_select_schedule": ([p, p, ctypes.POINTER(ctypes.c_int)], st),
        "lb_last_error": ([], ctypes.c_char_p),
        "lb_launch_count": ([], ctypes.c_uint64),
        "lb_version": ([], ctypes.c_char_p),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _check(status: int):
    if status != LB_OK:
        msg = lib().lb_last_error().decode()
        if status == LB_ERR_INVALID_CSR:
            raise InvalidCsr(status, msg)
        raise LbError(status, msg)


def last_error() -> str:
    return lib().lb_last_error().decode()


def launch_count() -> int:
    return int(lib().lb_launch_count())


def version() -> str:
    return lib().lb_version().decode()


def _stream(stream) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _sched(schedule) -> int:
    if isinstance(schedule, int):
        return schedule
    try:
        return SCHEDULES[schedule]
    except KeyError:
        raise ValueError(f"unknown schedule {schedule!r}; one of {sorted(SCHEDULES)}") from None


def _dev_tensor(t: torch.Tensor, dtype, name: str, n: int | None = None) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or t.device.type != "cuda":
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if n is not None and t.numel() != n:
        raise ValueError(f"{name} has {t.numel()} elements, expected {n}")
    return t


class CsrMatrix:
    """A borrowed CSR matrix on the GPU (lb_csr_t).  Keeps references to its tensors so they
    outlive the handle (include/lb.h ownership rule)."""

    def __init__(self, rows: int, cols: int, row_offsets: torch.Tensor, col_idx: torch.Tensor,
                 values: torch.Tensor, validate: bool = True, stream=None):
        self.rows, self.cols = int(rows), int(cols)
        self.row_offsets = _dev_tensor(row_offsets, torch.int32, "row_offsets", self.rows + 1)
        self.col_idx = _dev_tensor(col_idx, torch.int32, "col_idx")
        self.values = _dev_tensor(values, torch.float32, "values", self.col_idx.numel())
        self.nnz = int(self.col_idx.numel())
        self._h = ctypes.c_void_p()
        with torch.cuda.device(self.row_offsets.device):
            _check(lib().lb_csr_create(self.rows, self.cols, self.nnz, self.row_offsets.data_ptr(),
                                       self.col_idx.data_ptr() if self.nnz else None,
                                       self.values.data_ptr() if self.nnz else None, int(bool(validate)),
                                       _stream(stream), ctypes.byref(self._h)))
        self.device = self.row_offsets.device
        self.items_per_tile = 2040 if self.nnz < 8 * self.rows else DEFAULT_ITEMS_PER_TILE
        self._host_refs = []  # host tensors of enqueued spmv_host_async calls (alive until spmv_host_wait)

    @classmethod
    def from_csr(cls, A, device="cuda", validate: bool = True) -> "CsrMatrix":
        """From any object with rows, cols, row_offsets, col_idx, values (e.g. lbgen.Csr)."""
        return cls(A.rows, A.cols, A.row_offsets.to(device), A.col_idx.to(device), A.values.to(device),
                   validate=validate)

    @property
    def handle(self) -> ctypes.c_void_p:
        if not self._h:
            raise ValueError("CsrMatrix is closed")
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            lib().lb_csr_destroy(self._h)  # synchronises the handle's copy streams first
            self._h = ctypes.c_void_p()
        self._host_refs = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_items_per_tile(self, L: int):
        _check(lib().lb_csr_set_items_per_tile(self.handle, int(L)))
        self.items_per_tile = int(L) or (2040 if self.nnz < 8 * self.rows else DEFAULT_ITEMS_PER_TILE)

    def num_tiles(self, items_per_tile: int = 0) -> int:
        n = ctypes.c_int64()
        _check(lib().lb_partition_size(self.handle, int(items_per_tile), ctypes.byref(n)))
        return int(n.value)

    def partition(self, items_per_tile: int = 0, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """Merge-path tile coordinates, int32 [T+1, 2] of (row, nz) (lb_partition)."""
        T = self.num_tiles(items_per_tile)
        if out is None:
            out = torch.empty((T + 1, 2), dtype=torch.int32, device=self.device)
        _dev_tensor(out, torch.int32, "out", 2 * (T + 1))
        _check(lib().lb_partition(self.handle, int(items_per_tile), out.data_ptr(), _stream(stream)))
        return out

    def partition_nz(self, items_per_tile: int = 1016, stream=None) -> torch.Tensor:
        """Nonzero-splitting tile coordinates, int32 [T+1, 2] of (row, nz) (lb_partition_nz)."""
        L = int(items_per_tile) or 1016
        T = max(1, (self.nnz + L - 1) // L)
        out = torch.empty((T + 1, 2), dtype=torch.int32, device=self.device)
        _check(lib().lb_partition_nz(self.handle, L, out.data_ptr(), _stream(stream)))
        return out

    def spmv(self, x: torch.Tensor, y: torch.Tensor | None = None, schedule="merge_path",
             repartition: bool = False, stream=None) -> torch.Tensor:
        """y = A x (lb_spmv / lb_spmv_ex)."""
        _dev_tensor(x, torch.float32, "x", self.cols)
        if y is None:
            y = torch.empty(self.rows, dtype=torch.float32, device=self.device)
        _dev_tensor(y, torch.float32, "y", self.rows)
        flags = LB_SPMV_REPARTITION if repartition else 0
        _check(lib().lb_spmv_ex(self.handle, _sched(schedule), x.data_ptr() if self.cols else None,
                                y.data_ptr() if self.rows else None, flags, _stream(stream)))
        return y

    def select_schedule(self, stream=None) -> str:
        """The schedule LB_SCHED_AUTO resolves to for this matrix (lb_select_schedule)."""
        out = ctypes.c_int()
        _check(lib().lb_select_schedule(self.handle, _stream(stream), ctypes.byref(out)))
        return SCHEDULE_NAMES[out.value]

    def spmm(self, X: torch.Tensor, Y: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """Y = A X for a dense row-major X [cols, n] (lb_spmm, merge-path tiles)."""
        if X.dim() != 2 or X.shape[0] != self.cols:
            raise ValueError(f"X must be [cols={self.cols}, n]")
        if X.device.type != "cuda" or X.dtype != torch.float32 or X.stride(1) != 1:
            raise ValueError("X must be a CUDA float32 tensor with unit column stride")
        n = X.shape[1]
        if Y is None:
            Y = torch.empty((self.rows, n), dtype=torch.float32, device=self.device)
        if Y.shape != (self.rows, n) or Y.dtype != torch.float32 or Y.stride(1) != 1:
            raise ValueError("Y must be float32 [rows, n] with unit column stride")
        _check(lib().lb_spmm(self.handle, n, X.data_ptr() if X.numel() else None, max(X.stride(0), n),
                             Y.data_ptr() if Y.numel() else None, max(Y.stride(0), n), _stream(stream)))
        return Y

    def spmv_host(self, h_x: torch.Tensor, h_y: torch.Tensor, schedule="merge_path", repartition: bool = False,
                  stream=None, chunked: bool = False) -> torch.Tensor:
        """lb_spmv_host_x: y = A x with x and y in HOST memory (pinned for full bandwidth); the matrix stays
        on the device.  chunked: LB_SPMV_CHUNKED (y copied out per row chunk while the next computes).
        Returns h_y after the call has synchronised."""
        for t, n, nm in ((h_x, self.cols, "h_x"), (h_y, self.rows, "h_y")):
            if t.device.type != "cpu" or t.dtype != torch.float32 or not t.is_contiguous() or t.numel() != n:
                raise ValueError(f"{nm} must be a contiguous float32 CPU tensor of {n} elements")
        flags = (LB_SPMV_REPARTITION if repartition else 0) | (LB_SPMV_CHUNKED if chunked else 0)
        _check(lib().lb_spmv_host_x(self.handle, _sched(schedule), h_x.data_ptr() if h_x.numel() else None,
                                    h_y.data_ptr() if h_y.numel() else None, flags, _stream(stream)))
        return h_y

    def spmv_host_async(self, h_x: torch.Tensor, h_y: torch.Tensor, schedule="merge_path",
                        repartition: bool = False, stream=None) -> torch.Tensor:
        """lb_spmv_host_x_async: enqueue y = A x with HOST x and y (pinned) on two alternating staging
        slots; h_y is valid (and h_x may be reused) after spmv_host_wait()."""
        for t, n, nm in ((h_x, self.cols, "h_x"), (h_y, self.rows, "h_y")):
            if t.device.type != "cpu" or t.dtype != torch.float32 or not t.is_contiguous() or t.numel() != n:
                raise ValueError(f"{nm} must be a contiguous float32 CPU tensor of {n} elements")
        _check(lib().lb_spmv_host_x_async(self.handle, _sched(schedule), h_x.data_ptr() if h_x.numel() else None,
                                          h_y.data_ptr() if h_y.numel() else None, 1 if repartition else 0,
                                          _stream(stream)))
        # the copies run on the library's own streams, which PyTorch's caching host allocator does not
        # track: keep both tensors alive until spmv_host_wait
        self._host_refs.append((h_x, h_y))
        return h_y

    def spmv_host_wait(self) -> None:
        """lb_spmv_host_x_wait: block until every enqueued spmv_host_async's y is on the host."""
        _check(lib().lb_spmv_host_x_wait(self.handle))
        self._host_refs = []

    def chunk_rows(self, stream=None) -> np.ndarray:
        """The handle's LB_SPMV_CHUNKED cut rows padded to CHUNKS_MAX + 1 entries (lb_csr_chunk_rows)."""
        out = np.zeros(CHUNKS_MAX + 1, np.int64)
        _check(lib().lb_csr_chunk_rows(self.handle, CHUNKS_MAX, out.ctypes.data, _stream(stream)))
        return out

    def probe_stream(self, reps: int = 20, stream=None) -> float:
        """Milliseconds of one read-only pass over col_idx + values (lb_probe_stream)."""
        ms = ctypes.c_float(0.0)
        _check(lib().lb_probe_stream(self.handle, int(reps), _stream(stream), ctypes.byref(ms)))
        return float(ms.value)

    def probe_stream_gather(self, x: torch.Tensor, reps: int = 20, stream=None) -> float:
        """Milliseconds of one stream+gather pass over this matrix (lb_probe_stream_gather)."""
        ms = ctypes.c_float()
        _check(lib().lb_probe_stream_gather(self.handle, x.data_ptr(), int(reps), _stream(stream), ctypes.byref(ms)))
        return float(ms.value)

    def sssp(self, source: int, schedule="merge_path", dist: torch.Tensor | None = None,
             stream=None) -> tuple[torch.Tensor, int]:
        """Single-source shortest paths over this matrix as a graph (lb_sssp).  Returns (dist, rounds)."""
        if dist is None:
            dist = torch.empty(self.rows, dtype=torch.float32, device=self.device)
        _dev_tensor(dist, torch.float32, "dist", self.rows)
        r = ctypes.c_int32()
        _check(lib().lb_sssp(self.handle, int(source), _sched(schedule), dist.data_ptr() if self.rows else None,
                             _stream(stream), ctypes.byref(r)))
        return dist, int(r.value)

    def spmv_peers(self, x: torch.Tensor, y: torch.Tensor, peers: list, repartition: bool = False,
                   stream=None) -> torch.Tensor:
        """lb_spmv_peers: merge-path y = A x whose tile kernel also stores every final y value into each
        peer tensor (the fused multi-GPU epilogue exercised on one GPU)."""
        _dev_tensor(x, torch.float32, "x", self.cols)
        _dev_tensor(y, torch.float32, "y", self.rows)
        for q in peers:
            _dev_tensor(q, torch.float32, "peer", self.rows)
        arr = (ctypes.c_void_p * max(len(peers), 1))(*[q.data_ptr() for q in peers])
        _check(lib().lb_spmv_peers(self.handle, x.data_ptr(), y.data_ptr(), arr, len(peers),
                                   LB_SPMV_REPARTITION if repartition else 0, _stream(stream)))
        return y

    def plan_hot_x(self, slots: int = 0, warm: int = -1, stream=None) -> tuple[int, int]:
        """Build (slots >= 0; 0 = library default) or drop (slots < 0) the x-reuse plan
        (lb_csr_plan_hot_x; warm: 0 none, -1 auto, > 0 column budget, -2 compact x).  Returns (hot columns,
        stored entries in them); plan_info() has the warm tier."""
        n, h = ctypes.c_int32(), ctypes.c_int64()
        _check(lib().lb_csr_plan_hot_x(self.handle, int(slots), int(warm), _stream(stream), ctypes.byref(n),
                                       ctypes.byref(h)))
        return int(n.value), int(h.value)

    def plan_info(self) -> dict:
        n, h, wn, wh = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(lib().lb_csr_hot_plan(self.handle, ctypes.byref(n), ctypes.byref(h), ctypes.byref(wn), ctypes.byref(wh),
                                     None, None, None, None))
        return {"hot_cols": int(n.value), "hot_nnz": int(h.value), "warm_cols": int(wn.value),
                "warm_nnz": int(wh.value)}

    def bins(self, stream=None):
        """The BINNING schedule's three bins (lb_bins): (cta_rows, warp_rows, thread_rows), ascending int32."""
        ids = torch.empty(self.rows, dtype=torch.int32, device=self.row_offsets.device)
        sizes = (ctypes.c_int64 * 3)()
        _check(lib().lb_bins(self.handle, ids.data_ptr() if self.rows else None, sizes, _stream(stream)))
        n0, n1 = int(sizes[0]), int(sizes[1])
        return ids[:n0], ids[n0:n0 + n1], ids[n0 + n1:]

    def hot_plan(self, stream=None):
        """Copies of the plan's hot slot table, warm table and remapped column stream (None without a plan)."""
        info = self.plan_info()
        if info["hot_cols"] == 0:
            return None
        dev = self.row_offsets.device
        hot = torch.empty(info["hot_cols"], dtype=torch.int32, device=dev)
        warm = torch.empty(info["warm_cols"], dtype=torch.int32, device=dev)
        hcol = torch.empty(self.nnz, dtype=torch.int32, device=dev)
        n, h, wn, wh = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(lib().lb_csr_hot_plan(self.handle, ctypes.byref(n), ctypes.byref(h), ctypes.byref(wn), ctypes.byref(wh),
                                     hot.data_ptr(), warm.data_ptr() if warm.numel() else None, hcol.data_ptr(),
                                     _stream(stream)))
        return hot, warm, hcol

    def trace_phases(self, capacity: int) -> None:
        """lb_csr_trace_phases: record per-phase CUDA events for the next `capacity` SpMV calls."""
        _check(lib().lb_csr_trace_phases(self.handle, int(capacity)))
        self._trace_cap = int(capacity)

    def trace_read(self) -> np.ndarray:
        """lb_csr_trace_read: [n, 3] (partition, main, fix-up) ms of the traced calls; resets the trace."""
        cap = getattr(self, "_trace_cap", 0)
        buf = (ctypes.c_float * max(3 * cap, 3))()
        n = ctypes.c_int32()
        _check(lib().lb_csr_trace_read(self.handle, ctypes.byref(n), buf))
        return np.frombuffer(buf, dtype=np.float32, count=3 * n.value).reshape(n.value, 3).astype(np.float64)

    def kernel_name(self, schedule="merge_path") -> str:
        """Main kernel lb_spmv launches for `schedule` (lb_kernel_name)."""
        return lib().lb_kernel_name(self.handle, _sched(schedule)).decode()

    def phase_times(self, x: torch.Tensor, y: torch.Tensor, schedule="merge_path", stream=None) -> list[float]:
        """[partition, main, fixup] milliseconds of one call (lb_spmv_phase_times)."""
        ms = (ctypes.c_float * 3)()
        _check(lib().lb_spmv_phase_times(self.handle, _sched(schedule), x.data_ptr(), y.data_ptr(),
                                         _stream(stream), ms))
        return [float(v) for v in ms]


def spmv(A: CsrMatrix, x: torch.Tensor, schedule="merge_path", y=None) -> torch.Tensor:
    return A.spmv(x, y, schedule)


# ----------------------------------------------------------------------------- end to end (host buffers)

class HostSpmv:
    """End-to-end y = A x from host (pinned) buffers through lb_spmv_host: H2D copies of the
    CSR arrays and x, partition + SpMV, D2H copy of y, all inside the call."""

    def __init__(self, rows: int, cols: int, nnz: int, device="cuda"):
        self.rows, self.cols, self.nnz = rows, cols, nnz
        self.ws_bytes = int(lib().lb_spmv_host_workspace_size(rows, cols, nnz))
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=device)

    def __call__(self, row_offsets: torch.Tensor, col_idx: torch.Tensor, values: torch.Tensor, x: torch.Tensor,
                 y: torch.Tensor, schedule="merge_path", stream=None) -> torch.Tensor:
        for t, name in ((row_offsets, "row_offsets"), (col_idx, "col_idx"), (values, "values"), (x, "x"), (y, "y")):
            if t.device.type != "cpu" or not t.is_contiguous():
                raise ValueError(f"{name} must be a contiguous host tensor")
        with torch.cuda.device(self.ws.device):
            _check(lib().lb_spmv_host(self.rows, self.cols, self.nnz, row_offsets.data_ptr(), col_idx.data_ptr(),
                                      values.data_ptr(), x.data_ptr(), y.data_ptr(), _sched(schedule),
                                      self.ws.data_ptr(), self.ws_bytes, _stream(stream)))
        return y


# ----------------------------------------------------------------------------- multi-GPU host logic

def shard_bounds(row_offsets, nranks: int) -> np.ndarray:
    """Equal-nnz row-shard bounds (lb_shard_bounds, host-only)."""
    off = row_offsets.detach().cpu().numpy() if hasattr(row_offsets, "detach") else np.asarray(row_offsets)
    off = np.ascontiguousarray(off, dtype=np.int32)
    out = np.empty(nranks + 1, np.int64)
    _check(lib().lb_shard_bounds(off.ctypes.data, off.size - 1, int(nranks), out.ctypes.data))
    return out


def exchange_schedule(bounds, cut_rows=None) -> tuple[np.ndarray, np.ndarray]:
    """The broadcasts of the y exchange (lb_exchange_schedule, host-only): (offsets, counts), each int64
    [nchunks, nranks]; chunk c, root k broadcasts y_full[offsets[c, k] : offsets[c, k] + counts[c, k]].
    cut_rows: int64 [nranks, nchunks + 1] local cut rows of every rank (None: one chunk, the plain
    all-gather of lb_allgather_rows)."""
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    G = b.size - 1
    cuts = None if cut_rows is None else np.ascontiguousarray(cut_rows, dtype=np.int64)
    K = 1 if cuts is None else cuts.shape[1] - 1
    if cuts is not None and cuts.shape[0] != G:
        raise ValueError("cut_rows must be [nranks, nchunks + 1]")
    off = np.empty((K, G), np.int64)
    cnt = np.empty((K, G), np.int64)
    _check(lib().lb_exchange_schedule(G, b.ctypes.data, K, None if cuts is None else cuts.ctypes.data,
                                      off.ctypes.data, cnt.ctypes.data))
    return off, cnt


def gather_slices(bounds) -> list[tuple[int, int]]:
    """The y slice [b_k, b_{k+1}) each rank k contributes to the all-gather (lb_allgather_rows)."""
    off, cnt = exchange_schedule(bounds)
    return [(int(o), int(o + c)) for o, c in zip(off[0], cnt[0])]


def padded_rows(bounds) -> int:
    """P = the largest shard: the slot size of the padded all-gather layout (lb_padded_rows)."""
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    return int(lib().lb_padded_rows(b.size - 1, b.ctypes.data))


def remap_cols_padded(bounds, col_idx: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """A shard's global column ids -> padded-layout ids k*P + (c - b_k) (lb_remap_cols_padded)."""
    _dev_tensor(col_idx, torch.int32, "col_idx")
    if out is None:
        out = torch.empty_like(col_idx)
    _dev_tensor(out, torch.int32, "out", col_idx.numel())
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    _check(lib().lb_remap_cols_padded(b.size - 1, b.ctypes.data, col_idx.data_ptr() if col_idx.numel() else None,
                                      col_idx.numel(), out.data_ptr() if out.numel() else None, _stream(stream)))
    return out


def y_checksum(y: torch.Tensor, stream=None) -> int:
    """lb_y_checksum: sum_i mix64(i * 0x9E3779B97F4A7C15 + bits(y_i)) mod 2^64 (include/lb.h)."""
    _dev_tensor(y, torch.float32, "y")
    h = ctypes.c_uint64()
    _check(lib().lb_y_checksum(y.data_ptr() if y.numel() else None, y.numel(), _stream(stream), ctypes.byref(h)))
    return int(h.value)


def shard_csr(row_offsets: torch.Tensor, col_idx: torch.Tensor, values: torch.Tensor, bounds, rank: int):
    """Rows [b_r, b_{r+1}) of a CSR as its own CSR (offsets rebased to 0, global column ids).
    Returns fresh contiguous tensors on the same device (so 16-byte alignment holds)."""
    b0, b1 = int(bounds[rank]), int(bounds[rank + 1])
    off = row_offsets[b0:b1 + 1].to(torch.int64)
    base = int(off[0]) if off.numel() else 0
    end = int(off[-1]) if off.numel() else 0
    return ((off - base).to(torch.int32).contiguous(), col_idx[base:end].clone(), values[base:end].clone())


class Comm:
    """NCCL communicator owned by liblb (lb_comm_t)."""

    def __init__(self, uid: bytes, rank: int, nranks: int, device: int):
        self.rank, self.nranks, self.device = rank, nranks, device
        self._c = ctypes.c_void_p()
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        _check(lib().lb_comm_init(buf, rank, nranks, device, ctypes.byref(self._c)))

    @staticmethod
    def unique_id() -> bytes:
        buf = (ctypes.c_uint8 * 128)()
        _check(lib().lb_comm_unique_id(buf))
        return bytes(buf)

    @staticmethod
    def bootstrap_uid() -> bytes:
        """Rank 0 creates the NCCL unique id; torch.distributed (any backend) ships it to all ranks."""
        import torch.distributed as dist
        obj = [Comm.unique_id() if dist.get_rank() == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    @classmethod
    def from_process_group(cls, device: int) -> "Comm":
        """Bootstrap over torch.distributed: rank 0 makes the id, all ranks join the communicator."""
        import torch.distributed as dist
        uid = cls.bootstrap_uid()
        return cls(uid, dist.get_rank(), dist.get_world_size(), device)

    def close(self):
        if getattr(self, "_c", None):
            lib().lb_comm_destroy(self._c)
            self._c = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def spmv_multi(self, A_local: CsrMatrix, bounds, x_full: torch.Tensor, y_full: torch.Tensor,
                   schedule="merge_path", stream=None, repartition: bool = False,
                   chunked: bool = False, padded: bool = False) -> torch.Tensor:
        """lb_spmv_multi(_ex).  chunked: LB_SPMV_CHUNKED -- each chunk's rows are all-gathered while the
        next chunk computes; padded: LB_SPMV_PADDED -- x_full / y_full are nranks * padded_rows(bounds)
        long and A_local's columns were remapped with remap_cols_padded (collective: every rank passes the
        same flags)."""
        b = np.ascontiguousarray(bounds, dtype=np.int64)
        n_full = int(b[-1])
        if padded:
            n_full = self.nranks * padded_rows(b)
        _dev_tensor(x_full, torch.float32, "x_full", n_full if padded else A_local.cols)
        _dev_tensor(y_full, torch.float32, "y_full", n_full)
        if int(b[self.rank + 1] - b[self.rank]) != A_local.rows:
            raise ValueError("A_local's rows do not match bounds[rank + 1] - bounds[rank]")
        if repartition or chunked or padded:
            flags = ((LB_SPMV_REPARTITION if repartition else 0) | (LB_SPMV_CHUNKED if chunked else 0) |
                     (LB_SPMV_PADDED if padded else 0))
            _check(lib().lb_spmv_multi_ex(A_local.handle, self._c, _sched(schedule), b.ctypes.data, x_full.data_ptr(),
                                          y_full.data_ptr(), flags, _stream(stream)))
        else:
            _check(lib().lb_spmv_multi(A_local.handle, self._c, _sched(schedule), b.ctypes.data, x_full.data_ptr(),
                                       y_full.data_ptr(), _stream(stream)))
        return y_full

    def peer_buffer(self, y_full: torch.Tensor, stream=None) -> "PeerBuffer":
        return PeerBuffer(self, y_full, stream)

    def spmv_multi_fused(self, A_local: CsrMatrix, bounds, x_full: torch.Tensor, peer: "PeerBuffer",
                         schedule="merge_path", repartition: bool = False, stream=None) -> torch.Tensor:
        """lb_spmv_multi_fused: shard SpMV whose epilogue writes y into every rank's registered buffer."""
        b = np.ascontiguousarray(bounds, dtype=np.int64)
        _dev_tensor(x_full, torch.float32, "x_full", A_local.cols)
        _check(lib().lb_spmv_multi_fused(A_local.handle, peer._p, _sched(schedule), b.ctypes.data, x_full.data_ptr(),
                                         LB_SPMV_REPARTITION if repartition else 0, _stream(stream)))
        return peer.y

    def allgather_rows(self, bounds, y_full: torch.Tensor, stream=None) -> torch.Tensor:
        b = np.ascontiguousarray(bounds, dtype=np.int64)
        _dev_tensor(y_full, torch.float32, "y_full", int(b[-1]))
        _check(lib().lb_allgather_rows(self._c, b.ctypes.data, y_full.data_ptr(), _stream(stream)))
        return y_full

    def allgather_padded(self, bounds, y_pad: torch.Tensor, stream=None) -> torch.Tensor:
        """lb_allgather_padded: one ncclAllGather of the padded slots (slot r = y_pad[r*P : (r+1)*P])."""
        P = padded_rows(bounds)
        _dev_tensor(y_pad, torch.float32, "y_pad", self.nranks * P)
        _check(lib().lb_allgather_padded(self._c, P, y_pad.data_ptr(), _stream(stream)))
        return y_pad

    def check_replicas(self, y: torch.Tensor, stream=None) -> tuple[bool, int]:
        """lb_comm_check_replicas: (every rank's y is bitwise equal, this rank's hash)."""
        _dev_tensor(y, torch.float32, "y")
        eq, h = ctypes.c_int32(), ctypes.c_uint64()
        _check(lib().lb_comm_check_replicas(self._c, y.data_ptr() if y.numel() else None, y.numel(), _stream(stream),
                                            ctypes.byref(eq), ctypes.byref(h)))
        return bool(eq.value), int(h.value)


class PeerBuffer:
    """A y tensor registered with every rank of a Comm for the fused exchange (lb_peer_create)."""

    def __init__(self, comm: "Comm", y_full: torch.Tensor, stream=None):
        _dev_tensor(y_full, torch.float32, "y_full")
        self.y = y_full
        self.comm = comm
        self._p = ctypes.c_void_p()
        _check(lib().lb_peer_create(comm._c, y_full.data_ptr(), y_full.numel(), _stream(stream), ctypes.byref(self._p)))

    def close(self):
        if self._p:
            lib().lb_peer_destroy(self._p)
            self._p = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
