"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bars (BASELINE.json north_star):
  * partition coordinates: bit-exact;
  * y in integer mode (values {+-1,+-2}, x {-4..4}, every partial sum an exact fp32 integer):
    bit-exact, compared by value;
  * y in tolerance mode (values and x uniform in [-1,1) on a 2^-23 grid):
    |y_gpu - y_ref| <= 1e-5 * s_ref + 1e-30 per row, s_ref = sum_k |a_ik x_k|.
Sizes span several tiles and ragged tails; full BASELINE.json sizes are covered by
test_full_size_configs (partition bit-exact on every tile, every schedule on every row of C1-C5).
"""
import ctypes

import os

import numpy as np
import pytest
import torch

import lbgen
import oracle
import paper_2212_08964_b200 as lb

pytestmark = pytest.mark.gpu

SCHEDS = ["merge_path", "thread_mapped", "group_mapped", "block_mapped", "auto", "nonzero_split", "warp_mapped",
          "binning"]
TOL = 1e-5


def ref(A: lbgen.Csr, x: torch.Tensor):
    return oracle.spmv(A.row_offsets, A.col_idx, A.values, x, threads=A.nnz > 1_000_000)


def check_y(y_gpu: torch.Tensor, y_ref: np.ndarray, s_ref: np.ndarray, exact: bool, what=""):
    y = y_gpu.detach().double().cpu().numpy()
    assert y.shape == y_ref.shape
    if exact:
        bad = np.nonzero(y != y_ref)[0]
        assert bad.size == 0, f"{what}: {bad.size} rows differ, first {bad[:5]} gpu={y[bad[:5]]} ref={y_ref[bad[:5]]}"
    else:
        err = np.abs(y - y_ref)
        lim = TOL * s_ref + 1e-30
        bad = np.nonzero(err > lim)[0]
        assert bad.size == 0, f"{what}: {bad.size} rows out of tolerance, worst rel {np.max(err / (s_ref + 1e-30)):.3e}"


def run(A: lbgen.Csr, x: torch.Tensor, sched: str, L: int = 0) -> torch.Tensor:
    M = lb.CsrMatrix.from_csr(A)
    if L:
        M.set_items_per_tile(L)
    y = torch.full((A.rows,), float("nan"), device="cuda")
    M.spmv(x.cuda(), y, sched)
    torch.cuda.synchronize()
    return y


def random_csr(rng, rows, cols, max_len, p_empty, vmode):
    lens = rng.integers(0, max_len + 1, rows)
    lens[rng.random(rows) < p_empty] = 0
    off = np.zeros(rows + 1, np.int64)
    off[1:] = np.cumsum(lens)
    nnz = int(off[-1])
    col = np.sort(rng.integers(0, max(cols, 1), nnz))  # per-row order is irrelevant to SpMV
    val = rng.choice([-2.0, -1.0, 1.0, 2.0], nnz) if vmode == "int" else rng.integers(-(1 << 23), 1 << 23, nnz) * 2.0 ** -23
    return lbgen.Csr(rows, cols, torch.tensor(off, dtype=torch.int32), torch.tensor(col, dtype=torch.int32),
                     torch.tensor(val, dtype=torch.float32))


SMALL = {
    "rmat12": lambda vm: lbgen.rmat(12, 16, 3, vm),
    "rmat14": lambda vm: lbgen.rmat(14, 8, 7, vm),
    "stencil100": lambda vm: lbgen.stencil(100, 2, vm),
    "skewed": lambda vm: lbgen.skewed(1 << 13, 5, 20_000, 50_000, 4, vm),
    "c1": lambda vm: lbgen.make_config("c1", vm),
    "uniform_rows": lambda vm: lbgen.uniform_rows(13, 16, 6, vm),
}


# ---------------------------------------------------------------- partition (bit-exact)

@pytest.mark.parametrize("L", [1, 2, 3, 7, 256, 1016, 2048, 3064, 5000])
@pytest.mark.parametrize("name", ["rmat12", "stencil100", "skewed", "c1"])
def test_partition_bit_exact(name, L):
    A = SMALL[name]("int")
    M = lb.CsrMatrix.from_csr(A)
    got = M.partition(L).cpu().numpy()
    want = oracle.partition(A.row_offsets, L)
    assert np.array_equal(got, want)


def test_partition_random_every_diagonal():
    rng = np.random.default_rng(1)
    for trial in range(40):
        A = random_csr(rng, int(rng.integers(1, 300)), 50, int(rng.integers(0, 30)), float(rng.random()), "int")
        M = lb.CsrMatrix.from_csr(A)
        assert np.array_equal(M.partition(1).cpu().numpy(), oracle.partition(A.row_offsets, 1)), trial


@pytest.mark.parametrize("extra", [-1, 0, 1])
@pytest.mark.parametrize("shape", ["long_rows", "empty_runs"])
def test_partition_both_search_kernels(shape, extra):
    """The 16-lane group search (<= 32,768 boundaries) and the thread-per-boundary search (more) give
    the brute-force coordinates on both sides of the switch: T + 1 = 32,768 - 1 .. + 1 at L = 64."""
    L = 64
    rng = np.random.default_rng(7 + extra)
    target = (32768 - 1 + extra) * L - 1  # rows + nnz with T = ceil(total / L) = 32767 + extra
    rows = 200_000 if shape == "long_rows" else 1_500_000
    nnz = target - rows
    if shape == "long_rows":  # a few very long rows among short ones
        w = rng.pareto(1.2, rows) + 1e-3
    else:  # long runs of empty rows between short ones
        w = np.where(rng.random(rows) < 0.7, 0.0, rng.random(rows) + 0.1)
    cnt = np.floor(w / w.sum() * nnz).astype(np.int64)
    cnt[: nnz - int(cnt.sum())] += 1
    off = np.zeros(rows + 1, np.int64)
    np.cumsum(cnt, out=off[1:])
    assert off[-1] == nnz
    off_t = torch.from_numpy(off.astype(np.int32))
    A = lbgen.Csr(rows, 64, off_t, torch.zeros(nnz, dtype=torch.int32), torch.ones(nnz))
    M = lb.CsrMatrix.from_csr(A)
    assert M.num_tiles(L) == 32767 + extra
    assert np.array_equal(M.partition(L).cpu().numpy(), oracle.partition(off_t, L))


# ---------------------------------------------------------------- SpMV parity

@pytest.mark.parametrize("sched", SCHEDS)
@pytest.mark.parametrize("name", sorted(SMALL))
def test_spmv_integer_exact(name, sched):
    A = SMALL[name]("int")
    x = lbgen.make_x(A.cols, "int", 11)
    y_ref, s_ref = ref(A, x)
    assert np.all(s_ref < 2 ** 24)
    check_y(run(A, x, sched), y_ref, s_ref, True, f"{name}/{sched}")


@pytest.mark.parametrize("sched", SCHEDS)
@pytest.mark.parametrize("name", sorted(SMALL))
def test_spmv_tolerance(name, sched):
    A = SMALL[name]("float")
    x = lbgen.make_x(A.cols, "float", 12)
    y_ref, s_ref = ref(A, x)
    check_y(run(A, x, sched), y_ref, s_ref, False, f"{name}/{sched}")


@pytest.mark.parametrize("L", [504, 1016, 2040, 3064, 4088])
@pytest.mark.parametrize("vmode", ["int", "float"])
def test_merge_path_tile_lengths(L, vmode):
    A = lbgen.rmat(13, 16, 5, vmode)
    x = lbgen.make_x(A.cols, vmode, 3)
    y_ref, s_ref = ref(A, x)
    check_y(run(A, x, "merge_path", L), y_ref, s_ref, vmode == "int")


@pytest.mark.parametrize("sched", SCHEDS)
def test_random_ragged_matrices(sched):
    rng = np.random.default_rng(5)
    for trial in range(25):
        rows = int(rng.integers(1, 3000))
        A = random_csr(rng, rows, int(rng.integers(1, 500)), int(rng.integers(0, 60)), float(rng.random()) * 0.7, "int")
        x = lbgen.make_x(A.cols, "int", trial)
        y_ref, s_ref = ref(A, x)
        check_y(run(A, x, sched), y_ref, s_ref, True, f"trial {trial}")


@pytest.mark.parametrize("sched", SCHEDS)
def test_identity_and_diagonal_bit_exact(sched):
    n = 70_001
    idx = torch.arange(n, dtype=torch.int32)
    off = torch.arange(n + 1, dtype=torch.int32)
    x = lbgen.make_x(n, "float", 1)
    I = lbgen.Csr(n, n, off, idx, torch.ones(n))
    assert torch.equal(run(I, x, sched).cpu(), x)                       # y = x
    d = lbgen.make_x(n, "float", 2)
    D = lbgen.Csr(n, n, off, idx, d)
    assert torch.equal(run(D, x, sched).cpu(), d * x)                   # y_i = fl(d_i x_i)


@pytest.mark.parametrize("sched", SCHEDS)
@pytest.mark.parametrize("xmode", ["ones", "index"])
def test_stencil_closed_form(sched, xmode):
    N = 300
    A = lbgen.stencil(N, 2, "stencil")
    x = lbgen.make_x(N * N, xmode, 0)
    i = np.arange(N * N, dtype=np.int64)
    yy, xx = i // N, i % N
    missing = [(yy == 0, i - N), (xx == 0, i - 1), (xx == N - 1, i + 1), (yy == N - 1, i + N)]
    if xmode == "ones":
        expect = sum(m.astype(np.float64) for m, _ in missing)
    else:
        expect = sum(np.where(m, v, 0).astype(np.float64) for m, v in missing)
    y = run(A, x, sched).double().cpu().numpy()
    assert np.array_equal(y, expect)


# ---------------------------------------------------------------- edge cases

def _csr(off, cols, col=None, val=None):
    off = torch.tensor(off, dtype=torch.int32)
    nnz = int(off[-1])
    col = torch.zeros(nnz, dtype=torch.int32) if col is None else torch.tensor(col, dtype=torch.int32)
    val = torch.ones(nnz) if val is None else torch.tensor(val, dtype=torch.float32)
    return lbgen.Csr(off.numel() - 1, cols, off, col, val)


@pytest.mark.parametrize("sched", SCHEDS)
def test_edge_cases(sched):
    cases = {
        "no_nnz": _csr([0] * 5001, 3),
        "one_giant_row": _csr([0, 200_003], 1),
        "giant_last_row": _csr([0] * 3000 + [100_000], 1),
        "empty_rows_between": _csr([0, 1, 1, 1, 5, 5, 9], 1),
        "golden": _csr([0, 1, 3, 3, 6], 1),
        "single": _csr([0, 1], 1),
        "cols1_many_rows": _csr(list(range(0, 2 * 40_000 + 1, 2)), 1),
    }
    for name, A in cases.items():
        x = torch.full((A.cols,), 1.0)
        y_ref, s_ref = ref(A, x)
        check_y(run(A, x, sched), y_ref, s_ref, True, name)
    # golden example: y = [1, 2, 0, 3]
    assert run(cases["golden"], torch.ones(1), sched).tolist() == [1, 2, 0, 3]


def test_empty_matrix_is_noop():
    M = lb.CsrMatrix(0, 0, torch.zeros(1, dtype=torch.int32, device="cuda"),
                     torch.zeros(0, dtype=torch.int32, device="cuda"), torch.zeros(0, device="cuda"))
    y = torch.zeros(0, device="cuda")
    for s in SCHEDS:
        M.spmv(torch.zeros(0, device="cuda"), y, s)
    assert M.partition(16).cpu().tolist() == [[0, 0]]


def test_unaligned_arrays_use_scalar_path():
    A = lbgen.rmat(12, 8, 9, "int")
    x = lbgen.make_x(A.cols, "int", 4)
    y_ref, s_ref = ref(A, x)
    # shift col/val by one element inside a larger buffer -> not 16-byte aligned
    colbuf = torch.zeros(A.nnz + 1, dtype=torch.int32, device="cuda")
    valbuf = torch.zeros(A.nnz + 1, device="cuda")
    colbuf[1:] = A.col_idx.cuda()
    valbuf[1:] = A.values.cuda()
    M = lb.CsrMatrix(A.rows, A.cols, A.row_offsets.cuda(), colbuf[1:], valbuf[1:])
    y = M.spmv(x.cuda())
    check_y(y, y_ref, s_ref, True, "unaligned")


def test_validation_rejects_invalid_csr():
    dev = "cuda"
    with pytest.raises(lb.InvalidCsr, match="monotone at row 1"):
        lb.CsrMatrix(3, 4, torch.tensor([0, 2, 1, 3], dtype=torch.int32, device=dev),
                     torch.zeros(3, dtype=torch.int32, device=dev), torch.ones(3, device=dev))
    with pytest.raises(lb.InvalidCsr, match=r"col_idx\[2\]"):
        lb.CsrMatrix(2, 4, torch.tensor([0, 1, 3], dtype=torch.int32, device=dev),
                     torch.tensor([0, 3, 4], dtype=torch.int32, device=dev), torch.ones(3, device=dev))
    with pytest.raises(lb.InvalidCsr, match=r"row_offsets\[0\]"):
        lb.CsrMatrix(2, 4, torch.tensor([1, 1, 3], dtype=torch.int32, device=dev),
                     torch.zeros(3, dtype=torch.int32, device=dev), torch.ones(3, device=dev))
    with pytest.raises(lb.InvalidCsr, match="!= nnz"):
        lb.CsrMatrix(2, 4, torch.tensor([0, 1, 2], dtype=torch.int32, device=dev),
                     torch.zeros(3, dtype=torch.int32, device=dev), torch.ones(3, device=dev))


def test_argument_errors():
    A = lbgen.make_config("c1", "int")
    M = lb.CsrMatrix.from_csr(A)
    x = torch.ones(A.cols, device="cuda")
    with pytest.raises(ValueError):
        M.spmv(x, schedule="nonsense")
    with pytest.raises(lb.LbError):
        M.spmv(x, schedule=17)
    with pytest.raises(lb.LbError):
        M.set_items_per_tile(3000)
    with pytest.raises(lb.LbError):
        M.set_items_per_tile(2048)
    with pytest.raises(ValueError):
        M.spmv(torch.ones(A.cols + 1, device="cuda"))


def test_trace_phases_records_the_traced_calls():
    """lb_csr_trace_phases / lb_csr_trace_read (bench.py times the tile kernel inside its timed region
    with them): one (partition, main, fix-up) row per traced call up to the capacity, positive main
    times, y unchanged by tracing, reset after a read, disabled by capacity 0."""
    A = lbgen.rmat(14, 16, 4, "int")
    x = lbgen.make_x(A.cols, "int", 2).cuda()
    M = lb.CsrMatrix.from_csr(A)
    y0 = M.spmv(x, schedule="merge_path", repartition=True).clone()
    M.trace_phases(3)
    for _ in range(5):
        y = M.spmv(x, schedule="merge_path", repartition=True)
    tr = M.trace_read()
    assert tr.shape == (3, 3) and np.all(tr[:, 1] > 0) and np.all(tr >= 0)
    assert torch.equal(y, y0)
    assert M.trace_read().shape == (0, 3)  # reset by the read
    M.spmv(x, schedule="thread_mapped")
    assert M.trace_read().shape == (1, 3)  # capacity kept
    M.trace_phases(0)
    M.spmv(x, schedule="merge_path")
    assert M.trace_read().shape == (0, 3)


def test_deterministic_bitwise():
    A = lbgen.rmat(14, 16, 2, "float")
    x = lbgen.make_x(A.cols, "float", 8).cuda()
    M = lb.CsrMatrix.from_csr(A)
    for sched in SCHEDS:
        y1 = M.spmv(x, schedule=sched, repartition=True).clone()
        y2 = M.spmv(x, schedule=sched).clone()
        assert torch.equal(y1, y2)


def test_launch_count_and_phase_times():
    A = lbgen.rmat(12, 16, 2, "float")
    M = lb.CsrMatrix.from_csr(A)
    x = lbgen.make_x(A.cols, "float", 8).cuda()
    y = torch.empty(A.rows, device="cuda")
    n0 = lb.launch_count()
    M.spmv(x, y, "merge_path", repartition=True)
    assert lb.launch_count() - n0 in (2, 3)     # partition + tiles (+ fix-up kernel on the unaligned path)
    ms = M.phase_times(x, y, "merge_path")
    assert len(ms) == 3 and all(v >= 0 for v in ms) and ms[1] > 0


# ---------------------------------------------------------------- end to end + multi-GPU layer

@pytest.mark.parametrize("sched", SCHEDS)
def test_spmv_host_end_to_end(sched):
    A = lbgen.rmat(13, 16, 4, "int")
    x = lbgen.make_x(A.cols, "int", 5)
    y_ref, s_ref = ref(A, x)
    h = lb.HostSpmv(A.rows, A.cols, A.nnz)
    y = torch.empty(A.rows).pin_memory()
    h(A.row_offsets.pin_memory(), A.col_idx.pin_memory(), A.values.pin_memory(), x.pin_memory(), y, sched)
    check_y(y, y_ref, s_ref, True, "host")


@pytest.mark.parametrize("sched", SCHEDS)
def test_spmv_host_x_resident_matrix(sched):
    """lb_spmv_host_x: device-resident A, host x / y (pinned and pageable), repeated calls with new x,
    with and without the x-reuse plan; bit-exact in integer mode."""
    A = lbgen.rmat(13, 16, 6, "int")
    M = lb.CsrMatrix.from_csr(A)
    for it, pinned in enumerate((True, False, True)):
        x = lbgen.make_x(A.cols, "int", 20 + it)
        y_ref, s_ref = ref(A, x)
        hx = x.pin_memory() if pinned else x.clone()
        hy = torch.full((A.rows,), float("nan"))
        hy = hy.pin_memory() if pinned else hy
        M.spmv_host(hx, hy, sched, repartition=it == 0)
        check_y(hy, y_ref, s_ref, True, f"host_x/{sched}/{it}")
    if sched == "merge_path":
        M.plan_hot_x(256, 1000)
        x = lbgen.make_x(A.cols, "int", 40)
        y_ref, s_ref = ref(A, x)
        hy = torch.empty(A.rows)
        M.spmv_host(x, hy, sched, repartition=True)
        check_y(hy, y_ref, s_ref, True, "host_x/plan")
    with pytest.raises(ValueError):
        M.spmv_host(torch.zeros(A.cols + 1), torch.zeros(A.rows), sched)


@pytest.mark.parametrize("sched", ["merge_path", "thread_mapped"])
def test_spmv_host_x_async_pipeline(sched):
    """lb_spmv_host_x_async: five independent x vectors enqueued back to back on the three staging slots
    (each call overlaps the previous calls' copies), one wait; every h_y equals the oracle bit for bit
    in integer mode, with and without the x-reuse plan, and a second batch reuses the slots."""
    A = lbgen.rmat(13, 16, 7, "int")
    M = lb.CsrMatrix.from_csr(A)
    for batch in range(2):
        if batch == 1 and sched == "merge_path":
            M.plan_hot_x(256, 1000)
        xs = [lbgen.make_x(A.cols, "int", 60 + 10 * batch + i) for i in range(5)]
        hxs = [x.pin_memory() for x in xs]
        hys = [torch.full((A.rows,), float("nan")).pin_memory() for _ in xs]
        for i, (hx, hy) in enumerate(zip(hxs, hys)):
            M.spmv_host_async(hx, hy, sched, repartition=i == 0)
        M.spmv_host_wait()
        for i, (x, hy) in enumerate(zip(xs, hys)):
            y_ref, s_ref = ref(A, x)
            check_y(hy, y_ref, s_ref, True, f"host_x_async/{sched}/{batch}/{i}")
    with pytest.raises(ValueError):
        M.spmv_host_async(torch.zeros(A.cols + 1), torch.zeros(A.rows), sched)


@pytest.mark.parametrize("case", ["rmat13", "rmat15_float", "giant_row", "ragged"])
def test_spmv_host_x_chunked(case):
    """lb_spmv_host_x(LB_SPMV_CHUNKED): the hot-plan tile kernel as up to 4 launches over tile ranges cut
    at clean merge-path coordinates, y rows copied out per range.  Integer mode bit-exact against the
    oracle; float mode within tolerance; a giant row with no clean cut inside it; repeated calls with
    a new x reuse the cached cuts."""
    if case == "rmat13":
        A, vm = lbgen.rmat(13, 16, 21, "int"), "int"
    elif case == "rmat15_float":
        A, vm = lbgen.rmat(15, 16, 22, "float"), "float"
    elif case == "giant_row":
        A, vm = _csr([0, 3, 3, 200_003, 200_010] + [200_010 + 5 * i for i in range(1, 600)], 1), "int"
    else:
        A, vm = lbgen.skewed(16_384, 5, 20_000, 300_000, 23, "int"), "int"
    M = lb.CsrMatrix.from_csr(A)
    if M.plan_hot_x(64 if A.cols >= 64 else 1, 0)[0] == 0:
        pytest.skip("no hot plan for this matrix")
    for it in range(3):
        x = lbgen.make_x(A.cols, vm, 500 + it) if A.cols > 1 else torch.full((1,), float(it + 1))
        y_ref, s_ref = ref(A, x)
        hy = torch.full((A.rows,), float("nan")).pin_memory()
        M.spmv_host(x.pin_memory(), hy, "merge_path", repartition=it == 0, chunked=True)
        check_y(hy, y_ref, s_ref, vm == "int", f"chunked/{case}/{it}")


def test_spmv_host_x_chunked_full_size_c3():
    """LB_SPMV_CHUNKED at the bench's configuration (C3, default plan), integer mode: the host y equals
    the one-launch device call bit for bit (both exact)."""
    A = lbgen.make_config("c3", "int", device="cuda")
    x = lbgen.x_for_config("c3", A.cols, "int", device="cuda")
    M = lb.CsrMatrix.from_csr(A)
    M.plan_hot_x(0)
    y = M.spmv(x, schedule="merge_path", repartition=True)
    hy = torch.full((A.rows,), float("nan")).pin_memory()
    M.spmv_host(x.cpu().pin_memory(), hy, "merge_path", repartition=True, chunked=True)
    assert torch.equal(hy, y.cpu())


def test_spmv_host_x_async_edge_cases():
    """lb_spmv_host_x_async on degenerate shapes: no nonzeros (y = +0), one giant row, pageable host
    buffers, an odd number of calls (slot 0 used twice), and rows == 0 (no-op; wait returns)."""
    for name, A in {"no_nnz": _csr([0] * 5001, 3), "one_giant_row": _csr([0, 200_003], 1),
                    "empty_rows_between": _csr([0, 1, 1, 1, 5, 5, 9], 1)}.items():
        M = lb.CsrMatrix.from_csr(A)
        hys = []
        for i in range(3):
            x = torch.full((A.cols,), float(i + 1))
            hy = torch.full((A.rows,), float("nan"))
            M.spmv_host_async(x, hy, "merge_path")
            hys.append((x, hy))
        M.spmv_host_wait()
        for x, hy in hys:
            y_ref, s_ref = ref(A, x)
            check_y(hy, y_ref, s_ref, True, f"host_x_async/{name}")
    M = lb.CsrMatrix(0, 0, torch.zeros(1, dtype=torch.int32, device="cuda"),
                     torch.zeros(0, dtype=torch.int32, device="cuda"), torch.zeros(0, device="cuda"))
    M.spmv_host_async(torch.zeros(0), torch.zeros(0))
    M.spmv_host_wait()


@pytest.mark.parametrize("G", [2, 3, 8])
def test_row_shards_concatenate_bit_identical(G):
    """G equal-nnz shards run one after another on one GPU, concatenated,
    equal the single-GPU y bit for bit in integer mode."""
    A = lbgen.rmat(13, 16, 6, "int")
    x = lbgen.make_x(A.cols, "int", 6).cuda()
    full = run(A, x.cpu(), "merge_path")
    b = lb.shard_bounds(A.row_offsets, G)
    ys = []
    for r in range(G):
        off, col, val = lb.shard_csr(A.row_offsets.cuda(), A.col_idx.cuda(), A.values.cuda(), b, r)
        M = lb.CsrMatrix(int(b[r + 1] - b[r]), A.cols, off, col, val)
        ys.append(M.spmv(x))
    assert torch.equal(torch.cat(ys), full)


@pytest.mark.parametrize("plan", [True, False])
def test_spmv_multi_chunked_single_rank_nccl(plan):
    """lb_spmv_multi_ex(LB_SPMV_CHUNKED) at world size 1: tile-range launches, the cut-table exchange
    and one broadcast group per chunk on the exchange stream; bit-exact against the oracle in integer
    mode, repeated with a new x, with and without a plan (no plan: one chunk, same collectives)."""
    A = lbgen.rmat(14, 16, 8, "int")
    uid = lb.Comm.unique_id()
    comm = lb.Comm(uid, 0, 1, torch.cuda.current_device())
    b = lb.shard_bounds(A.row_offsets, 1)
    M = lb.CsrMatrix.from_csr(A)
    if plan:
        M.plan_hot_x(256, 0)
    for it in range(3):
        x = lbgen.make_x(A.cols, "int", 40 + it)
        y_ref, s_ref = ref(A, x)
        y = torch.full((A.rows,), float("nan"), device="cuda")
        comm.spmv_multi(M, b, x.cuda(), y, "merge_path", repartition=it == 0, chunked=True)
        torch.cuda.synchronize()
        check_y(y, y_ref, s_ref, True, f"multi_chunked/plan{plan}/{it}")


def test_spmv_multi_single_rank_nccl():
    A = lbgen.rmat(12, 16, 6, "int")
    x = lbgen.make_x(A.cols, "int", 6)
    y_ref, s_ref = ref(A, x)
    uid = lb.Comm.unique_id()
    comm = lb.Comm(uid, 0, 1, torch.cuda.current_device())
    b = lb.shard_bounds(A.row_offsets, 1)
    M = lb.CsrMatrix.from_csr(A)
    y = torch.empty(A.rows, device="cuda")
    comm.spmv_multi(M, b, x.cuda(), y)
    torch.cuda.synchronize()
    check_y(y, y_ref, s_ref, True, "multi")
    comm.close()


# ---------------------------------------------------------------- full BASELINE.json sizes

def _sample_rows(A_dev: lbgen.Csr, coords: np.ndarray, n_random: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    rows = A_dev.rows
    tile_rows = np.unique(np.clip(coords[:, 0].astype(np.int64), 0, rows - 1))
    lens = (A_dev.row_offsets[1:] - A_dev.row_offsets[:-1])
    top = torch.topk(lens, min(64, rows)).indices.cpu().numpy()
    pick = np.concatenate([rng.integers(0, rows, n_random), tile_rows[:: max(1, tile_rows.size // 20000)], top,
                           [0, rows - 1]])
    return np.unique(pick)


def _packed(A_dev: lbgen.Csr, sel: np.ndarray):
    off = A_dev.row_offsets.to(torch.int64)
    s = torch.as_tensor(sel, device=off.device)
    b, e = off[s], off[s + 1]
    lens = e - b
    so = torch.zeros(sel.size + 1, dtype=torch.int64, device=off.device)
    so[1:] = torch.cumsum(lens, 0)
    idx = torch.repeat_interleave(b - so[:-1], lens) + torch.arange(int(so[-1]), device=off.device)
    return so.cpu(), A_dev.col_idx[idx].cpu(), A_dev.values[idx].cpu()


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4", "c5"])
def test_full_size_configs(cfg):
    """Every schedule at the BASELINE.json size of each config (merge-path at the launch
    configuration bench.py times), against the oracle on EVERY row: partition bit-exact on every
    tile; integer mode bit-exact; tolerance mode within 1e-5 * s + 1e-30."""
    torch.cuda.empty_cache()
    for vmode in ("int", "float"):
        A = lbgen.make_config(cfg, vmode, device="cuda")
        x = lbgen.x_for_config(cfg, A.cols, vmode, device="cuda")
        M = lb.CsrMatrix.from_csr(A, device="cuda")
        coords = M.partition().cpu().numpy()
        if vmode == "int":
            assert np.array_equal(coords, oracle.partition(A.row_offsets.cpu(), M.items_per_tile)), "partition"
        del coords
        y_ref, s_ref = oracle.spmv(A.row_offsets.cpu(), A.col_idx.cpu(), A.values.cpu(), x.cpu(), threads=True)
        for sched in SCHEDS:
            y = torch.full((A.rows,), float("nan"), device="cuda")
            M.spmv(x, y, sched, repartition=True)
            torch.cuda.synchronize()
            check_y(y, y_ref, s_ref, vmode == "int", f"{cfg}/{vmode}/{sched}")
            del y
        del M, A, x, y_ref, s_ref
        torch.cuda.empty_cache()


# ---------------------------------------------------------------- every tile kernel

@pytest.mark.parametrize("aligned", [True, False])
@pytest.mark.parametrize("L", [504, 1016, 2040, 3064, 4088])
def test_every_tile_kernel(L, aligned):
    """The tile processor of each tile length (32-byte aligned col/val: warp-streamed or CTA tiles;
    otherwise the 128-bit / scalar fallback + fix-up kernel) is bit-exact in integer mode and within
    tolerance in float mode, on R-MAT, skewed and edge-case matrices."""
    cases = [("rmat", lambda vm: lbgen.rmat(13, 16, 5, vm)),
             ("skewed", lambda vm: lbgen.skewed(1 << 12, 3, 30_000, 20_000, 8, vm)),
             ("stencil", lambda vm: lbgen.stencil(70, 2, vm))]

    def run_L(A, x):
        if aligned:
            M = lb.CsrMatrix.from_csr(A)
        else:  # col / val one element past a 32-byte boundary
            col = torch.zeros(A.nnz + 1, dtype=torch.int32, device="cuda")
            val = torch.zeros(A.nnz + 1, device="cuda")
            col[1:] = A.col_idx.cuda()
            val[1:] = A.values.cuda()
            M = lb.CsrMatrix(A.rows, A.cols, A.row_offsets.cuda(), col[1:], val[1:])
        M.set_items_per_tile(L)
        assert M.kernel_name().startswith("merge_tile_kernel") != aligned or A.nnz == 0, M.kernel_name()
        y = torch.full((A.rows,), float("nan"), device="cuda")
        M.spmv(x.cuda(), y, "merge_path", repartition=True)
        torch.cuda.synchronize()
        return y

    for name, mk in cases:
        for vm in ("int", "float"):
            A = mk(vm)
            x = lbgen.make_x(A.cols, vm, 9)
            y_ref, s_ref = ref(A, x)
            check_y(run_L(A, x), y_ref, s_ref, vm == "int", f"L{L}/{aligned}/{name}/{vm}")
    for name, A in {"giant": _csr([0, 100_003], 1), "no_nnz": _csr([0] * 3001, 3),
                    "golden": _csr([0, 1, 3, 3, 6], 1)}.items():
        x = torch.ones(A.cols)
        y_ref, s_ref = ref(A, x)
        check_y(run_L(A, x), y_ref, s_ref, True, f"L{L}/{aligned}/{name}")


# ---------------------------------------------------------------- binning (Alg.4, NEXT-3)

def _check_bins(A: lbgen.Csr, what: str):
    M = lb.CsrMatrix.from_csr(A, device="cuda")
    got = [b.cpu().numpy() for b in M.bins()]
    want = oracle.bins(A.row_offsets.cpu())
    for g, w, name in zip(got, want, ("cta", "warp", "thread")):
        assert np.array_equal(g, w), f"{what}: {name} bin differs ({g.size} vs {w.size} rows)"


def test_bins_bit_exact():
    """lb_bins (the BINNING schedule's device-built bins) equal oracle_bins exactly: generators whose rows
    fall in all three bins, ragged random matrices spanning many compaction blocks (1024 rows) with a
    ragged tail, and the edge cases (one row, all-empty rows, thresholds 31/32 and 255/256)."""
    rng = np.random.default_rng(21)
    cases = {"rmat": lbgen.rmat(14, 16, 5, "int"), "skewed": lbgen.skewed(1 << 13, 7, 5000, 90_000, 8, "int"),
             "stencil": lbgen.stencil(90, 2, "int"), "random": random_csr(rng, 5000, 700, 700, 0.4, "int"),
             "one_row": _csr([0, 300], 5), "empty_rows": _csr([0] * 2050, 4),
             "thresholds": _csr([0, 31, 63, 318, 574, 574], 9)}
    for name, A in cases.items():
        _check_bins(A, name)


@pytest.mark.parametrize("cfg", ["c3", "c4"])
def test_bins_full_size(cfg):
    """The bins at BASELINE.json sizes (C3: all three bins populated; C4: the 1,000 giant rows)."""
    torch.cuda.empty_cache()
    A = lbgen.make_config(cfg, "int", device="cuda")
    _check_bins(A, cfg)
    del A
    torch.cuda.empty_cache()


# ---------------------------------------------------------------- AUTO schedule (P:1149 + reading R18)

def test_auto_schedule_selection_and_parity():
    cases = {
        "tiny (alpha/beta rule)": (_csr(list(range(0, 401)), 300), "thread_mapped"),
        "stencil (regular rows)": (lbgen.stencil(120, 2, "int"), "thread_mapped"),
        "rmat (power law)": (lbgen.rmat(13, 16, 5, "int"), "merge_path"),
        "skewed (giant rows)": (lbgen.skewed(1 << 12, 3, 30_000, 20_000, 8, "int"), "merge_path"),
    }
    for name, (A, want) in cases.items():
        M = lb.CsrMatrix.from_csr(A)
        assert M.select_schedule() == want, name
        x = lbgen.make_x(A.cols, "int", 2)
        y_ref, s_ref = ref(A, x)
        check_y(M.spmv(x.cuda(), schedule="auto"), y_ref, s_ref, True, name)


# ---------------------------------------------------------------- SpMM (NEXT-2)

def check_Y(Y_gpu, Y_ref, S_ref, exact, what=""):
    Y = Y_gpu.detach().double().cpu().numpy()
    assert Y.shape == Y_ref.shape
    if exact:
        bad = np.argwhere(Y != Y_ref)
        assert bad.size == 0, f"{what}: {len(bad)} entries differ, first {bad[:3].tolist()}"
    else:
        err = np.abs(Y - Y_ref)
        assert np.all(err <= TOL * S_ref + 1e-30), f"{what}: worst rel {np.max(err / (S_ref + 1e-30)):.3e}"


@pytest.mark.parametrize("kernel", ["default", "lanes"])
@pytest.mark.parametrize("n", [1, 3, 4, 5, 8, 16, 24, 32, 45])
@pytest.mark.parametrize("name", ["rmat12", "stencil100", "skewed", "c1"])
def test_spmm_parity(name, n, kernel, monkeypatch):
    """Both SpMM tile processors: lanes over columns (merge_spmm_cols_kernel, panels of 32/16) and
    lanes over nonzeros (merge_spmm_kernel: panels of 8/4/1; every panel with LB_SPMM=lanes)."""
    if kernel != "default":
        monkeypatch.setenv("LB_SPMM", kernel)
    for vm in ("int", "float"):
        A = SMALL[name](vm)
        X = lbgen.make_x(A.cols * n, vm, 21).reshape(A.cols, n)
        Y_ref, S_ref = oracle.spmm(A.row_offsets, A.col_idx, A.values, X)
        M = lb.CsrMatrix.from_csr(A)
        Y = M.spmm(X.cuda())
        torch.cuda.synchronize()
        check_Y(Y, Y_ref, S_ref, vm == "int", f"{name}/n={n}/{vm}")


def test_spmm_strided_and_edge_cases():
    A = lbgen.rmat(11, 16, 4, "int")
    Xbig = lbgen.make_x(A.cols * 7, "int", 3).reshape(A.cols, 7).cuda()
    X = Xbig[:, 1:6]                     # ldx = 7, misaligned base: scalar-column path
    Y_ref, S_ref = oracle.spmm(A.row_offsets, A.col_idx, A.values, X.cpu().contiguous())
    M = lb.CsrMatrix.from_csr(A)
    check_Y(M.spmm(X), Y_ref, S_ref, True, "strided")
    # ldx = 16 with panels starting at columns 0 and 8 (8-column panels) and at 4 (misaligned for 8:
    # a 4-column panel first), plus a 13-column view: 8 + 4 + 1
    X16 = lbgen.make_x(A.cols * 16, "int", 4).reshape(A.cols, 16).cuda()
    for lo, hi in ((0, 16), (4, 16), (0, 13), (8, 16)):
        Xv = X16[:, lo:hi]
        Y_ref, S_ref = oracle.spmm(A.row_offsets, A.col_idx, A.values, Xv.cpu().contiguous())
        check_Y(M.spmm(Xv), Y_ref, S_ref, True, f"ldx16[{lo}:{hi}]")
    for nm, B in {"giant": _csr([0, 50_001], 1), "no_nnz": _csr([0] * 2001, 3),
                  "golden": _csr([0, 1, 3, 3, 6], 1),
                  "giant_mid": _csr([0, 0, 3, 40_003, 40_003, 40_010] + [40_010] * 700, 5),
                  "empty_runs": _csr([0] + [0] * 3000 + [2] + [2] * 5000 + [9], 7)}.items():
        for n in (4, 8, 16, 32):
            X = lbgen.make_x(B.cols * n, "int", 9).reshape(B.cols, n)
            Y_ref, S_ref = oracle.spmm(B.row_offsets, B.col_idx, B.values, X)
            for mode in ("default", "lanes"):
                if mode == "lanes":
                    os.environ["LB_SPMM"] = "lanes"
                try:
                    check_Y(lb.CsrMatrix.from_csr(B).spmm(X.cuda()), Y_ref, S_ref, True, f"{nm}/n={n}/{mode}")
                finally:
                    os.environ.pop("LB_SPMM", None)
    # Y with a leading dimension (ldy = 40) and a misaligned Y view (Y + 1: scalar fallback panels)
    X = lbgen.make_x(A.cols * 32, "int", 10).reshape(A.cols, 32).cuda()
    Y_ref, S_ref = oracle.spmm(A.row_offsets, A.col_idx, A.values, X.cpu())
    for off in (0, 1, 4):
        Ybig = torch.full((A.rows, 40), 7.0, device="cuda")
        Yv = Ybig[:, off:off + 32]
        M.spmm(X, Yv)
        check_Y(Yv, Y_ref, S_ref, True, f"ldy40+{off}")
        assert torch.all(Ybig[:, :off] == 7.0) and torch.all(Ybig[:, off + 32:] == 7.0), "wrote outside the view"
    # SpMM column j equals SpMV with x = X[:, j] (same tiles, same arithmetic per column)
    A = lbgen.rmat(12, 16, 8, "float")
    X = lbgen.make_x(A.cols * 4, "float", 5).reshape(A.cols, 4).cuda()
    M = lb.CsrMatrix.from_csr(A)
    Y = M.spmm(X)
    Y_ref, S_ref = oracle.spmm(A.row_offsets, A.col_idx, A.values, X.cpu())
    check_Y(Y, Y_ref, S_ref, False, "float n=4")


@pytest.mark.parametrize("cfg,n", [("c3", 4), ("c4", 4), ("c3", 8), ("c3", 16), ("c4", 32)])
def test_spmm_full_size(cfg, n):
    """Full-size SpMM: 4-column panels, and an 8-column panel (one 256-bit gather per nonzero)."""
    torch.cuda.empty_cache()
    A = lbgen.make_config(cfg, "int", device="cuda")
    X = lbgen.make_x(A.cols * n, "int", 77, device="cuda").reshape(A.cols, n)
    M = lb.CsrMatrix.from_csr(A)
    Y = M.spmm(X)
    torch.cuda.synchronize()
    Yh = Y.cpu()
    for j in range(n):   # column by column through the oracle SpMV (exact in integer mode)
        y_ref, s_ref = oracle.spmv(A.row_offsets.cpu(), A.col_idx.cpu(), A.values.cpu(), X[:, j].cpu(), threads=True)
        check_y(Yh[:, j], y_ref, s_ref, True, f"{cfg} col {j}")
    del M, A, X, Y
    torch.cuda.empty_cache()



# ---------------------------------------------------------------- nonzero-split partition (NEXT-3)

@pytest.mark.parametrize("L", [1, 3, 64, 1016])
@pytest.mark.parametrize("name", ["rmat12", "stencil100", "skewed", "c1"])
def test_partition_nz_bit_exact(name, L):
    A = SMALL[name]("int")
    M = lb.CsrMatrix.from_csr(A)
    assert np.array_equal(M.partition_nz(L).cpu().numpy(), oracle.partition_nz(A.row_offsets, L))


def test_nonzero_split_many_empty_rows():
    """Tiles spanning >65535 empty rows (32-bit row ids) and long empty runs between nonzeros."""
    rows = 200_000
    lens = np.zeros(rows, np.int64)
    lens[[5, 70_000, 70_001, 150_000, rows - 1]] = [3, 2000, 1, 5, 7]
    off = np.zeros(rows + 1, np.int64)
    off[1:] = np.cumsum(lens)
    A = _csr(off.tolist(), 4, col=[0] * int(off[-1]), val=[1.0] * int(off[-1]))
    x = torch.ones(4)
    y_ref, s_ref = ref(A, x)
    for sched in ("nonzero_split", "merge_path"):
        check_y(run(A, x, sched), y_ref, s_ref, True, sched)


# ---------------------------------------------------------------- CUDA graph capture

@pytest.mark.parametrize("sched", SCHEDS)
def test_cuda_graph_capture_and_replay(sched):
    """lb_spmv_ex(REPARTITION) is stream-ordered with handle-owned scratch, so after one warm-up call (first
    use allocates lazy workspaces / sets kernel attributes) it can be captured into a CUDA graph; every
    replay with a new x (copied into the captured buffer) is bit-exact against the oracle in integer mode."""
    A = lbgen.rmat(13, 16, 7, "int")
    M = lb.CsrMatrix.from_csr(A)
    if sched == "merge_path":
        M.plan_hot_x(256, 0)  # the planned tile kernel + the fused partition / x_hot gather launch
    xs = [lbgen.make_x(A.cols, "int", s) for s in (11, 12, 13)]
    x = xs[0].cuda().clone()
    y = torch.full((A.rows,), float("nan"), device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        M.spmv(x, y, sched, repartition=True, stream=s)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        M.spmv(x, y, sched, repartition=True)
    for xi in xs:
        x.copy_(xi.cuda())
        y.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        y_ref, s_ref = ref(A, xi)
        check_y(y, y_ref, s_ref, True, f"graph/{sched}")


# ---------------------------------------------------------------- the int32 / int64 limits

def test_maximum_size_merge_items():
    """The largest problem the API accepts, rows + nnz = 2^31 - 2^16 - 1 (nnz = 2^30, ragged rows, a third
    of them empty, a 200,001-nonzero row and a ~65K-nonzero last row): the partition is bit-exact on every
    tile (brute-force oracle over all merge items) and y is bit-exact (integer mode) on sampled rows for the
    merge-path, nonzero-split and binning schedules; one more merge item is rejected."""
    torch.cuda.empty_cache()
    A = lbgen.max_size(31, "int", device="cuda")
    assert A.rows + A.nnz == lbgen.MAX_MERGE_ITEMS
    h = ctypes.c_void_p()  # shape checks come before any access to the arrays
    st = lb.lib().lb_csr_create(A.rows + 1, A.cols, A.nnz, A.row_offsets.data_ptr(), A.col_idx.data_ptr(),
                                A.values.data_ptr(), 0, None, ctypes.byref(h))
    assert st == lb.lb.LB_ERR_INVALID_ARG and not h
    x = lbgen.make_x(A.cols, "int", 8, device="cuda")
    M = lb.CsrMatrix.from_csr(A, device="cuda", validate=True)
    coords = M.partition().cpu().numpy()
    assert coords[-1].tolist() == [A.rows, A.nnz]
    assert np.array_equal(coords, oracle.partition(A.row_offsets.cpu(), M.items_per_tile)), "partition"
    sel = _sample_rows(A, coords, 20_000, 3)
    so, sc, sv = _packed(A, sel)
    y_ref, s_ref = oracle.spmv_packed(so, sc, sv, x.cpu())
    sel_d = torch.as_tensor(sel, device="cuda")
    for sched in ("merge_path", "nonzero_split", "binning"):
        y = torch.full((A.rows,), float("nan"), device="cuda")
        M.spmv(x, y, sched, repartition=True)
        torch.cuda.synchronize()
        check_y(y[sel_d], y_ref, s_ref, True, f"max_size/{sched}")
        del y
    del M, A, x
    torch.cuda.empty_cache()
