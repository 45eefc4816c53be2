"""GPU parity of the x-reuse plan (lb_csr_plan_hot_x) through the C ABI.

* the plan (hot slot table, warm table, remapped column stream) is integer work: bit-exact against
  oracle.x_plan (small matrices) or against the test-side sort derivation pinned to the oracle in
  tests/test_oracle_pins.py (full BASELINE.json sizes);
* y with the plan: bit-exact vs the oracle in integer mode, within 1e-5 * s + 1e-30 in float mode,
  and bitwise identical to the merge-path call without a plan (same products, same order).
"""
import numpy as np
import pytest
import torch

import lbgen
import oracle
import paper_2212_08964_b200 as lb
from test_gpu_parity import SMALL, _csr, check_y, random_csr, ref
from test_oracle_pins import hot_columns_by_sort, hot_slot_table_by_sort, warm_table_by_levels

pytestmark = pytest.mark.gpu


def _plan_matches(M: lb.CsrMatrix, A: lbgen.Csr, slots: int, warm: int, ref_fn):
    n, hn = M.plan_hot_x(slots, warm)
    sc, wc, rm, hn_ref, wn_ref = ref_fn(A.col_idx.cpu().numpy(), A.cols, slots, warm)
    info = M.plan_info()
    assert n == sc.size and hn == hn_ref, (n, sc.size, hn, hn_ref)
    assert info["warm_cols"] == wc.size and info["warm_nnz"] == wn_ref
    if n:
        hot, wt, hcol = M.hot_plan()
        assert np.array_equal(hot.cpu().numpy(), sc), "slot table"
        assert np.array_equal(wt.cpu().numpy(), wc), "warm table"
        assert np.array_equal(hcol.cpu().numpy(), rm), "remapped column stream"
    return n


@pytest.mark.parametrize("warm", [0, 1, 100, 5000, 10 ** 7])
@pytest.mark.parametrize("slots", [1, 5, 333, 4096, 32768, 45056])
@pytest.mark.parametrize("name", ["rmat12", "rmat14", "skewed", "c1", "stencil100", "uniform_rows"])
def test_plan_bit_exact(name, slots, warm):
    A = SMALL[name]("int")
    M = lb.CsrMatrix.from_csr(A)
    fn = oracle.x_plan if A.cols * min(slots, A.cols) <= 2e8 else hot_columns_by_sort
    _plan_matches(M, A, slots, warm, fn)


@pytest.mark.parametrize("L", [504, 1016])
@pytest.mark.parametrize("vmode", ["int", "float"])
@pytest.mark.parametrize("name", sorted(SMALL))
def test_spmv_with_plan(name, vmode, L):
    A = SMALL[name](vmode)
    x = lbgen.make_x(A.cols, vmode, 21)
    y_ref, s_ref = ref(A, x)
    M = lb.CsrMatrix.from_csr(A)
    M.set_items_per_tile(L)
    xd = x.cuda()
    y0 = M.spmv(xd, schedule="merge_path", repartition=True).clone()
    for slots, warm in ((7, 0), (2048, 0), (0, 0), (7, 300), (64, 10 ** 6)):
        n, _ = M.plan_hot_x(slots, warm)
        assert n > 0 or name == "stencil100"
        y = torch.full((A.rows,), float("nan"), device="cuda")
        M.spmv(xd, y, "merge_path", repartition=True)
        torch.cuda.synchronize()
        check_y(y, y_ref, s_ref, vmode == "int", f"{name}/{vmode}/L{L}/slots{slots}")
        assert torch.equal(y, y0), "plan changed the bits of y"
        y.fill_(float("nan"))
        M.spmv(xd, y, "merge_path")  # cached partition: x_hot gather alone before the tile kernel
        torch.cuda.synchronize()
        assert torch.equal(y, y0)


@pytest.mark.parametrize("W", ["8", "16"])
def test_plan_kernel_widths(W, monkeypatch):
    monkeypatch.setenv("LB_HOT_W", W)
    rng = np.random.default_rng(int(W))
    for trial in range(8):
        A = random_csr(rng, int(rng.integers(1, 4000)), int(rng.integers(1, 700)), int(rng.integers(0, 80)),
                       float(rng.random()) * 0.6, "int")
        x = lbgen.make_x(A.cols, "int", trial)
        y_ref, s_ref = ref(A, x)
        M = lb.CsrMatrix.from_csr(A)
        M.plan_hot_x(int(rng.integers(1, 600)), int(rng.integers(0, 3000)))
        for L in (504, 1016):
            M.set_items_per_tile(L)
            check_y(M.spmv(x.cuda(), schedule="merge_path"), y_ref, s_ref, True, f"W{W}/trial{trial}/L{L}")


def test_plan_edge_cases():
    # x changes between calls: the hot x values are re-gathered every call
    A = lbgen.rmat(12, 16, 3, "int")
    M = lb.CsrMatrix.from_csr(A)
    assert M.plan_hot_x(1000, 500)[0] == 1000
    assert M.plan_info()["warm_cols"] > 0
    for seed in range(3):
        x = lbgen.make_x(A.cols, "int", 100 + seed)
        y_ref, s_ref = ref(A, x)
        check_y(M.spmv(x.cuda(), schedule="merge_path"), y_ref, s_ref, True, f"x seed {seed}")
    # drop the plan
    assert M.plan_hot_x(-1) == (0, 0)
    assert M.plan_info()["warm_cols"] == 0
    assert M.hot_plan() is None
    assert "hot" not in M.kernel_name("merge_path")
    # no column with two entries: no plan is kept
    D = _csr(list(range(0, 1001)), 1000, col=list(range(1000)))
    MD = lb.CsrMatrix.from_csr(D)
    assert MD.plan_hot_x(0) == (0, 0)
    # one giant row, every column hot
    G = _csr([0, 50_000], 64, col=list(np.arange(50_000) % 64))
    MG = lb.CsrMatrix.from_csr(G)
    assert MG.plan_hot_x(0)[0] == 64
    x = lbgen.make_x(64, "int", 5)
    y_ref, s_ref = ref(G, x)
    check_y(MG.spmv(x.cuda(), schedule="merge_path"), y_ref, s_ref, True, "giant row")
    with pytest.raises(lb.LbError):
        M.plan_hot_x(10 ** 6)


@pytest.mark.parametrize("cfg", ["c3", "c4", "c5"])
def test_plan_full_size(cfg):
    """The plan at BASELINE.json sizes with the default slot budget (what bench.py times): slot table
    and remapped stream bit-exact vs the sort derivation; y bitwise equal to the plan-less
    merge path on every row and within tolerance of the oracle on every row."""
    torch.cuda.empty_cache()
    A = lbgen.make_config(cfg, "float", device="cuda")
    x = lbgen.x_for_config(cfg, A.cols, "float", device="cuda")
    M = lb.CsrMatrix.from_csr(A, device="cuda")
    y0 = M.spmv(x, schedule="merge_path", repartition=True).clone()
    n, hn = M.plan_hot_x(0, -1)  # library defaults: what bench.py times
    info = M.plan_info()
    # tables by the sort derivation (degrees by torch.bincount, test-side), remapped stream checked
    # on the device by decoding it through the tables
    deg = torch.bincount(A.col_idx.long(), minlength=A.cols).cpu().numpy()
    sc = hot_slot_table_by_sort(deg, 16384)  # library default slot budget
    warm_budget = (48 << 20) // 4 if 4 * A.cols > torch.cuda.get_device_properties(0).L2_cache_size else 0
    wc = warm_table_by_levels(deg, sc, 16384, warm_budget)
    assert n == sc.size and hn == int(deg[sc].sum())
    assert info["warm_cols"] == wc.size and info["warm_nnz"] == int(deg[wc].sum())
    hot, wt, hcol = M.hot_plan()
    assert np.array_equal(hot.cpu().numpy(), sc)
    assert np.array_equal(wt.cpu().numpy(), wc)
    table = torch.cat([hot, wt])
    cold = (hcol >= 0) & (hcol < A.cols)
    idx = torch.where(hcol < 0, ~hcol, hcol - A.cols + hot.numel()).clamp(min=0, max=max(table.numel() - 1, 0))
    dec = torch.where(cold, hcol, table[idx.long()])
    assert torch.equal(dec, A.col_idx)
    tier = torch.full((A.cols,), 2, dtype=torch.int8, device="cuda")
    tier[wt.long()] = 1
    tier[hot.long()] = 0
    got_tier = torch.where(hcol < 0, 0, torch.where(hcol >= A.cols, 1, 2)).to(torch.int8)
    assert torch.equal(got_tier, tier[A.col_idx.long()])
    neg = None
    del hcol, dec, neg
    y = torch.full((A.rows,), float("nan"), device="cuda")
    M.spmv(x, y, "merge_path", repartition=True)
    torch.cuda.synchronize()
    assert torch.equal(y, y0)
    y_ref, s_ref = oracle.spmv(A.row_offsets.cpu(), A.col_idx.cpu(), A.values.cpu(), x.cpu(), threads=True)
    check_y(y, y_ref, s_ref, False, f"{cfg}/plan")


def test_probes_diagnostics():
    """lb_probe_stream / lb_probe_stream_gather (bench.py's live ceilings): positive times, the
    stream-only pass no slower than the stream+gather pass by more than noise, argument errors."""
    A = SMALL["rmat14"]("float")
    M = lb.CsrMatrix.from_csr(A, device="cuda")
    x = lbgen.make_x(A.cols, "float", 7).cuda()
    ms_s = M.probe_stream(reps=5)
    ms_g = M.probe_stream_gather(x, reps=5)
    assert ms_s > 0 and ms_g > 0
    with pytest.raises(lb.LbError):
        M.probe_stream(reps=0)
    # empty matrix: valid, nothing to stream
    E = lb.CsrMatrix(4, 4, torch.zeros(5, dtype=torch.int32, device="cuda"),
                     torch.zeros(0, dtype=torch.int32, device="cuda"), torch.zeros(0, device="cuda"))
    try:
        assert E.probe_stream(reps=2) >= 0
    except lb.LbError as e:  # unaligned (null) arrays are reported, not run
        assert "aligned" in str(e)


@pytest.mark.parametrize("scale,cols_trim", [(12, 0), (13, 0), (12, 37), (12, 3)])
def test_compact_plan_matches_oracle(scale, cols_trim):
    """warm_cols = -2 (compact x): every referenced non-hot column is warm, x_warm is built per call
    by mask compaction and the TIER-1 kernel gathers from it.  Integer mode: bit-exact against the
    oracle at both tile lengths, for several x, with cols not a multiple of 4 or 32 (columns >= the
    trimmed width are dropped from the R-MAT matrix), and y bitwise equal to the plan-less call."""
    A = lbgen.rmat(scale, 16, 11, "int")
    if cols_trim:
        keep = A.col_idx < A.cols - cols_trim
        rows_of = torch.repeat_interleave(torch.arange(A.rows), A.row_offsets[1:] - A.row_offsets[:-1])
        cnt = torch.bincount(rows_of[keep], minlength=A.rows)
        off = torch.zeros(A.rows + 1, dtype=torch.int32)
        off[1:] = torch.cumsum(cnt, 0).to(torch.int32)
        A = lbgen.Csr(A.rows, A.cols - cols_trim, off, A.col_idx[keep].contiguous(), A.values[keep].contiguous())
    M = lb.CsrMatrix.from_csr(A)
    hot, _ = M.plan_hot_x(256, -2)
    info = M.plan_info()
    deg = torch.bincount(A.col_idx.long(), minlength=A.cols)
    assert hot == 256 and info["warm_cols"] == int((deg > 0).sum()) - 256
    assert info["hot_nnz"] + info["warm_nnz"] == A.nnz
    P = lb.CsrMatrix.from_csr(A)
    for seed in range(3):
        x = lbgen.make_x(A.cols, "int", 300 + seed)
        y_ref, s_ref = ref(A, x)
        for L in (504, 1016):
            M.set_items_per_tile(L)
            P.set_items_per_tile(L)
            y = M.spmv(x.cuda(), schedule="merge_path", repartition=True)
            check_y(y, y_ref, s_ref, True, f"compact/seed{seed}/L{L}")
            assert torch.equal(y, P.spmv(x.cuda(), schedule="merge_path", repartition=True))
