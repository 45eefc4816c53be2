"""Pins for the CPU oracle (-m "not gpu").

The oracle (oracle/) is checked against things other than itself: hand-derived worked
examples (tests/golden/, cited), independent derivations of the merge-path coordinate
(closed-form count and a CUB-style binary search), dense brute force, closed forms
(identity, diagonal, stencil), row sums, and the partition invariants of SURVEY.md 8(c) p2.
A plausible mistake in the oracle -- a dropped term, a wrong tie-break, an off-by-one in
the diagonal, a transposed operand -- fails at least one of these.
"""
import json
import os

import numpy as np
import pytest
import torch

import lbgen
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "merge_path_examples.json")


# ---------------------------------------------------------------- independent derivations

def coord_closed_form(off: np.ndarray, d: int) -> tuple[int, int]:
    """i(d) = #{k < rows : k + off[k+1] < d}: row end k sits at merge position k + off[k+1]."""
    rows = off.size - 1
    pos = np.arange(rows, dtype=np.int64) + off[1:].astype(np.int64)
    i = int(np.count_nonzero(pos < d))
    return i, d - i


def coord_binary_search(off: list[int], d: int) -> tuple[int, int]:
    """CUB-style merge-path search along diagonal d: go right iff off[p+1] <= d - p - 1."""
    rows = len(off) - 1
    nnz = off[-1]
    lo, hi = max(0, d - nnz), min(d, rows)
    while lo < hi:
        p = (lo + hi) // 2
        if off[p + 1] <= d - p - 1:
            lo = p + 1
        else:
            hi = p
    return lo, d - lo


def dense_spmv(A: lbgen.Csr, x: torch.Tensor) -> np.ndarray:
    """Densify (summing duplicates) and multiply in float64 with numpy's matmul."""
    D = np.zeros((A.rows, A.cols), np.float64)
    off = A.row_offsets.numpy().astype(np.int64)
    r = np.repeat(np.arange(A.rows), np.diff(off))
    np.add.at(D, (r, A.col_idx.numpy()), A.values.numpy().astype(np.float64))
    return D @ x.numpy().astype(np.float64)


def random_csr(rng: np.random.Generator, rows: int, cols: int, max_len: int, p_empty: float,
               vmode: str) -> lbgen.Csr:
    lens = rng.integers(0, max_len + 1, rows)
    lens[rng.random(rows) < p_empty] = 0
    off = np.zeros(rows + 1, np.int64)
    off[1:] = np.cumsum(lens)
    nnz = int(off[-1])
    col = rng.integers(0, max(cols, 1), nnz)
    for i in range(rows):  # sorted columns per row (duplicates allowed)
        col[off[i]:off[i + 1]].sort()
    if vmode == "int":
        val = rng.choice([-2.0, -1.0, 1.0, 2.0], nnz)
    else:
        val = (rng.integers(-(1 << 23), 1 << 23, nnz) * 2.0 ** -23)
    return lbgen.Csr(rows, cols, torch.tensor(off, dtype=torch.int32), torch.tensor(col, dtype=torch.int32),
                     torch.tensor(val, dtype=torch.float32))


# ---------------------------------------------------------------- partition pins

def test_partition_golden_examples():
    ex = json.load(open(GOLDEN))["examples"]
    for e in ex:
        got = oracle.partition(np.array(e["off"], np.int32), e["L"])
        assert got.tolist() == e["coords"], e
        # diagonal identity i + j = d_t
        assert [int(a + b) for a, b in got] == e["diagonals"]


def test_partition_three_derivations_agree_every_diagonal():
    """two-pointer oracle == closed form == binary search on every diagonal."""
    rng = np.random.default_rng(7)
    for trial in range(300):
        rows = int(rng.integers(0, 60))
        A = random_csr(rng, rows, 50, int(rng.integers(0, 12)), float(rng.random()), "int")
        off = A.row_offsets.numpy()
        coords = oracle.partition(off, 1)  # L = 1: every diagonal 0..rows+nnz
        total = rows + A.nnz
        assert coords.shape == (total + 1, 2)
        offl = off.tolist()
        for d in range(total + 1):
            cf = coord_closed_form(off, d)
            bs = coord_binary_search(offl, d)
            assert tuple(coords[d]) == cf == bs, (trial, d)


def test_partition_large_random_against_closed_form():
    rng = np.random.default_rng(11)
    A = random_csr(rng, 3000, 100, 9, 0.3, "int")
    off = A.row_offsets.numpy()
    for L in (1, 2, 3, 7, 64, 255, 2048, 10 ** 6):
        c = oracle.partition(off, L)
        total = A.rows + A.nnz
        for t in range(c.shape[0]):
            d = min(t * L, total)
            assert tuple(c[t]) == coord_closed_form(off, d)


def check_partition_invariants(off: np.ndarray, L: int, coords: np.ndarray):
    """SURVEY 8(c) p2 (must also hold bit-exactly on GPU output)."""
    rows = off.size - 1
    nnz = int(off[-1]) if rows else 0
    total = rows + nnz
    T = (total + L - 1) // L
    assert coords.shape == (T + 1, 2)
    assert tuple(coords[0]) == (0, 0) and tuple(coords[-1]) == (rows, nnz)
    d = np.minimum(np.arange(T + 1, dtype=np.int64) * L, total)
    assert np.array_equal(coords[:, 0].astype(np.int64) + coords[:, 1], d)
    assert np.all(np.diff(coords[:, 0]) >= 0) and np.all(np.diff(coords[:, 1]) >= 0)
    i, j = coords[:, 0].astype(np.int64), coords[:, 1].astype(np.int64)
    inner = i < rows
    assert np.all(off[i[inner]] <= j[inner]) and np.all(j[inner] <= off[i[inner] + 1])
    assert np.all(j[~inner] == nnz)
    if T > 1:
        assert np.all(np.diff(d)[:-1] == L)


@pytest.mark.parametrize("gen", ["rmat", "stencil", "skewed", "uniform"])
@pytest.mark.parametrize("L", [1, 5, 256, 2048])
def test_partition_invariants_on_generators(gen, L):
    A = {"rmat": lambda: lbgen.rmat(10, 8, 3, "int"),
         "stencil": lambda: lbgen.stencil(20, 2, "stencil"),
         "skewed": lambda: lbgen.skewed(1 << 10, 4, 3000, 5000, 4, "int"),
         "uniform": lambda: lbgen.make_config("c1", "int")}[gen]()
    off = A.row_offsets.numpy()
    check_partition_invariants(off, L, oracle.partition(off, L))


def test_partition_edge_cases():
    # empty matrix
    c = oracle.partition(np.array([0], np.int32), 8)
    assert c.tolist() == [[0, 0]]
    # rows but no nonzeros: every item is a row end
    c = oracle.partition(np.zeros(6, np.int32), 2)
    assert c.tolist() == [[0, 0], [2, 0], [4, 0], [5, 0]]
    # one giant row
    c = oracle.partition(np.array([0, 10], np.int32), 4)
    assert c.tolist() == [[0, 0], [0, 4], [0, 8], [1, 10]]


# ---------------------------------------------------------------- SpMV pins

@pytest.mark.parametrize("vmode", ["int", "float"])
def test_spmv_dense_brute_force(vmode):
    """equals dense brute force (exact: products of 24-bit-grid values are exact
    in double and the sums of <= 64 such terms stay within 53 bits)."""
    rng = np.random.default_rng(3)
    for trial in range(200):
        rows = int(rng.integers(0, 40))
        cols = int(rng.integers(1, 40))
        A = random_csr(rng, rows, cols, int(rng.integers(0, 20)), float(rng.random() * 0.5), vmode)
        x = lbgen.make_x(cols, vmode, trial)
        y, s = oracle.spmv(A.row_offsets, A.col_idx, A.values, x)
        yd = dense_spmv(A, x)
        assert np.array_equal(y, yd), trial
        assert np.all(s >= np.abs(y))


def test_spmv_golden_ones():
    for e in json.load(open(GOLDEN))["examples"]:
        off = np.array(e["off"], np.int32)
        nnz = int(off[-1])
        y, s = oracle.spmv(off, np.zeros(nnz, np.int32), np.ones(nnz, np.float32), np.ones(1, np.float32))
        assert y.tolist() == e["ones_y"]
        assert s.tolist() == e["ones_y"]


def test_spmv_identity_and_diagonal_closed_forms():
    n = 257
    off = np.arange(n + 1, dtype=np.int32)
    col = np.arange(n, dtype=np.int32)
    x = lbgen.make_x(n, "float", 5).numpy()
    y, _ = oracle.spmv(off, col, np.ones(n, np.float32), x)
    assert np.array_equal(y, x.astype(np.float64))          # identity: y = x
    d = lbgen.make_x(n, "float", 6).numpy()
    y, s = oracle.spmv(off, col, d, x)
    assert np.array_equal(y, d.astype(np.float64) * x.astype(np.float64))  # diagonal: y_i = d_i x_i
    assert np.array_equal(s, np.abs(y))


def test_spmv_row_sums_with_ones():
    """with x = 1, y_i = sum of row i's values (bincount formulation)."""
    A = lbgen.rmat(11, 8, 9, "int")
    off = A.row_offsets.numpy().astype(np.int64)
    rid = np.repeat(np.arange(A.rows), np.diff(off))
    expect = np.bincount(rid, weights=A.values.numpy().astype(np.float64), minlength=A.rows)
    y, _ = oracle.spmv(A.row_offsets, A.col_idx, A.values, np.ones(A.cols, np.float32))
    assert np.array_equal(y, expect)


def stencil_closed_form(N: int, xmode: str) -> np.ndarray:
    """5-point stencil (4 on the diagonal, -1 per present neighbour).
    x = 1:        y_i = 4 - #present neighbours  (0 interior, 1 edge, 2 corner)
    x_i = i:      y_i = 4 i - sum(present j) = sum of the MISSING neighbour indices."""
    i = np.arange(N * N, dtype=np.int64)
    yy, xx = i // N, i % N
    missing = [(yy == 0, i - N), (xx == 0, i - 1), (xx == N - 1, i + 1), (yy == N - 1, i + N)]
    if xmode == "ones":
        return sum(m.astype(np.float64) for m, _ in missing)
    return sum(np.where(m, v, 0).astype(np.float64) for m, v in missing)


@pytest.mark.parametrize("xmode", ["ones", "index"])
def test_spmv_stencil_closed_form(xmode):
    N = 64
    A = lbgen.stencil(N, 2, "stencil")
    x = lbgen.make_x(N * N, xmode, 0)
    y, _ = oracle.spmv(A.row_offsets, A.col_idx, A.values, x)
    expect = stencil_closed_form(N, xmode)
    assert np.array_equal(y, expect)
    if xmode == "index":
        assert y[0] == -(N + 1) and y[N - 1] == N - 1 and y[N * N - 1] == 2 * (N * N - 1) + 1 + N


def test_spmv_omp_matches_serial():
    A = lbgen.rmat(12, 8, 4, "float")
    x = lbgen.make_x(A.cols, "float", 1)
    y1, s1 = oracle.spmv(A.row_offsets, A.col_idx, A.values, x)
    y2, s2 = oracle.spmv(A.row_offsets, A.col_idx, A.values, x, threads=True)
    assert np.array_equal(y1, y2) and np.array_equal(s1, s2)


def test_spmv_packed_matches_full():
    A = lbgen.rmat(10, 8, 5, "float")
    x = lbgen.make_x(A.cols, "float", 2)
    y, s = oracle.spmv(A.row_offsets, A.col_idx, A.values, x)
    sel = np.array([0, 5, 17, 1023, 500])
    off = A.row_offsets.numpy().astype(np.int64)
    lens = off[sel + 1] - off[sel]
    so = np.zeros(sel.size + 1, np.int64)
    so[1:] = np.cumsum(lens)
    idx = np.concatenate([np.arange(off[r], off[r + 1]) for r in sel])
    yp, sp = oracle.spmv_packed(so, A.col_idx.numpy()[idx], A.values.numpy()[idx], x)
    assert np.array_equal(yp, y[sel]) and np.array_equal(sp, s[sel])


# ---------------------------------------------------------------- Alg.3 executable check

def alg3_tiles_then_fixup(off, col, val, x, L):
    """Pure-Python Alg.3 with the DESIGN.md readings R2-R5: walk each tile's merge
    items from its coordinates, write y[row] at row ends, emit a carry at tile end, then fix up.
    Checks that tile walk + fix-up reproduces y = A x (the decomposition the kernels use)."""
    coords = oracle.partition(off, L)
    rows = off.size - 1
    y = np.zeros(rows)
    carries = []
    for t in range(coords.shape[0] - 1):
        (i, j), (i1, j1) = coords[t], coords[t + 1]
        acc = 0.0
        while i < i1 or j < j1:
            if i < i1 and off[i + 1] <= j:
                y[i] = acc
                acc = 0.0
                i += 1
            else:
                acc += float(val[j]) * float(x[col[j]])
                j += 1
        carries.append((int(i1), acc))
    for r, v in carries:
        if r < rows:
            y[r] += v
    return y


@pytest.mark.parametrize("L", [1, 2, 3, 16, 100])
def test_alg3_decomposition_reproduces_oracle(L):
    rng = np.random.default_rng(L)
    for trial in range(30):
        A = random_csr(rng, int(rng.integers(0, 50)), 30, int(rng.integers(0, 25)), 0.3, "int")
        x = lbgen.make_x(30, "int", trial).numpy()
        off = A.row_offsets.numpy()
        y_ref, _ = oracle.spmv(off, A.col_idx, A.values, x)
        y = alg3_tiles_then_fixup(off, A.col_idx.numpy(), A.values.numpy(), x, L)
        assert np.array_equal(y, y_ref)


def test_alg3_golden_trace():
    e = json.load(open(GOLDEN))["examples"][0]
    off = np.array(e["off"], np.int32)
    y = alg3_tiles_then_fixup(off, np.zeros(6, np.int32), np.ones(6, np.float32), np.ones(1, np.float32), 2)
    assert y.tolist() == e["ones_y"]


# ---------------------------------------------------------------- shard bounds

@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_shard_bounds(G):
    for A in (lbgen.rmat(11, 8, 1, "ones"), lbgen.skewed(1 << 11, 3, 4000, 9000, 2, "ones"),
              lbgen.stencil(30, 2, "stencil"), lbgen.Csr(0, 0, torch.zeros(1, dtype=torch.int32),
                                                         torch.zeros(0, dtype=torch.int32),
                                                         torch.zeros(0))):
        off = A.row_offsets.numpy().astype(np.int64)
        b = oracle.shard_bounds(A.row_offsets, G)
        nnz = int(off[-1])
        targets = [-(-g * nnz // G) for g in range(G + 1)]
        expect = [int(np.searchsorted(off, t, side="left")) for t in targets]  # first r with off[r] >= t
        expect[0], expect[G] = 0, A.rows
        assert b.tolist() == expect
        assert np.all(np.diff(b) >= 0)
        maxrow = int(np.diff(off).max()) if A.rows else 0
        per = off[b[1:]] - off[b[:-1]]
        assert per.sum() == nnz
        assert np.all(per <= -(-nnz // G) + maxrow)


# ---------------------------------------------------------------- SpMM (NEXT-2) pins

@pytest.mark.parametrize("n", [1, 3, 4, 8])
def test_spmm_dense_brute_force(n):
    """Y = A X equals the dense product (numpy matmul after densifying) exactly."""
    rng = np.random.default_rng(n)
    for trial in range(60):
        rows, cols = int(rng.integers(0, 30)), int(rng.integers(1, 30))
        A = random_csr(rng, rows, cols, int(rng.integers(0, 15)), 0.3, "float")
        X = (rng.integers(-(1 << 23), 1 << 23, (cols, n)) * 2.0 ** -23).astype(np.float32)
        Y, S = oracle.spmm(A.row_offsets, A.col_idx, A.values, X)
        D = np.zeros((rows, cols))
        off = A.row_offsets.numpy().astype(np.int64)
        np.add.at(D, (np.repeat(np.arange(rows), np.diff(off)), A.col_idx.numpy()), A.values.numpy().astype(np.float64))
        assert np.array_equal(Y, D @ X.astype(np.float64)), trial
        assert np.all(S >= np.abs(Y))


def test_spmm_identity_closed_form():
    n = 100
    off = np.arange(n + 1, dtype=np.int32)
    X = lbgen.make_x(n * 5, "float", 3).numpy().reshape(n, 5)
    Y, _ = oracle.spmm(off, np.arange(n, dtype=np.int32), np.ones(n, np.float32), X)
    assert np.array_equal(Y, X.astype(np.float64))


# ---------------------------------------------------------------- nonzero-split (NEXT-3) pins

def test_partition_nz_worked_example_and_merge_path_points():
    """Hand-derived: off = [0,1,3,3,6], L = 2 -> j = 0,2,4,6; rows ending at or before j:
    j=2 -> rows 0 (end 1); j=4 -> rows 0,1,2 (ends 1,3,3); last = (4, 6)."""
    c = oracle.partition_nz(np.array([0, 1, 3, 3, 6], np.int32), 2)
    assert c.tolist() == [[0, 0], [1, 2], [3, 4], [4, 6]]
    # every nonzero-split coordinate is a point on the merge path: off[i] <= j <= off[i+1] for i < rows
    rng = np.random.default_rng(4)
    for trial in range(200):
        A = random_csr(rng, int(rng.integers(0, 60)), 20, int(rng.integers(0, 9)), float(rng.random()), "int")
        off = A.row_offsets.numpy().astype(np.int64)
        for L in (1, 3, 16):
            c = oracle.partition_nz(A.row_offsets, L).astype(np.int64)
            i, j = c[:, 0], c[:, 1]
            assert tuple(c[0]) == (0, 0) and tuple(c[-1]) == (A.rows, A.nnz)
            assert np.all(np.diff(i) >= 0) and np.all(np.diff(j) >= 0)
            assert np.all(np.diff(j)[:-1] == L) if c.shape[0] > 2 else True
            inner = i < A.rows
            assert np.all(off[i[inner]] <= j[inner]) and np.all(j[inner] <= off[i[inner] + 1])
            # i_t (0 < t < T) is the closed-form count #{r : off[r+1] <= j_t}
            for t in range(1, c.shape[0] - 1):
                assert i[t] == np.count_nonzero(off[1:] <= j[t])


# ---------------------------------------------------------------- hot-column plan

HOT_GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "hot_columns_examples.json")


def hot_slot_table_by_sort(deg: np.ndarray, slots: int) -> np.ndarray:
    """Slot table of the plan from column degrees: lexsort (the oracle uses repeated maximum search)."""
    cand = np.nonzero(deg >= 2)[0]
    if cand.size < slots:
        return cand.astype(np.int32)
    order = np.lexsort((cand, -deg[cand]))  # deg descending, then column ascending
    hot = np.sort(cand[order[:slots]])
    tau = deg[hot].min()
    return np.concatenate([hot[deg[hot] > tau], hot[deg[hot] == tau]]).astype(np.int32)


def warm_table_by_levels(deg: np.ndarray, slot_cols: np.ndarray, slots: int, warm: int) -> np.ndarray:
    """Warm tier from degrees: whole degree levels via a sorted degree array (the oracle scans levels)."""
    cand = np.nonzero(deg >= 2)[0]
    if warm <= 0 or cand.size < slots or slot_cols.size == 0:
        return np.zeros(0, np.int32)
    tau1 = deg[slot_cols].min()
    ds = np.sort(deg[cand])[::-1]  # descending
    k = slots + warm
    # smallest d >= 2 with #{deg >= d} <= k: the level just above position k in the sorted list
    tau2 = 2 if ds.size <= k else int(ds[k]) + 1
    if tau2 > tau1:
        return np.zeros(0, np.int32)
    hot = np.zeros(deg.size, bool)
    hot[slot_cols] = True
    return np.nonzero(~hot & (deg >= tau2))[0].astype(np.int32)


def hot_columns_by_sort(col: np.ndarray, cols: int, slots: int, warm: int = 0):
    """Independent derivation of the plan: bincount + lexsort + sorted degree levels."""
    deg = np.bincount(col, minlength=cols).astype(np.int64) if col.size else np.zeros(cols, np.int64)
    slot_cols = hot_slot_table_by_sort(deg, slots)
    warm_cols = warm_table_by_levels(deg, slot_cols, slots, warm)
    tier = np.full(cols, -1, np.int64)
    tier[slot_cols] = np.arange(slot_cols.size)
    tier[warm_cols] = slot_cols.size + np.arange(warm_cols.size)
    t = tier[col] if col.size else np.zeros(0, np.int64)
    remapped = np.where(t < 0, col, np.where(t < slot_cols.size, ~t, cols + t - slot_cols.size)).astype(np.int32)
    return slot_cols, warm_cols, remapped, int(deg[slot_cols].sum()), int(deg[warm_cols].sum())


def test_hot_columns_worked_examples():
    g = json.load(open(HOT_GOLDEN))
    col = np.array(g["col_idx"], np.int32)
    for case in g["cases"]:
        sc, rm, hn = oracle.hot_columns(col, g["cols"], case["slots"])
        assert sc.tolist() == case["slot_cols"], case
        assert hn == case["hot_nnz"], case
        slot_of = {c: i for i, c in enumerate(case["slot_cols"])}
        assert rm.tolist() == [~slot_of[c] if c in slot_of else c for c in g["col_idx"]]
    w = g["warm"]
    for case in w["cases"]:
        sc, wc, rm, hn, wn = oracle.x_plan(w["col_idx"], w["cols"], case["slots"], case["warm"])
        assert sc.tolist() == case["slot_cols"] and wc.tolist() == case["warm_cols"], case
        assert (hn, wn) == (case["hot_nnz"], case["warm_nnz"]), case
        slot_of = {c: i for i, c in enumerate(case["slot_cols"])}
        warm_of = {c: i for i, c in enumerate(case["warm_cols"])}
        assert rm.tolist() == [~slot_of[c] if c in slot_of else (w["cols"] + warm_of[c] if c in warm_of else c)
                               for c in w["col_idx"]], case


@pytest.mark.parametrize("seed", range(40))
def test_hot_columns_match_sort_derivation(seed):
    rng = np.random.default_rng(seed)
    cols = int(rng.integers(1, 400))
    nnz = int(rng.integers(0, 3000))
    # skewed column popularity (power-law-ish) with many ties
    w = rng.pareto(1.2, cols) + 0.05
    col = rng.choice(cols, size=nnz, p=w / w.sum()).astype(np.int32)
    for slots in (1, 2, 7, int(rng.integers(1, cols + 5)), cols + 10):
        for warm in (0, 1, int(rng.integers(1, cols + 5)), 10 * cols):
            sc, wc, rm, hn, wn = oracle.x_plan(col, cols, slots, warm)
            sc2, wc2, rm2, hn2, wn2 = hot_columns_by_sort(col, cols, slots, warm)
            assert np.array_equal(sc, sc2), (seed, slots, warm)
            assert np.array_equal(wc, wc2), (seed, slots, warm)
            assert np.array_equal(rm, rm2), (seed, slots, warm)
            assert (hn, wn) == (hn2, wn2)
            # invariants: hot columns are at least as popular as warm ones, warm ones at least as
            # popular as the remaining candidates; the warm tier respects its budget; decoding the
            # remapped stream through the tables gives col_idx back
            deg = np.bincount(col, minlength=cols)
            rest = np.ones(cols, bool)
            rest[sc] = False
            rest[wc] = False
            rest &= deg >= 2
            if sc.size and wc.size:
                assert deg[sc].min() >= deg[wc].max()
            if wc.size and rest.any():
                assert deg[wc].min() > deg[rest].max()  # whole degree levels
            assert wc.size <= max(warm, 0)
            dec = np.where(rm < 0, sc[np.where(rm < 0, ~rm, 0)] if sc.size else 0,
                           np.where(rm >= cols, wc[np.clip(rm - cols, 0, max(wc.size - 1, 0))] if wc.size else 0, rm))
            assert np.array_equal(dec, col)
            assert sc.size == min(slots, int((deg >= 2).sum()))


# ---------------------------------------------------------------- SSSP (NEXT-4, Listing 5)

SSSP_GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "sssp_examples.json")


def bellman_ford_f32(off, col, w, n, source):
    """Independent derivation: synchronous Bellman-Ford rounds over all edges with fp32 adds until no
    change (the least fixed point of dist[v] = min(dist[v], fl(dist[u] + w)), like Dijkstra's)."""
    dist = np.full(n, np.inf, np.float32)
    dist[source] = 0
    src = np.repeat(np.arange(n), np.diff(off))
    for _ in range(n + 1):
        cand = (dist[src] + w.astype(np.float32)).astype(np.float32)
        new = dist.copy()
        np.minimum.at(new, col, cand)
        if np.array_equal(new, dist):
            return dist
        dist = new
    raise AssertionError("no convergence")


def test_sssp_worked_examples():
    for c in json.load(open(SSSP_GOLDEN))["cases"]:
        got = oracle.sssp(c["off"], c["col"], c["w"], c["source"])
        want = np.array([np.inf if v == "inf" else v for v in c["dist"]], np.float32)
        assert np.array_equal(got, want), c["name"]


def test_sssp_negative_weight_rejected():
    with pytest.raises(ValueError):
        oracle.sssp([0, 1, 1], [1], [-1.0], 0)


@pytest.mark.parametrize("seed", range(30))
def test_sssp_matches_bellman_ford(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 300))
    deg = rng.integers(0, 12, n) * (rng.random(n) < 0.8)
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum(deg)
    col = rng.integers(0, n, int(off[-1])).astype(np.int32)
    w = (rng.random(int(off[-1])) * rng.choice([1.0, 1e-3, 100.0])).astype(np.float32)
    w[rng.random(w.size) < 0.05] = 0.0
    src = int(rng.integers(0, n))
    got = oracle.sssp(off, col, w, src)
    assert np.array_equal(got, bellman_ford_f32(off, col, w, n, src))


def test_sssp_unit_weights_are_bfs_levels():
    A = lbgen.rmat(10, 8, 3, "int")
    off, col = A.row_offsets.numpy(), A.col_idx.numpy()
    n = A.rows
    # BFS by frontier sets (closed form: unit weights -> hop counts)
    level = np.full(n, np.inf, np.float32)
    level[0] = 0
    frontier, d = [0], 0
    while frontier:
        d += 1
        nxt = set()
        for u in frontier:
            for v in col[off[u]:off[u + 1]]:
                if level[v] == np.inf:
                    level[v] = d
                    nxt.add(int(v))
        frontier = sorted(nxt)
    got = oracle.sssp(off, col, np.ones(col.size, np.float32), 0)
    assert np.array_equal(got, level)


# ---------------------------------------------------------------- binning (Alg.4) pins

BIN_GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "binning_examples.json")


def test_bins_worked_examples():
    """Hand-derived bins on both sides of each threshold (tests/golden/binning_examples.json)."""
    with open(BIN_GOLDEN) as f:
        ex = json.load(f)["examples"]
    for e in ex:
        off = np.concatenate([[0], np.cumsum(e["lengths"])]).astype(np.int32)
        cta, warp, thread = oracle.bins(off, e["block_size"], e["warp_size"])
        assert cta.tolist() == e["cta"] and warp.tolist() == e["warp"] and thread.tolist() == e["thread"], e


@pytest.mark.parametrize("gen", ["rmat", "stencil", "skewed", "uniform", "random"])
def test_bins_invariants_and_counts(gen):
    """The bins partition the rows, each bin is ascending, every row satisfies its bin's predicate, and
    the bin sizes equal an independent histogram of the row lengths (np.digitize + bincount)."""
    if gen == "random":
        A = random_csr(np.random.default_rng(5), 3000, 500, 600, 0.3, "int")
    else:
        A = {"rmat": lambda: lbgen.rmat(11, 16, 3, "int"), "stencil": lambda: lbgen.stencil(40, 2, "int"),
             "skewed": lambda: lbgen.skewed(4096, 10, 3000, 60000, 4, "int"),
             "uniform": lambda: lbgen.uniform(500, 0.2, 1, "int")}[gen]()
    off = A.row_offsets.numpy().astype(np.int64)
    lens = np.diff(off)
    cta, warp, thread = oracle.bins(A.row_offsets, 256, 32)
    allr = np.concatenate([cta, warp, thread])
    assert np.array_equal(np.sort(allr), np.arange(A.rows))
    for b in (cta, warp, thread):
        assert np.all(np.diff(b) > 0)
    assert np.all(lens[cta] >= 256) and np.all((lens[warp] >= 32) & (lens[warp] < 256)) and np.all(lens[thread] < 32)
    hist = np.bincount(np.digitize(lens, [32, 256]), minlength=3)  # 0: < 32, 1: [32, 256), 2: >= 256
    assert (thread.size, warp.size, cta.size) == tuple(hist)


def test_bins_closed_forms():
    """Special cases fixed by construction: a stencil's rows (<= 5 nonzeros) are all thread-binned; the
    skewed generator's giant rows (3000 nonzeros) are exactly the CTA bin and its other rows (< 32) the
    thread bin; the identity matrix is all thread bin; an empty matrix has three empty bins."""
    S = lbgen.stencil(30, 2, "int")
    c, w, t = oracle.bins(S.row_offsets)
    assert c.size == 0 and w.size == 0 and np.array_equal(t, np.arange(S.rows))
    K = lbgen.skewed(4096, 10, 3000, 60000, 4, "int")
    lens = np.diff(K.row_offsets.numpy())
    c, w, t = oracle.bins(K.row_offsets)
    assert np.array_equal(c, np.flatnonzero(lens == 3000)) and c.size == 10 and w.size == 0
    assert t.size == K.rows - 10
    c, w, t = oracle.bins(np.arange(65, dtype=np.int32))
    assert c.size == 0 and w.size == 0 and np.array_equal(t, np.arange(64))
    c, w, t = oracle.bins(np.zeros(1, np.int32))
    assert c.size == w.size == t.size == 0
