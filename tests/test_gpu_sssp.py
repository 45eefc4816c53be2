"""GPU parity of SSSP (NEXT-4, lb_sssp, Listing 5) through the C ABI.

Small graphs: bit-exact against oracle.sssp (Dijkstra with fp32 path sums) for every schedule.
Full size (R-MAT scale 24 = C3's structure, weights |value|): a certificate that holds at any size
and characterises the fp32 shortest-path distances exactly -- dist[s] = 0; every edge is feasible,
dist[v] <= fl(dist[u] + w); every vertex with finite distance is reached from s through tight
edges (dist[v] == fl(dist[u] + w)); a feasible d is <= the true distances and a tight path makes it
>=, so together d equals them.
"""
import json
import os

import numpy as np
import pytest
import torch

import lbgen
import oracle
import paper_2212_08964_b200 as lb

pytestmark = pytest.mark.gpu
SCHEDS = ["merge_path", "thread_mapped", "group_mapped"]
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "sssp_examples.json")


def graph(off, col, w, n):
    return lbgen.Csr(n, n, torch.tensor(off, dtype=torch.int32), torch.tensor(col, dtype=torch.int32),
                     torch.tensor(w, dtype=torch.float32))


@pytest.mark.parametrize("sched", SCHEDS)
def test_sssp_worked_examples(sched):
    for c in json.load(open(GOLDEN))["cases"]:
        G = graph(c["off"], c["col"], c["w"], len(c["off"]) - 1)
        d, rounds = lb.CsrMatrix.from_csr(G).sssp(c["source"], sched)
        want = np.array([np.inf if v == "inf" else v for v in c["dist"]], np.float32)
        assert np.array_equal(d.cpu().numpy(), want), (c["name"], sched)


@pytest.mark.parametrize("sched", SCHEDS)
def test_sssp_random_graphs_equal_dijkstra(sched):
    rng = np.random.default_rng(7)
    for trial in range(40):
        n = int(rng.integers(1, 2000))
        deg = rng.integers(0, 20, n) * (rng.random(n) < 0.8)
        if trial % 5 == 0:
            deg[rng.integers(0, n)] = 3000  # a hub: unbalanced frontier
        off = np.zeros(n + 1, np.int64)
        off[1:] = np.cumsum(deg)
        col = rng.integers(0, n, int(off[-1]))
        w = (rng.random(int(off[-1])) * rng.choice([1.0, 1e-3, 100.0])).astype(np.float32)
        w[rng.random(w.size) < 0.05] = 0.0
        if trial % 4 == 0:
            w = np.round(w * 10).astype(np.float32)  # integer weights: many equal-length paths
        G = graph(off, col, w, n)
        src = int(rng.integers(0, n))
        d, _ = lb.CsrMatrix.from_csr(G).sssp(src, sched)
        want = oracle.sssp(off, col, w, src)
        assert np.array_equal(d.cpu().numpy(), want), (trial, sched)


@pytest.mark.parametrize("sched", SCHEDS)
def test_sssp_rmat_equal_dijkstra(sched):
    A = lbgen.rmat(13, 16, 9, "float")
    w = A.values.abs()
    G = lbgen.Csr(A.rows, A.cols, A.row_offsets, A.col_idx, w)
    src = int(torch.argmax(A.row_offsets[1:] - A.row_offsets[:-1]))  # a hub (vertex 0 may be isolated)
    d, rounds = lb.CsrMatrix.from_csr(G).sssp(src, sched)
    assert rounds > 1
    assert np.array_equal(d.cpu().numpy(), oracle.sssp(A.row_offsets, A.col_idx, w, src))


def test_sssp_errors_and_edges():
    G = graph([0, 1, 1], [1], [-1.0], 2)
    with pytest.raises(lb.LbError):
        lb.CsrMatrix.from_csr(G).sssp(0)
    G = graph([0, 1, 1], [1], [float("nan")], 2)
    with pytest.raises(lb.LbError):
        lb.CsrMatrix.from_csr(G).sssp(0)
    G = graph([0, 1, 1], [1], [1.0], 2)
    with pytest.raises(lb.LbError):
        lb.CsrMatrix.from_csr(G).sssp(5)
    R = lbgen.Csr(2, 3, torch.tensor([0, 1, 1], dtype=torch.int32), torch.tensor([2], dtype=torch.int32),
                  torch.ones(1))
    with pytest.raises(lb.LbError):
        lb.CsrMatrix.from_csr(R).sssp(0)
    # isolated source: one round, everything else unreachable
    G = graph([0, 0, 1], [0], [1.0], 2)
    d, rounds = lb.CsrMatrix.from_csr(G).sssp(0)
    assert d.cpu().tolist() == [0.0, float("inf")] and rounds == 1


def certify(off, col, w, d, src):
    """The any-size certificate of the module docstring (torch on the device, test side)."""
    n = off.numel() - 1
    rows = torch.repeat_interleave(torch.arange(n, device=off.device), (off[1:] - off[:-1]).long())
    du, dv = d[rows], d[col.long()]
    cand = du + w  # fp32 add, like the relaxation
    fin = torch.isfinite(du)
    assert d[src].item() == 0.0
    assert bool(torch.all(dv[fin] <= cand[fin])), "an edge is not relaxed"
    tight = fin & (dv == cand)
    reached = torch.zeros(n, dtype=torch.bool, device=off.device)
    reached[src] = True
    while True:
        new = reached.clone()
        new[col.long()[tight & reached[rows]]] = True
        if torch.equal(new, reached):
            break
        reached = new
    assert torch.equal(reached, torch.isfinite(d)), "a finite distance has no tight path from the source"


@pytest.mark.parametrize("sched", SCHEDS)
def test_sssp_full_size_certificate(sched):
    torch.cuda.empty_cache()
    A = lbgen.make_config("c3", "float", device="cuda")
    w = A.values.abs()
    M = lb.CsrMatrix(A.rows, A.cols, A.row_offsets, A.col_idx, w)
    src = int(torch.argmax(A.row_offsets[1:] - A.row_offsets[:-1]).item())  # a hub: large reachable set
    d, rounds = M.sssp(src, sched)
    torch.cuda.synchronize()
    assert rounds > 3
    assert int(torch.isfinite(d).sum()) > A.rows // 4
    certify(A.row_offsets, A.col_idx, w, d, src)
    if sched == "merge_path":  # schedules agree bit for bit
        d2, _ = M.sssp(src, "thread_mapped")
        assert torch.equal(d, d2)
