"""The fused multi-GPU epilogue (NEXT-1: lb_spmv_peers / lb_spmv_multi_fused) on one GPU.

The tile kernel stores every final y value into its own y and into each peer buffer (NVLink peer
stores on a multi-GPU node; here the "peers" are other buffers on the same GPU, which exercises the
same kernel code).  Bar: y and every peer buffer are bitwise equal to the plain merge-path result
(all buffers start as NaN, so a row the epilogue forgets is caught), with and without the x-reuse
plan, at both warp-streamed tile lengths, on matrices with giant rows, empty rows and ragged tails.
"""
import numpy as np
import pytest
import torch

import lbgen
import paper_2212_08964_b200 as lb
from test_gpu_parity import SMALL, _csr, check_y, random_csr, ref

pytestmark = pytest.mark.gpu


def _run_peers(A, x, L, plan, npeers=3):
    M = lb.CsrMatrix.from_csr(A)
    M.set_items_per_tile(L)
    xd = x.cuda()
    y0 = M.spmv(xd, schedule="merge_path", repartition=True).clone()
    if plan is not None:
        M.plan_hot_x(*plan)
    y = torch.full((A.rows,), float("nan"), device="cuda")
    peers = [torch.full((A.rows,), float("nan"), device="cuda") for _ in range(npeers)]
    M.spmv_peers(xd, y, peers, repartition=True)
    torch.cuda.synchronize()
    assert torch.equal(y, y0), "local y differs"
    for i, q in enumerate(peers):
        assert torch.equal(q, y0), f"peer {i} differs: {int((q != y0).sum())} rows"
    return y0


@pytest.mark.parametrize("plan", [None, (512, 0), (64, 4000)])
@pytest.mark.parametrize("L", [504, 1016])
@pytest.mark.parametrize("name", sorted(SMALL))
def test_peers_bitwise(name, L, plan):
    A = SMALL[name]("int")
    x = lbgen.make_x(A.cols, "int", 17)
    y0 = _run_peers(A, x, L, plan)
    y_ref, s_ref = ref(A, x)
    check_y(y0, y_ref, s_ref, True, name)


@pytest.mark.parametrize("npeers", [0, 1, 7])
def test_peers_edge_cases(npeers):
    rng = np.random.default_rng(npeers)
    mats = [_csr([0, 100_003], 1), _csr([0] * 3001, 3), _csr([0, 1, 3, 3, 6], 1),
            lbgen.skewed(1 << 12, 3, 30_000, 20_000, 8, "int")]
    mats += [random_csr(rng, int(rng.integers(1, 3000)), int(rng.integers(1, 400)), int(rng.integers(0, 80)),
                        float(rng.random()) * 0.7, "int") for _ in range(6)]
    for A in mats:
        x = lbgen.make_x(A.cols, "int", 3) if A.cols > 1 else torch.ones(A.cols)
        for L in (504, 1016):
            _run_peers(A, x, L, None, npeers)
            _run_peers(A, x, L, (7, 50), npeers)


def test_peers_errors():
    A = lbgen.stencil(40, 2, "int")
    M = lb.CsrMatrix.from_csr(A)
    M.set_items_per_tile(2040)  # CTA-tile kernel: no fused epilogue
    y = torch.empty(A.rows, device="cuda")
    with pytest.raises(lb.LbError):
        M.spmv_peers(torch.ones(A.cols, device="cuda"), y, [torch.empty(A.rows, device="cuda")])
    M.set_items_per_tile(1016)
    with pytest.raises(lb.LbError):
        M.spmv_peers(torch.ones(A.cols, device="cuda"), y, [torch.empty(A.rows, device="cuda")] * 8)


@pytest.mark.parametrize("cfg", ["c3", "c5"])
def test_peers_full_size(cfg):
    torch.cuda.empty_cache()
    A = lbgen.make_config(cfg, "float", device="cuda")
    x = lbgen.x_for_config(cfg, A.cols, "float", device="cuda")
    M = lb.CsrMatrix.from_csr(A)
    y0 = M.spmv(x, schedule="merge_path", repartition=True).clone()
    M.plan_hot_x(0, -1)
    y = torch.full((A.rows,), float("nan"), device="cuda")
    peer = torch.full((A.rows,), float("nan"), device="cuda")
    M.spmv_peers(x, y, [peer], repartition=True)
    torch.cuda.synchronize()
    assert torch.equal(y, y0) and torch.equal(peer, y0)


def test_multi_fused_single_rank_nccl():
    A = lbgen.rmat(12, 16, 6, "int")
    x = lbgen.make_x(A.cols, "int", 6)
    y_ref, s_ref = ref(A, x)
    comm = lb.Comm(lb.Comm.unique_id(), 0, 1, torch.cuda.current_device())
    b = lb.shard_bounds(A.row_offsets, 1)
    M = lb.CsrMatrix.from_csr(A)
    y = torch.full((A.rows,), float("nan"), device="cuda")
    peer = comm.peer_buffer(y)
    for plan in (None, (256, 1000)):
        if plan:
            M.plan_hot_x(*plan)
        y.fill_(float("nan"))
        comm.spmv_multi_fused(M, b, x.cuda(), peer, repartition=True)
        torch.cuda.synchronize()
        check_y(y, y_ref, s_ref, True, f"fused multi plan={plan}")
    peer.close()
    comm.close()
