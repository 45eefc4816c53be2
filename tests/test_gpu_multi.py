"""GPU side of the multi-GPU layer at world size 1 (the only size this run's single-GPU boxes allow):

* lb_y_checksum's device kernel against the host formula of include/lb.h (tests/test_multi_gloo.py);
* lb_comm_check_replicas through NCCL all-reduces;
* lb_remap_cols_padded against a numpy derivation, and lb_spmv_multi_ex(LB_SPMV_PADDED) with one rank;
* lb_allgather_rows at world size 1 (one in-place NCCL broadcast: the same code path as N > 1);
* lb_csr_chunk_rows: the cut table a rank contributes to the chunked exchange is a valid schedule.
The exchange at N > 1 is covered on CPU by tests/test_multi_gloo.py (the library's own schedule).
"""
import numpy as np
import pytest
import torch

import lbgen
import paper_2212_08964_b200 as lb
from test_gpu_parity import check_y, ref
from test_multi_gloo import y_checksum_host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm():
    c = lb.Comm(lb.Comm.unique_id(), 0, 1, torch.cuda.current_device())
    yield c
    c.close()


@pytest.mark.parametrize("n", [0, 1, 31, 1000, 1 << 20, 3_000_001])
def test_checksum_kernel_matches_host_formula(n):
    y = torch.randn(n, generator=torch.Generator().manual_seed(n)).cuda()
    if n > 4:
        y[2] = -0.0
        y[3] = float("inf")
    assert lb.y_checksum(y) == y_checksum_host(y.cpu().numpy())


def test_checksum_detects_single_bit_flip():
    y = torch.randn(100_000).cuda()
    h = lb.y_checksum(y)
    z = y.clone()
    z.view(torch.int32)[77_777] ^= 1
    assert lb.y_checksum(z) != h
    assert lb.y_checksum(y) == h  # deterministic


def test_check_replicas_single_rank(comm):
    y = torch.randn(123_457).cuda()
    eq, h = comm.check_replicas(y)
    assert eq and h == lb.y_checksum(y)


@pytest.mark.parametrize("G", [1, 3, 8])
def test_remap_cols_padded_matches_numpy(G):
    A = lbgen.rmat(13, 16, 6, "int")
    b = lb.shard_bounds(A.row_offsets, G)
    P = lb.padded_rows(b)
    col = A.col_idx.cuda()
    got = lb.remap_cols_padded(b, col).cpu().numpy()
    c = A.col_idx.numpy().astype(np.int64)
    k = np.searchsorted(b, c, side="right") - 1
    assert np.array_equal(got, (k * P + c - b[k]).astype(np.int32))
    same = lb.remap_cols_padded(b, col, out=col)  # in place
    assert np.array_equal(same.cpu().numpy(), got)


def test_spmv_multi_padded_single_rank(comm):
    A = lbgen.rmat(13, 16, 7, "int")
    b = lb.shard_bounds(A.row_offsets, 1)
    assert lb.padded_rows(b) == A.rows
    pcol = lb.remap_cols_padded(b, A.col_idx.cuda())
    assert torch.equal(pcol.cpu(), A.col_idx)  # one rank: the identity
    M = lb.CsrMatrix(A.rows, A.cols, A.row_offsets.cuda(), pcol, A.values.cuda())
    x = lbgen.make_x(A.cols, "int", 3)
    y_ref, s_ref = ref(A, x)
    y = torch.full((A.rows,), float("nan"), device="cuda")
    comm.spmv_multi(M, b, x.cuda(), y, padded=True, repartition=True)
    torch.cuda.synchronize()
    check_y(y, y_ref, s_ref, True, "padded")
    with pytest.raises(lb.LbError):
        comm.spmv_multi(M, b, x.cuda(), y, padded=True, chunked=True)


def test_allgather_rows_single_rank_runs_nccl(comm):
    A = lbgen.rmat(12, 16, 6, "int")
    b = lb.shard_bounds(A.row_offsets, 1)
    y = torch.randn(A.rows).cuda()
    y0 = y.clone()
    comm.allgather_rows(b, y)  # one in-place broadcast, root 0
    torch.cuda.synchronize()
    assert torch.equal(y, y0)
    with pytest.raises(ValueError):
        comm.allgather_rows(b, y[:-1])


@pytest.mark.parametrize("plan", [True, False])
def test_chunk_rows_form_a_valid_schedule(plan):
    A = lbgen.rmat(15, 16, 9, "int")
    M = lb.CsrMatrix.from_csr(A)
    if plan:
        M.plan_hot_x(1024, 0)
    cuts = M.chunk_rows()
    assert cuts[0] == 0 and cuts[-1] == A.rows and np.all(np.diff(cuts) >= 0)
    if plan:
        assert np.count_nonzero(np.diff(cuts)) > 1  # really chunked
        # every cut is a clean merge-path coordinate: it never splits a row
        off = A.row_offsets.numpy()
        assert all(0 <= c <= A.rows for c in cuts)
    else:
        assert np.array_equal(cuts, [0] + [A.rows] * lb.CHUNKS_MAX)
    off, cnt = lb.exchange_schedule(np.array([0, A.rows]), cuts[None, :])
    assert cnt.sum() == A.rows


def test_spmv_multi_validates_buffers(comm):
    A = lbgen.rmat(11, 16, 6, "int")
    b = lb.shard_bounds(A.row_offsets, 1)
    M = lb.CsrMatrix.from_csr(A)
    x = torch.zeros(A.cols, device="cuda")
    with pytest.raises(ValueError):
        comm.spmv_multi(M, b, x, torch.zeros(A.rows - 1, device="cuda"))
    with pytest.raises(ValueError):
        comm.spmv_multi(M, b, x[:-1], torch.zeros(A.rows, device="cuda"))
    with pytest.raises(ValueError):
        comm.spmv_multi(M, b, x.double(), torch.zeros(A.rows, device="cuda"))
