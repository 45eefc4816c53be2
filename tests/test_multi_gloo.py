"""Multi-GPU host logic on CPU with world_size 2 (gloo): the equal-nnz shard plan
(lb_shard_bounds), the rebased shard CSR, the NCCL unique-id bootstrap over torch.distributed
and the variable-size all-gather assembly of y that lb_spmv_multi performs with NCCL.
The per-shard SpMV is the oracle here (test-side stand-in for the GPU kernel)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import lbgen
import oracle
import paper_2212_08964_b200 as lb


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        A = {"rmat": lambda: lbgen.rmat(11, 16, 3, "int"),
             "skewed": lambda: lbgen.skewed(1 << 11, 4, 9000, 8000, 2, "int"),
             "stencil": lambda: lbgen.stencil(40, 2, "stencil")}[cfg]()
        x = lbgen.make_x(A.cols, "int", 4)
        b = lb.shard_bounds(A.row_offsets, world)                 # product host logic
        off, col, val = lb.shard_csr(A.row_offsets, A.col_idx, A.values, b, rank)
        assert int(off[0]) == 0 and off.numel() == b[rank + 1] - b[rank] + 1
        y_local, _ = oracle.spmv(off, col, val, x)                 # stand-in for the GPU shard SpMV
        # variable-size all-gather of the y slices (what lb_allgather_rows does with broadcasts)
        y_full = torch.zeros(A.rows, dtype=torch.float64)
        y_full[int(b[rank]):int(b[rank + 1])] = torch.from_numpy(y_local)
        for k, (s0, s1) in enumerate(lb.gather_slices(b)):
            seg = y_full[s0:s1].clone()
            dist.broadcast(seg, src=k)
            y_full[s0:s1] = seg
        y_ref, _ = oracle.spmv(A.row_offsets, A.col_idx, A.values, x)
        ok = bool(np.array_equal(y_full.numpy(), y_ref))
        # every rank holds the same y: compare a checksum across ranks
        h = torch.tensor([float(y_full.sum()), float((y_full * torch.arange(A.rows)).sum())], dtype=torch.float64)
        hs = [torch.zeros_like(h) for _ in range(world)]
        dist.all_gather(hs, h)
        same = all(torch.equal(hs[0], t) for t in hs)
        # NCCL unique id bootstrap through torch.distributed
        uid = lb.Comm.bootstrap_uid()
        u = torch.tensor(list(uid), dtype=torch.int64)
        us = [torch.zeros_like(u) for _ in range(world)]
        dist.all_gather(us, u)
        uid_same = all(torch.equal(us[0], t) for t in us) and len(uid) == 128
        q.put((rank, ok, same, uid_same, list(b)))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e), False, False, None))


@pytest.mark.parametrize("cfg", ["rmat", "skewed", "stencil"])
def test_sharded_spmv_allgather_gloo(cfg):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    for rank, ok, same, uid_same, b in res:
        assert ok is True, (rank, ok)
        assert same and uid_same, (rank, same, uid_same)
    assert res[0][4] == res[1][4]  # identical bounds on every rank
