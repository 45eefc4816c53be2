"""The row-sharded multi-GPU iteration with the real CUDA shard SpMV, several ranks on one B200.

NCCL refuses two ranks on one device, so this run has no NCCL exchange at world size > 1; instead
every rank is a separate process on cuda:0 (its own context and handle), computes its equal-nnz
shard (lb_shard_bounds / shard_csr) with the library's merge-path kernels -- plain and with the
x-reuse plan -- and the y exchange is the library's own schedule (lb_exchange_schedule: one chunk,
or the handle's LB_SPMV_CHUNKED cut rows exchanged between ranks as lb_spmv_multi_ex does) executed
as gloo broadcasts of host copies.  Two iterations (x_{k+1} = y_k) in integer mode: the assembled y of
the first equals the single-process oracle bit for bit (every partial sum an integer below 2^24), the
second (its sums leave fp32's exact-integer range) is within the tolerance of the oracle applied to the
first's y; the replica check of SURVEY 8(c) p10 uses the device checksum kernel (lb_y_checksum) on
every rank.
"""
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

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _matrix(cfg):
    return {"rmat": lambda: lbgen.rmat(14, 16, 3, "int"),
            "skewed": lambda: lbgen.skewed(1 << 13, 4, 30000, 20000, 2, "int"),
            "stencil": lambda: lbgen.stencil(120, 2, "int")}[cfg]()


def _exchange(y_full: torch.Tensor, bounds, cuts_all, world):
    off, cnt = lb.exchange_schedule(bounds, cuts_all)
    for c in range(off.shape[0]):
        for k in range(world):
            if cnt[c, k] == 0:
                continue
            s0, s1 = int(off[c, k]), int(off[c, k] + cnt[c, k])
            seg = y_full[s0:s1].clone()
            dist.broadcast(seg, src=k)
            y_full[s0:s1] = seg
    return y_full


def _worker(rank, world, port, cfg, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        A = _matrix(cfg)
        n = A.rows
        b = lb.shard_bounds(A.row_offsets, world)
        off, col, val = lb.shard_csr(A.row_offsets, A.col_idx, A.values, b, rank)
        b0, b1 = int(b[rank]), int(b[rank + 1])
        M = lb.CsrMatrix(b1 - b0, A.cols, off.cuda(), col.cuda(), val.cuda(), validate=True)
        x0 = lbgen.make_x(A.cols, "int", 4)
        r1, _ = oracle.spmv(A.row_offsets, A.col_idx, A.values, x0)
        assert np.abs(r1).max() < 2 ** 24
        r2, s2 = oracle.spmv(A.row_offsets, A.col_idx, A.values, torch.from_numpy(r1.astype(np.float32)))
        res = {}
        for plan in (False, True):
            if plan:
                M.set_items_per_tile(1016)
                M.plan_hot_x(512, -1)
            for mode in ("plain", "chunked"):
                if mode == "chunked":  # the handle's real LB_SPMV_CHUNKED cut rows, exchanged between ranks
                    mine = torch.from_numpy(M.chunk_rows())
                    allc = [torch.zeros_like(mine) for _ in range(world)]
                    dist.all_gather(allc, mine)
                    cuts = torch.stack(allc).numpy()
                else:
                    cuts = None
                x = x0.clone()
                for it in range(2):
                    if mode == "chunked" and plan:  # the chunked launches themselves (LB_SPMV_CHUNKED)
                        y_loc = M.spmv_host(x.contiguous().pin_memory(), torch.empty(b1 - b0).pin_memory(),
                                            "merge_path", repartition=True, chunked=True)
                    else:
                        y_loc = M.spmv(x.cuda(), schedule="merge_path", repartition=True)  # the CUDA shard SpMV
                    y_full = torch.zeros(n, dtype=torch.float32)
                    y_full[b0:b1] = y_loc.cpu()
                    x = _exchange(y_full, b, cuts, world)
                    if it == 0:
                        res[f"plan={plan}/{mode}/iter1_exact"] = bool(np.array_equal(x.double().numpy(), r1))
                err = np.abs(x.double().numpy() - r2)
                res[f"plan={plan}/{mode}/iter2_tol"] = bool(np.all(err <= 1e-5 * s2 + 1e-30))
        # replica check (p10) with the device checksum kernel on every rank
        h = lb.y_checksum(x.cuda())
        hs = torch.tensor([h - (1 << 63)], dtype=torch.int64)
        lo, hi = hs.clone(), hs.clone()
        dist.all_reduce(lo, op=dist.ReduceOp.MIN)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX)
        res["replicas"] = bool(lo == hi)
        q.put((rank, res, [int(v) for v in b]))
        M.close()
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, {"error": traceback.format_exc()}, None))


@pytest.mark.parametrize("cfg,world", [("rmat", 2), ("skewed", 2), ("stencil", 3), ("rmat", 4)])
def test_sharded_iteration_real_kernels(cfg, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in ps:
        p.join(timeout=120)
    for rank, r, b in res:
        assert "error" not in r, r.get("error")
        assert all(r.values()), (rank, r)
    assert all(r[2] == res[0][2] for r in res)
