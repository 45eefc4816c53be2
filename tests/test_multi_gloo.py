"""Multi-GPU host logic on CPU (gloo, world sizes 2-8), running the library's own host code.

* lb_shard_bounds (equal-nnz row shards) and the rebased shard CSR;
* lb_exchange_schedule -- the broadcasts every exchange path of liblb issues (lb_allgather_rows: one
  chunk; lb_spmv_multi_ex(LB_SPMV_CHUNKED): the exchanged cut table, one broadcast group per chunk).
  Here the same schedule drives gloo broadcasts of CPU tensors, in the library's order;
* the padded all-gather layout (lb_padded_rows; columns remapped to k*P + (c - b_k)) as one all_gather;
* the replica check of SURVEY 8(c) p10 with lb_y_checksum's documented hash (the device kernel is
  checked against the same formula in tests/test_gpu_multi.py);
* the NCCL unique-id bootstrap over torch.distributed.
The per-shard SpMV is the oracle (a stand-in for the GPU kernel: no GPU here); two iterations
(x_{k+1} = y_k) so the assembled y is used as the next x.
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

MASK64 = (1 << 64) - 1


def y_checksum_host(y: np.ndarray) -> int:
    """include/lb.h lb_y_checksum: sum_i mix64(i * 0x9E3779B97F4A7C15 + bits(y_i)) mod 2^64."""
    bits = np.ascontiguousarray(y, dtype=np.float32).view(np.uint32).astype(np.uint64)
    with np.errstate(over="ignore"):
        z = np.arange(bits.size, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15) + bits
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return int(z.sum(dtype=np.uint64)) & MASK64


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _matrix(cfg):
    return {"rmat": lambda: lbgen.rmat(11, 16, 3, "int"),
            "skewed": lambda: lbgen.skewed(1 << 11, 4, 9000, 8000, 2, "int"),
            "stencil": lambda: lbgen.stencil(40, 2, "int")}[cfg]()


def _random_cuts(rng, n: int, K: int) -> np.ndarray:
    """K chunks of a shard of n rows: sorted cut rows 0 = c_0 <= ... <= c_K = n (empty chunks allowed)."""
    inner = np.sort(rng.integers(0, n + 1, K - 1)) if K > 1 else np.zeros(0, np.int64)
    return np.concatenate([[0], inner, [n]]).astype(np.int64)


def _exchange(y_full: torch.Tensor, bounds, cuts_all, world):
    """The library's exchange schedule, executed with gloo broadcasts (chunk by chunk, root by root)."""
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
        dist.init_process_group("gloo", rank=rank, world_size=world)
        A = _matrix(cfg)
        n = A.rows
        b = lb.shard_bounds(A.row_offsets, world)                 # product host logic
        off, col, val = lb.shard_csr(A.row_offsets, A.col_idx, A.values, b, rank)
        assert int(off[0]) == 0 and off.numel() == b[rank + 1] - b[rank] + 1
        n_loc = int(b[rank + 1] - b[rank])
        x0 = lbgen.make_x(A.cols, "int", 4)
        # reference: two iterations on one process
        r1, _ = oracle.spmv(A.row_offsets, A.col_idx, A.values, x0)
        r2, _ = oracle.spmv(A.row_offsets, A.col_idx, A.values, torch.from_numpy(r1))
        res = {}
        # (1) plain all-gather(v) and (2) the chunked exchange with an exchanged cut table
        rng = np.random.default_rng(100 + rank)
        for mode in ("plain", "chunked"):
            if mode == "chunked":  # every rank's cut rows, exchanged as lb_spmv_multi_ex does it
                mine = torch.from_numpy(_random_cuts(rng, n_loc, lb.CHUNKS_MAX))
                allc = [torch.zeros_like(mine) for _ in range(world)]
                dist.all_gather(allc, mine)
                cuts = torch.stack(allc).numpy()
            else:
                cuts = None
            x = x0.double()
            for it in range(2):
                y_loc, _ = oracle.spmv(off, col, val, x.float())    # stand-in for the GPU shard SpMV
                y_full = torch.zeros(n, dtype=torch.float64)
                y_full[int(b[rank]):int(b[rank + 1])] = torch.from_numpy(y_loc)
                y_full = _exchange(y_full, b, cuts, world)
                x = y_full
            res[mode] = bool(np.array_equal(x.numpy(), r2))
        # (3) padded layout: columns remapped once to k*P + (c - b_k); one all_gather of P-sized slots
        P = lb.padded_rows(b)
        shard_of = np.searchsorted(b, col.numpy(), side="right") - 1
        pcol = torch.from_numpy((shard_of * P + (col.numpy() - b[shard_of])).astype(np.int32))
        xp = torch.zeros(world * P, dtype=torch.float64)
        for k in range(world):
            xp[k * P:k * P + int(b[k + 1] - b[k])] = x0[int(b[k]):int(b[k + 1])].double()
        for it in range(2):
            y_loc, _ = oracle.spmv(off, pcol, val, xp.float())
            slot = torch.zeros(P, dtype=torch.float64)
            slot[:n_loc] = torch.from_numpy(y_loc)
            slots = [torch.zeros(P, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(slots, slot)
            xp = torch.cat(slots)
        unpadded = torch.cat([xp[k * P:k * P + int(b[k + 1] - b[k])] for k in range(world)])
        res["padded"] = bool(np.array_equal(unpadded.numpy(), r2))
        # (4) replica check (p10): every rank's hash of its y, min == max
        h = y_checksum_host(x.numpy().astype(np.float32))
        hs = torch.tensor([h - (1 << 63)], dtype=torch.int64)  # shift into int64's range
        lo, hi = hs.clone(), hs.clone()
        dist.all_reduce(lo, op=dist.ReduceOp.MIN)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX)
        res["replicas"] = bool(lo == hi)
        # NCCL unique id bootstrap through torch.distributed
        uid = lb.Comm.bootstrap_uid()
        u = torch.tensor(list(uid), dtype=torch.int64)
        us = [torch.zeros_like(u) for _ in range(world)]
        dist.all_gather(us, u)
        res["uid"] = all(torch.equal(us[0], t) for t in us) and len(uid) == 128
        q.put((rank, res, list(b)))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, {"error": traceback.format_exc()}, None))


@pytest.mark.parametrize("cfg,world", [("rmat", 2), ("skewed", 2), ("stencil", 2), ("rmat", 3), ("skewed", 4),
                                       ("rmat", 8)])
def test_sharded_spmv_exchange_gloo(cfg, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    for rank, r, b in res:
        assert "error" not in r, r.get("error")
        assert all(r.values()), (rank, r)
    assert all(r[2] == res[0][2] for r in res)  # identical bounds on every rank


# ---------------------------------------------------------------- the schedule itself, any world size

@pytest.mark.parametrize("world", [1, 2, 3, 5, 8])
def test_exchange_schedule_tiles_y_exactly_once(world):
    """Over all (chunk, root) the broadcast ranges tile [0, rows) exactly once, each range inside its
    root's shard, chunk c of root k = its local rows [cut[k][c], cut[k][c+1])."""
    rng = np.random.default_rng(world)
    for trial in range(20):
        rows = int(rng.integers(0, 5000))
        inner = np.sort(rng.integers(0, rows + 1, world - 1))
        b = np.concatenate([[0], inner, [rows]]).astype(np.int64)
        for K in (1, 3, lb.CHUNKS_MAX):
            cuts = np.stack([_random_cuts(rng, int(b[k + 1] - b[k]), K) for k in range(world)])
            off, cnt = lb.exchange_schedule(b, cuts)
            assert off.shape == cnt.shape == (K, world)
            cover = np.zeros(rows, np.int64)
            for c in range(K):
                for k in range(world):
                    assert b[k] <= off[c, k] and off[c, k] + cnt[c, k] <= b[k + 1]
                    assert off[c, k] == b[k] + cuts[k, c] and cnt[c, k] == cuts[k, c + 1] - cuts[k, c]
                    cover[off[c, k]:off[c, k] + cnt[c, k]] += 1
            assert np.all(cover == 1)
        off, cnt = lb.exchange_schedule(b)  # plain all-gather: one chunk, each rank's whole slice
        assert np.array_equal(off[0], b[:-1]) and np.array_equal(cnt[0], np.diff(b))
        assert lb.gather_slices(b) == [(int(b[k]), int(b[k + 1])) for k in range(world)]
        assert lb.padded_rows(b) == int(np.diff(b).max(initial=0))


def test_exchange_schedule_rejects_bad_tables():
    b = np.array([0, 5, 9], np.int64)
    with pytest.raises(lb.LbError):
        lb.exchange_schedule(np.array([0, 5, 4], np.int64))              # bounds not monotone
    with pytest.raises(lb.LbError):
        lb.exchange_schedule(np.array([1, 5, 9], np.int64))              # bounds[0] != 0
    with pytest.raises(lb.LbError):
        lb.exchange_schedule(b, np.array([[0, 3, 5], [0, 2, 3]]))        # rank 1 cuts end at 3, not 4
    with pytest.raises(lb.LbError):
        lb.exchange_schedule(b, np.array([[0, 4, 3, 5], [0, 1, 2, 4]]))  # not monotone
    with pytest.raises(ValueError):
        lb.exchange_schedule(b, np.zeros((3, 4), np.int64))              # wrong rank count


def test_checksum_formula_properties():
    """The host formula of lb_y_checksum: position-dependent, bitwise (-0 != +0), order-free sum."""
    y = np.random.default_rng(0).standard_normal(1000).astype(np.float32)
    h = y_checksum_host(y)
    z = y.copy()
    z[[3, 7]] = z[[7, 3]]
    assert y_checksum_host(z) != h
    z = y.copy()
    z[5] = np.nextafter(z[5], np.float32(np.inf))
    assert y_checksum_host(z) != h
    assert y_checksum_host(np.array([0.0], np.float32)) != y_checksum_host(np.array([-0.0], np.float32))
    assert y_checksum_host(np.zeros(0, np.float32)) == 0
