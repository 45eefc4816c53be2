"""Seeded synthetic CSR inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no SpMV, no partition, no search).
It only draws matrices and vectors from a counter-based hash so that the CPU and the
GPU regenerate bit-identical inputs.

Every random draw is ``splitmix64(seed * 0x9E3779B97F4A7C15 + counter)`` evaluated with
wrapping int64 tensor arithmetic (identical on CPU and CUDA).  Matrix classes follow the
workloads BASELINE.json names (uniform, 2-D 5-point stencil, R-MAT power law, few giant
rows).  Values are assigned by CSR position k so any class can be drawn in any value mode:

  * ``"int"``    values in {+-1, +-2}           (integer-exact mode)
  * ``"float"``  values uniform in [-1, 1) on a 2^-23 grid (exact in fp32; tolerance mode p9)
  * ``"ones"``   all values 1
  * ``"stencil"`` 4 on the diagonal, -1 off it (only meaningful for the stencil class)

x vectors: ``"int"`` {-4..4}, ``"float"`` as above, ``"ones"``, ``"index"`` (x_i = i).
"""
from __future__ import annotations

import dataclasses
import torch

_M64 = (1 << 64) - 1


def _s64(v: int) -> int:
    """Map an unsigned 64-bit constant to the int64 with the same bit pattern."""
    v &= _M64
    return v - (1 << 64) if v >= (1 << 63) else v


_GOLD = _s64(0x9E3779B97F4A7C15)
_C1 = _s64(0xBF58476D1CE4E5B9)
_C2 = _s64(0x94D049BB133111EB)


def _srl(z: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of an int64 tensor (torch's >> is arithmetic)."""
    return (z >> k) & ((1 << (64 - k)) - 1)


def splitmix64(z: torch.Tensor) -> torch.Tensor:
    z = z + _GOLD
    z = (z ^ _srl(z, 30)) * _C1
    z = (z ^ _srl(z, 27)) * _C2
    return z ^ _srl(z, 31)


def hash64(seed: int, ctr: torch.Tensor) -> torch.Tensor:
    """u64 draw number ``ctr`` of stream ``seed`` (as an int64 bit pattern)."""
    return splitmix64(ctr + _s64(seed * 0x9E3779B97F4A7C15))


def u24(seed: int, ctr: torch.Tensor) -> torch.Tensor:
    """Top 24 bits of the draw, as int64 in [0, 2^24)."""
    return _srl(hash64(seed, ctr), 40)


def _arange(n: int, device) -> torch.Tensor:
    return torch.arange(n, dtype=torch.int64, device=device)


def values_from_bits(u: torch.Tensor, mode: str) -> torch.Tensor:
    """fp32 values from 24-bit draws."""
    if mode == "float":
        return ((u - (1 << 23)).to(torch.float64) * 2.0 ** -23).to(torch.float32)
    if mode == "int":
        sign = 1 - 2 * (u & 1)
        mag = 1 + ((u >> 1) & 1)
        return (sign * mag).to(torch.float32)
    if mode == "xint":
        return ((u % 9) - 4).to(torch.float32)
    if mode == "pos":  # same-sign: uniform [0, 1) on the 2^-24 grid (exact in fp32)
        return (u.to(torch.float64) * 2.0 ** -24).to(torch.float32)
    raise ValueError(mode)


def _perm_bits(v: torch.Tensor, bits: int, seed: int) -> torch.Tensor:
    """Seeded bijection on [0, 2^bits): xor-constant, odd multiply and xorshift rounds."""
    mask = (1 << bits) - 1
    k = int(u24(seed, torch.tensor([0, 1, 2], dtype=torch.int64))[0])  # scalar key from the stream
    v = (v ^ (k & mask)) & mask
    for mult in (0x9E3779B1, 0x85EBCA77, 0xC2B2AE3D):
        v = (v * mult) & mask          # odd multiplier: bijective mod 2^bits
        v = v ^ (v >> max(1, bits // 2))  # xorshift: bijective
    return v & mask


@dataclasses.dataclass
class Csr:
    rows: int
    cols: int
    row_offsets: torch.Tensor  # int32 [rows+1]
    col_idx: torch.Tensor      # int32 [nnz]
    values: torch.Tensor       # float32 [nnz]
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.col_idx.numel())

    def to(self, device) -> "Csr":
        return Csr(self.rows, self.cols, self.row_offsets.to(device), self.col_idx.to(device),
                   self.values.to(device), self.name)


def _offsets_from_row_ids(row_ids: torch.Tensor, rows: int) -> torch.Tensor:
    counts = torch.bincount(row_ids, minlength=rows)
    off = torch.zeros(rows + 1, dtype=torch.int64, device=row_ids.device)
    off[1:] = torch.cumsum(counts, 0)
    return off.to(torch.int32)


def _offsets_from_lengths(lengths: torch.Tensor) -> torch.Tensor:
    off = torch.zeros(lengths.numel() + 1, dtype=torch.int64, device=lengths.device)
    off[1:] = torch.cumsum(lengths.to(torch.int64), 0)
    return off


def assign_values(nnz: int, mode: str, seed: int, device) -> torch.Tensor:
    if mode == "ones":
        return torch.ones(nnz, dtype=torch.float32, device=device)
    if mode == "tenth":  # same-sign constant fl32(0.1): the worst case for sequential fp32 sums
        return torch.full((nnz,), 0.1, dtype=torch.float32, device=device)
    out = torch.empty(nnz, dtype=torch.float32, device=device)
    chunk = 1 << 26
    for s in range(0, nnz, chunk):
        e = min(nnz, s + chunk)
        out[s:e] = values_from_bits(u24(seed + 7919, _arange(e - s, device) + s), mode)
    return out


def make_x(n: int, mode: str, seed: int, device="cpu") -> torch.Tensor:
    """Dense input vector x (fp32)."""
    if mode == "ones":
        return torch.ones(n, dtype=torch.float32, device=device)
    if mode == "index":
        return torch.arange(n, dtype=torch.float32, device=device)
    if mode == "int":
        return values_from_bits(u24(seed, _arange(n, device)), "xint")
    return values_from_bits(u24(seed, _arange(n, device)), mode)


# --------------------------------------------------------------------------- classes

def uniform(n: int, p: float, seed: int, vmode: str, device="cpu") -> Csr:
    """n x n Bernoulli(p): entry (i, j) present iff u24(hash(i*n+j)) < p*2^24."""
    thr = int(round(p * (1 << 24)))
    idx = _arange(n * n, device)
    keep = u24(seed, idx) < thr
    lin = idx[keep]
    rows_ = lin // n
    cols_ = (lin % n).to(torch.int32)
    off = _offsets_from_row_ids(rows_, n)
    vals = assign_values(lin.numel(), vmode, seed, device)
    return Csr(n, n, off, cols_, vals, f"uniform{n}p{p}")


def stencil(N: int, seed: int, vmode: str, device="cpu") -> Csr:
    """2-D 5-point Poisson stencil on an N x N grid; node i = yy*N + xx; entries sorted by column."""
    rows = N * N
    node = _arange(rows, device)
    yy, xx = node // N, node % N
    cand = torch.stack([node - N, node - 1, node, node + 1, node + N], 1)
    ok = torch.stack([yy > 0, xx > 0, torch.ones_like(yy, dtype=torch.bool), xx < N - 1, yy < N - 1], 1)
    lengths = ok.sum(1)
    cols_ = cand[ok].to(torch.int32)
    off = _offsets_from_lengths(lengths).to(torch.int32)
    nnz = cols_.numel()
    if vmode == "stencil":
        diag = torch.zeros_like(ok)
        diag[:, 2] = True
        vals = torch.where(diag[ok], 4.0, -1.0).to(torch.float32)
    else:
        vals = assign_values(nnz, vmode, seed, device)
    return Csr(rows, rows, off, cols_, vals, f"stencil{N}")


RMAT_ABCD = (0.57, 0.19, 0.19, 0.05)  # Graph500 initiator


def rmat(scale: int, edge_factor: int, seed: int, vmode: str, device="cpu", chunk: int = 1 << 25) -> Csr:
    """R-MAT power-law matrix: E = edge_factor * 2^scale directed edges, one quadrant draw per level,
    vertex ids relabeled by a seeded bijection, sorted by (row, col); duplicates and self loops kept."""
    n = 1 << scale
    E = edge_factor * n
    a, b, c, _ = RMAT_ABCD
    ta = int(round(a * (1 << 24)))
    tb = int(round((a + b) * (1 << 24)))
    tc = int(round((a + b + c) * (1 << 24)))
    keys = torch.empty(E, dtype=torch.int64, device=device)
    for s in range(0, E, chunk):
        e = min(E, s + chunk)
        eid = _arange(e - s, device) + s
        r = torch.zeros_like(eid)
        cc = torch.zeros_like(eid)
        for lvl in range(scale):
            u = u24(seed, eid * scale + lvl)
            rbit = (u >= tb).to(torch.int64)                     # quadrants c, d
            cbit = ((u >= ta) & (u < tb) | (u >= tc)).to(torch.int64)  # quadrants b, d
            r |= rbit << lvl
            cc |= cbit << lvl
            del u, rbit, cbit
        r = _perm_bits(r, scale, seed + 1)
        cc = _perm_bits(cc, scale, seed + 1)
        keys[s:e] = (r << scale) | cc
        del eid, r, cc
    keys, _ = torch.sort(keys)
    rows_ = keys >> scale
    cols_ = (keys & (n - 1)).to(torch.int32)
    del keys
    off = _offsets_from_row_ids(rows_, n)
    del rows_
    vals = assign_values(E, vmode, seed, device)
    return Csr(n, n, off, cols_, vals, f"rmat{scale}ef{edge_factor}")


def skewed(rows: int, n_giant: int, giant_len: int, nnz_rest: int, seed: int, vmode: str,
           device="cpu", cols: int | None = None) -> Csr:
    """Few giant rows: n_giant rows at seeded positions with giant_len nnz each; the remaining
    rows share nnz_rest as evenly as possible (floor or ceil); columns uniform with
    replacement, sorted per row."""
    cols = rows if cols is None else cols
    bits = (rows - 1).bit_length()
    assert rows == 1 << bits, "skewed generator needs a power-of-two row count"
    giant_pos = _perm_bits(_arange(n_giant, device), bits, seed + 3)
    is_giant = torch.zeros(rows, dtype=torch.bool, device=device)
    is_giant[giant_pos] = True
    n_rest = rows - n_giant
    base, extra = divmod(nnz_rest, n_rest)
    rank = torch.cumsum((~is_giant).to(torch.int64), 0) - 1
    lengths = torch.where(is_giant, giant_len, base + (rank < extra).to(torch.int64))
    off64 = _offsets_from_lengths(lengths)
    nnz = int(off64[-1])
    row_ids = torch.repeat_interleave(_arange(rows, device), lengths)
    cbits = (cols - 1).bit_length()
    c = _srl(hash64(seed, _arange(nnz, device)), 64 - cbits) if cols == 1 << cbits else \
        _srl(hash64(seed, _arange(nnz, device)), 1) % cols
    key = row_ids * cols + c
    del row_ids, c
    key, _ = torch.sort(key)
    cols_ = (key % cols).to(torch.int32)
    del key
    vals = assign_values(nnz, vmode, seed, device)
    return Csr(rows, cols, off64.to(torch.int32), cols_, vals, f"skewed{rows}g{n_giant}x{giant_len}")


def from_dense_pattern(off: list[int], cols: int, col_idx: list[int], vals: list[float], name="explicit") -> Csr:
    return Csr(len(off) - 1, cols, torch.tensor(off, dtype=torch.int32), torch.tensor(col_idx, dtype=torch.int32),
               torch.tensor(vals, dtype=torch.float32), name)


# --------------------------------------------------------------------------- named configs
# BASELINE.json configs[0..4] = C1..C5; seeds 1..5; x seed = 1000 + config#.
CONFIGS = {
    "c1": dict(kind="uniform", n=1000, p=0.01, seed=1),
    "c2": dict(kind="stencil", N=2048, seed=2),
    "c3": dict(kind="rmat", scale=24, ef=16, seed=3),
    "c4": dict(kind="skewed", rows=1 << 22, n_giant=1000, giant_len=100_000, nnz_rest=100_000_000, seed=4),
    "c5": dict(kind="rmat", scale=26, ef=16, seed=5),
    "c6": dict(kind="uniform_rows", scale=24, per_row=16, seed=6),
}

CONFIG_DESC = {
    "c1": "uniform random CSR 1,000x1,000, p=0.01 (~10k nnz)",
    "c2": "2D 5-point Poisson stencil on a 2048x2048 grid (4,194,304 rows, 20,963,328 nnz)",
    "c3": "R-MAT scale-24, edge factor 16 (16,777,216 rows, 268,435,456 nnz)",
    "c4": "skewed: 4,194,304 rows, 1,000 giant rows x 100,000 nnz + 100M nnz spread (200M nnz)",
    "c5": "R-MAT scale-26, edge factor 16 (67,108,864 rows, 1,073,741,824 nnz)",
}


def uniform_rows(scale: int, per_row: int, seed: int, vmode: str, device="cpu") -> Csr:
    rows = 1 << scale
    return skewed(rows, 0, 0, rows * per_row, seed, vmode, device)


MAX_MERGE_ITEMS = (1 << 31) - (1 << 16) - 1  # largest rows + nnz the C ABI accepts (include/lb.h)


def max_size(seed: int, vmode: str, device="cpu", cols: int = 1 << 20, giant: int = 200_000) -> Csr:
    """The largest merge-path problem the API accepts: rows + nnz = MAX_MERGE_ITEMS exactly, nnz = 2^30.
    Ragged rows repeating (2, 0, 1) nonzeros (a third of the rows empty), row 5 a giant row of
    1 + `giant` nonzeros paid for by emptying `giant` / 2 of the 2-rows after it, and the last row taking
    the remainder that makes nnz exact.  Columns: counter hash, uniform over `cols`."""
    nnz = 1 << 30
    rows = MAX_MERGE_ITEMS - nnz
    r = _arange(rows, device)
    lengths = torch.where(r % 3 == 0, 2, torch.where(r % 3 == 1, 0, 1))
    del r
    lengths[5] += giant
    lengths[6:6 + 3 * (giant // 2):3] = 0  # rows 6, 9, ... (each had 2)
    lengths[-1] = 0
    rest = nnz - int(lengths.sum())
    assert rest >= 0
    lengths[-1] = rest
    off64 = _offsets_from_lengths(lengths)
    del lengths
    assert int(off64[-1]) == nnz
    col = torch.empty(nnz, dtype=torch.int32, device=device)
    cbits = (cols - 1).bit_length()
    assert cols == 1 << cbits
    chunk = 1 << 26
    for s in range(0, nnz, chunk):
        e = min(nnz, s + chunk)
        col[s:e] = _srl(hash64(seed, _arange(e - s, device) + s), 64 - cbits).to(torch.int32)
    vals = assign_values(nnz, vmode, seed, device)
    return Csr(rows, cols, off64.to(torch.int32), col, vals, "max_size")


def make_config(name: str, vmode: str = "float", device="cpu") -> Csr:
    c = dict(CONFIGS[name])
    kind = c.pop("kind")
    if kind == "uniform":
        A = uniform(c["n"], c["p"], c["seed"], vmode, device)
    elif kind == "stencil":
        A = stencil(c["N"], c["seed"], vmode, device)
    elif kind == "rmat":
        A = rmat(c["scale"], c["ef"], c["seed"], vmode, device)
    elif kind == "skewed":
        A = skewed(c["rows"], c["n_giant"], c["giant_len"], c["nnz_rest"], c["seed"], vmode, device)
    elif kind == "uniform_rows":
        A = uniform_rows(c["scale"], c["per_row"], c["seed"], vmode, device)
    else:
        raise ValueError(kind)
    A.name = name
    return A


def x_for_config(name: str, n: int, mode: str, device="cpu") -> torch.Tensor:
    return make_x(n, mode, 1000 + int(name[1:]), device)
