// k_spmm.cuh -- sm_100a device code (arXiv 2212.08964).  Citations "P:L" = PAPER.md line L.
// SpMM on merge-path tiles (NEXT-2, Listing 4).
#pragma once
#include "dev_common.cuh"

namespace lbk {

// ----------------------------------------------------------------------------- SpMM (NEXT-2)
// Y = A X for a panel of P (1, 4 or 8) columns of a row-major X (Listing 4: "a simple loop
// wrapped around SpMV"), on the same merge-path tiles as SpMV (L = 1016, lb_partition's output is
// reused).  Warp-streamed like merge_stream_kernel, with 4 nonzeros per lane per round (128 per
// warp-round, 8 rounds per tile) and one P-wide gather X[col, c0 .. c0+P) per nonzero: with P = 4
// a single 16-byte gather feeds 4 outputs, which is what lifts SpMM above SpMV's gather bound.
struct SpmmArgs {
  const int* off;
  const int* col;
  const float* val;
  const float* X;  // panel base: &X[0, c0]
  float* Y;        // panel base: &Y[0, c0]
  int64_t ldx, ldy;
  const int2* coords;
  int rows, nnz;
  int num_tiles;
  int tiles_per_warp;
  int* carry_row;
  float* carry_val;  // [warps * P]
  unsigned* ticket;
  int vec;           // col/val 16-byte aligned -> 128-bit loads
};

template <int P>
struct PVec;
template <>
struct PVec<1> {
  float v[1];
};
template <>
struct PVec<4> {
  float v[4];
};
template <>
struct PVec<8> {
  float v[8];
};

template <int P>
__device__ __forceinline__ void spmm_gather(const SpmmArgs& a, int c, PVec<P>& out) {
  const float* src = a.X + (int64_t)c * a.ldx;
  if (P == 8) {  // one 32-byte sector per nonzero: a single 256-bit gather
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(out.v[0]), "=f"(out.v[1]), "=f"(out.v[2]), "=f"(out.v[3]), "=f"(out.v[4]), "=f"(out.v[5]),
          "=f"(out.v[6]), "=f"(out.v[7])
        : "l"(src));
  } else if (P == 4) {
    const float4 t = __ldg(reinterpret_cast<const float4*>(src));
    out.v[0] = t.x; out.v[1] = t.y; out.v[2] = t.z; out.v[3] = t.w;
  } else {
    out.v[0] = __ldg(src);
  }
}

template <int P>
__device__ __forceinline__ void spmm_store(const SpmmArgs& a, int row, const float (&v)[P]) {
  float* dst = a.Y + (int64_t)row * a.ldy;
  if (P == 8) {
    __stcs(reinterpret_cast<float4*>(dst), make_float4(v[0], v[1], v[2], v[3]));
    __stcs(reinterpret_cast<float4*>(dst) + 1, make_float4(v[4], v[5], v[6], v[7]));
  } else if (P == 4) {
    __stcs(reinterpret_cast<float4*>(dst), make_float4(v[0], v[1], v[2], v[3]));
  } else {
    __stcs(dst, v[0]);
  }
}

// E consecutive nonzeros per lane per round (a round = 32 E nonzeros)
template <int E>
struct SpmmRound {
  int col[E];
  float val[E];
};

template <int E>
__device__ __forceinline__ void spmm_load(const SpmmArgs& a, int4 c, int k, int lane, SpmmRound<E>& d) {
  const int g = (c.y & ~7) + 32 * E * k + E * lane;
  if (a.vec && g < c.w && g + E <= a.nnz) {
    if constexpr (E == 4) {
      const int4 ci = ld_cs_v4(a.col + g);
      const float4 vi = ld_cs_v4(a.val + g);
      d.col[0] = ci.x; d.col[1] = ci.y; d.col[2] = ci.z; d.col[3] = ci.w;
      d.val[0] = vi.x; d.val[1] = vi.y; d.val[2] = vi.z; d.val[3] = vi.w;
    } else {
      static_assert(E == 2, "E: 2 or 4 nonzeros per lane");
      const int2 ci = __ldcs(reinterpret_cast<const int2*>(a.col + g));
      const float2 vi = __ldcs(reinterpret_cast<const float2*>(a.val + g));
      d.col[0] = ci.x; d.col[1] = ci.y;
      d.val[0] = vi.x; d.val[1] = vi.y;
    }
  } else {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const bool ok = g + e < c.w;
      d.col[e] = ok ? ld_cs(a.col + g + e) : 0;
      d.val[e] = ok ? ld_cs(a.val + g + e) : 0.f;
    }
  }
}

template <int P, int E>
__device__ __forceinline__ void spmm_gather_round(const SpmmArgs& a, int4 c, int k, int lane, SpmmRound<E>& d,
                                                  PVec<P> (&xv)[E]) {
  const int q0 = 32 * E * k + E * lane, lo = c.y & 7, hi = c.w - (c.y & ~7);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const bool ok = q0 + e >= lo && q0 + e < hi;
    if (ok) spmm_gather<P>(a, d.col[e], xv[e]);
    else {
#pragma unroll
      for (int j = 0; j < P; ++j) xv[e].v[j] = 0.f;
      d.val[e] = 0.f;
    }
  }
}

template <int W, int P, int MINB, int E = 4>
__global__ void __launch_bounds__(W * 32, MINB) merge_spmm_kernel(SpmmArgs a) {
  constexpr int kCap = 1024, R = kCap / (32 * E);  // tile positions, rounds of 32 E per tile (L = 1016)
  constexpr int K = 2;
  __shared__ __align__(16) unsigned short s_tail[W][kCap];
  __shared__ int s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = blockIdx.x * W + warp;
  const int t_begin = min(a.num_tiles, gw * a.tiles_per_warp);
  const int t_end = min(a.num_tiles, t_begin + a.tiles_per_warp);
  unsigned short* tail = s_tail[warp];
  for (int w = lane; w < kCap / 8; w += 32) reinterpret_cast<uint4*>(tail)[w] = make_uint4(0u, 0u, 0u, 0u);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncwarp();

  // reuse the SpMV row pass (it only reads off/coords and writes y = 0 for empty rows: for SpMM the
  // empty rows are written here instead, so give it a TileArgs whose y is unused (nullptr never hit
  // because we handle empty rows ourselves below)
  TileArgs pa;
  pa.off = a.off; pa.coords = a.coords; pa.rows = a.rows; pa.nnz = a.nnz;
  float rc[P], rcc[P];  // the open row's partials, compensated (rc + rcc)
#pragma unroll
  for (int j = 0; j < P; ++j) rc[j] = rcc[j] = 0.f;
  int i_last = t_begin < t_end ? __ldg(&a.coords[t_end].x) : a.rows;
  if (t_begin < t_end) {
    const int nsteps = (t_end - t_begin) * R;
    int4 cT = tile_coords(pa, t_begin);
    int4 cT1 = t_begin + 1 < t_end ? tile_coords(pa, t_begin + 1) : cT;
    int4 cT2 = t_begin + 2 < t_end ? tile_coords(pa, t_begin + 2) : cT1;
    int olo[K], ohi[K];
    // row pass writing empty rows of Y (rows r > 0 without a nonzero in the tile)
    auto row_pass = [&](int4 c) -> bool {
      const int i0 = c.x, nrows = c.z - c.x, jA = c.y & ~7, lo = c.y - jA;
      bool row0_empty = false;
      for (int j = 0; 32 * j < nrows; ++j) {
        const int r = lane + 32 * j;
        if (r < nrows) {
          int ob, oe;
          if (j < K) {
#pragma unroll
            for (int q = 0; q < K; ++q)
              if (q == j) { ob = olo[q]; oe = ohi[q]; }
          } else {
            ob = __ldcs(a.off + i0 + r);
            oe = __ldcs(a.off + i0 + r + 1);
          }
          const int e = oe - jA;
          const int s = r == 0 ? lo : ob - jA;
          if (e > s) tail[e - 1] = (unsigned short)(r + 1);
          else if (r > 0) {
            float z[P];
#pragma unroll
            for (int q = 0; q < P; ++q) z[q] = 0.f;
            spmm_store<P>(a, i0 + r, z);
          } else row0_empty = true;
        }
      }
      return __shfl_sync(kFull, (int)row0_empty, 0) != 0;
    };
    stream_prefetch_offsets<4, K>(pa, cT, lane, olo, ohi);
    bool r0e = row_pass(cT);
    if (t_begin + 1 < t_end) stream_prefetch_offsets<4, K>(pa, cT1, lane, olo, ohi);
    __syncwarp();
    SpmmRound<E> d0, d1, d2;
    PVec<P> x0[E], x1[E];
    spmm_load<E>(a, cT, 0, lane, d0);
    if (1 < nsteps) spmm_load<E>(a, R > 1 ? cT : cT1, R > 1 ? 1 : 0, lane, d1);
    spmm_gather_round<P, E>(a, cT, 0, lane, d0, x0);
    int t = t_begin, k = 0;
    for (int st = 0; st < nsteps; ++st) {
      if (st + 1 < nsteps) {
        const bool same = k + 1 < R;
        spmm_gather_round<P, E>(a, same ? cT : cT1, same ? k + 1 : k + 1 - R, lane, d1, x1);
      }
      if (st + 2 < nsteps) {
        const int k2 = k + 2;
        const bool same = k2 < R;
        spmm_load<E>(a, same ? cT : cT1, same ? k2 : k2 - R, lane, d2);
      }
      const int i0 = cT.x;
      if (k == 0 && r0e) {
        float rv[P];
#pragma unroll
        for (int j = 0; j < P; ++j) rv[j] = rc[j] + rcc[j];
        if (lane == 0) spmm_store<P>(a, i0, rv);
#pragma unroll
        for (int j = 0; j < P; ++j) rc[j] = rcc[j] = 0.f;
      }
      unsigned rid[E];
      uint2 tq = make_uint2(0u, 0u);
      if constexpr (E == 4) {
        tq = *reinterpret_cast<const uint2*>(&tail[128 * k + 4 * lane]);
        rid[0] = tq.x & 0xFFFFu; rid[1] = tq.x >> 16; rid[2] = tq.y & 0xFFFFu; rid[3] = tq.y >> 16;
      } else {
        tq.x = *reinterpret_cast<const unsigned*>(&tail[64 * k + 2 * lane]);
        rid[0] = tq.x & 0xFFFFu; rid[1] = tq.x >> 16;
      }
      float run[P], first_val[P];
#pragma unroll
      for (int j = 0; j < P; ++j) { run[j] = 0.f; first_val[j] = 0.f; }
      int first_r = -1;
#pragma unroll
      for (int e = 0; e < E; ++e) {
#pragma unroll
        for (int j = 0; j < P; ++j) run[j] = fmaf(d0.val[e], x0[e].v[j], run[j]);
        if (rid[e]) {
          const int r = (int)rid[e] - 1;
          if (first_r < 0) {
            first_r = r;
#pragma unroll
            for (int j = 0; j < P; ++j) first_val[j] = run[j];
          } else {
            spmm_store<P>(a, i0 + r, run);
          }
#pragma unroll
          for (int j = 0; j < P; ++j) run[j] = 0.f;
        }
      }
      // segmented scan of the P partial sums (one flag, P values)
      bool f = first_r >= 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int fo = __shfl_up_sync(kFull, (int)f, o);
        float vo[P];
#pragma unroll
        for (int j = 0; j < P; ++j) vo[j] = __shfl_up_sync(kFull, run[j], o);
        if (lane >= o) {
          if (!f) {
#pragma unroll
            for (int j = 0; j < P; ++j) run[j] = vo[j] + run[j];
          }
          f = f || fo;
        }
      }
      const int lf = __shfl_up_sync(kFull, (int)f, 1);
      const int agg_f = __shfl_sync(kFull, (int)f, 31);
      float lval[P], agg_v[P];
#pragma unroll
      for (int j = 0; j < P; ++j) {
        lval[j] = __shfl_up_sync(kFull, run[j], 1);
        agg_v[j] = __shfl_sync(kFull, run[j], 31);
      }
      if (first_r >= 0) {
        float yv[P];
#pragma unroll
        for (int j = 0; j < P; ++j) {
          const float rcs = rc[j] + rcc[j];
          yv[j] = (lane == 0 ? rcs : (lf ? lval[j] : rcs + lval[j])) + first_val[j];
        }
        spmm_store<P>(a, i0 + first_r, yv);
      }
      if (tq.x | tq.y) {
        if constexpr (E == 4) *reinterpret_cast<uint2*>(&tail[128 * k + 4 * lane]) = make_uint2(0u, 0u);
        else *reinterpret_cast<unsigned*>(&tail[64 * k + 2 * lane]) = 0u;
      }
#pragma unroll
      for (int j = 0; j < P; ++j) {
        rc[j] = agg_f ? 0.f : rc[j];
        rcc[j] = agg_f ? 0.f : rcc[j];
        csum_add(rc[j], rcc[j], agg_v[j]);
      }
#pragma unroll
      for (int e = 0; e < E; ++e) {
        d0.val[e] = d1.val[e];
        x0[e] = x1[e];
        d1.col[e] = d2.col[e];
        d1.val[e] = d2.val[e];
      }
      if (++k == R) {
        k = 0;
        ++t;
        __syncwarp();
        if (t < t_end) {
          r0e = row_pass(cT1);
          if (t + 1 < t_end) stream_prefetch_offsets<4, K>(pa, cT2, lane, olo, ohi);
          cT = cT1;
          cT1 = cT2;
          if (t + 2 < t_end) cT2 = tile_coords(pa, t + 2);
        }
      }
      __syncwarp();
    }
  }

  if (lane == 0) {
    a.carry_row[gw] = i_last;
#pragma unroll
    for (int j = 0; j < P; ++j) a.carry_val[(int64_t)gw * P + j] = rc[j] + rcc[j];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned done = atomicAdd(a.ticket, 1u);
    s_last = done == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    const int nc = (int)gridDim.x * W;
    for (int c = threadIdx.x; c < nc; c += W * 32) {
      const int r = __ldcg(a.carry_row + c);
      if (r >= a.rows) continue;
      if (c > 0 && __ldcg(a.carry_row + c - 1) == r) continue;
      float* dst = a.Y + (int64_t)r * a.ldy;
      float sum[P], comp[P];
#pragma unroll
      for (int j = 0; j < P; ++j) { sum[j] = __ldcg(dst + j); comp[j] = 0.f; }
      for (int kk = c; kk < nc && __ldcg(a.carry_row + kk) == r; ++kk)
#pragma unroll
        for (int j = 0; j < P; ++j) csum_add(sum[j], comp[j], __ldcg(a.carry_val + (int64_t)kk * P + j));
#pragma unroll
      for (int j = 0; j < P; ++j) dst[j] = sum[j] + comp[j];
    }
    if (threadIdx.x == 0) *a.ticket = 0u;
  }
}

// ----------------------------------------------------------------------------- SpMM, lanes over columns
// Y = A X for a panel of P (8, 16 or 32) columns on the same merge-path tiles (L = 1016): a warp is
// NG = 32 / P groups of P lanes and lane (g, c) owns column c of the panel.  A round is 32 NG
// consecutive nonzero positions, 32 per group.  The warp loads the round's col/val coalesced (NG
// positions per lane, one 16/8/4-byte load each), zeroes the values outside the tile and stages them
// in a two-slot shared ring; every lane then reads its group's 32 columns / values with broadcast
// 16-byte shared loads and gathers X[col, c] -- the P lanes of a group read one contiguous 4P-byte
// segment per nonzero.  Each lane sums its 32 products in one FMA chain, row ends inside the chain are
// stored directly (P contiguous floats per group), and the open row's partial crosses groups with a
// log2(NG)-step segmented scan that moves values by P lanes (same column).  Row ends come from the
// same per-warp marker buffer as SpMV.  Compared with merge_spmm_kernel (lanes over nonzeros, P values
// per lane), the per-column scans across 32 lanes disappear and a round carries 1024 products.
template <int P>
__device__ __forceinline__ void spmm_zero_row(const SpmmArgs& a, int row) {
  float4* dst = reinterpret_cast<float4*>(a.Y + (int64_t)row * a.ldy);
#pragma unroll
  for (int q = 0; q < P / 4; ++q) __stcs(dst + q, make_float4(0.f, 0.f, 0.f, 0.f));
}

template <int NG>
struct SpmmColsLoad {  // one lane's share of a round: NG consecutive positions
  int col[NG];
  float val[NG];
};

// dynamic shared memory of merge_spmm_cols_kernel<W, R, P> (the col/val staging ring)
__host__ __device__ constexpr int spmm_cols_dyn_bytes(int W, int P) { return W * 2 * (32 / P) * 36 * 4 * 2; }

template <int W, int R, int P>
__global__ void __launch_bounds__(W * 32, 1) merge_spmm_cols_kernel(SpmmArgs a) {
  static_assert(P == 8 || P == 16 || P == 32, "P");
  constexpr int NG = 32 / P;              // groups per warp
  constexpr int EG = 32;                  // positions per group per round
  constexpr int kCap = 256 * R;           // tile positions (L = kCap - 8)
  constexpr int RP = EG * NG;             // positions per round
  constexpr int RT = kCap / RP;           // rounds per tile
  constexpr int GS = EG + 4;              // padded group stride of the staging ring (words)
  constexpr int K = 2;
  __shared__ __align__(16) unsigned short s_tail[W][kCap];
  __shared__ int s_last;
  // staging ring in dynamic shared memory: [W][2 slots][NG * GS] columns, then the same for values
  extern __shared__ __align__(16) int s_dyn[];
  int (*s_col)[2][NG * GS] = reinterpret_cast<int (*)[2][NG * GS]>(s_dyn);
  float (*s_val)[2][NG * GS] = reinterpret_cast<float (*)[2][NG * GS]>(s_dyn + W * 2 * NG * GS);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / P, cl = lane % P;
  const int gw = blockIdx.x * W + warp;
  const int t_begin = min(a.num_tiles, gw * a.tiles_per_warp);
  const int t_end = min(a.num_tiles, t_begin + a.tiles_per_warp);
  const uint64_t spol = policy_evict_first();
  unsigned short* tail = s_tail[warp];
  for (int w = lane; w < kCap / 8; w += 32) reinterpret_cast<uint4*>(tail)[w] = make_uint4(0u, 0u, 0u, 0u);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncwarp();

  TileArgs pa;
  pa.off = a.off; pa.coords = a.coords; pa.rows = a.rows; pa.nnz = a.nnz;
  float rc = 0.f, rcc = 0.f;  // partial of the open row, column cl (the same in every group), compensated
  int i_last = t_begin < t_end ? __ldg(&a.coords[t_end].x) : a.rows;
  if (t_begin < t_end) {
    const float* __restrict__ Xc = a.X + cl;
    const int nsteps = (t_end - t_begin) * RT;
    int4 cT = tile_coords(pa, t_begin);
    int4 cT1 = t_begin + 1 < t_end ? tile_coords(pa, t_begin + 1) : cT;
    int4 cT2 = t_begin + 2 < t_end ? tile_coords(pa, t_begin + 2) : cT1;
    int olo[K], ohi[K];
    bool r0e = false;  // (warp-uniform) row i0 of the current tile has no nonzero in it
    // row pass: marks row ends in tail[], writes the zero rows (rows r > 0 without a nonzero here)
    auto row_pass = [&](int4 c) -> bool {
      const int i0 = c.x, nrows = c.z - c.x, jA = c.y & ~7, lo = c.y - jA;
      bool row0_empty = false;
      for (int j = 0; 32 * j < nrows; ++j) {
        const int r = lane + 32 * j;
        if (r < nrows) {
          int ob, oe;
          if (j < K) {
#pragma unroll
            for (int q = 0; q < K; ++q)
              if (q == j) { ob = olo[q]; oe = ohi[q]; }
          } else {
            ob = __ldcs(a.off + i0 + r);
            oe = __ldcs(a.off + i0 + r + 1);
          }
          const int e = oe - jA;
          const int s = r == 0 ? lo : ob - jA;
          if (e > s) tail[e - 1] = (unsigned short)(r + 1);
          else if (r > 0) spmm_zero_row<P>(a, i0 + r);
          else row0_empty = true;
        }
      }
      return __shfl_sync(kFull, (int)row0_empty, 0) != 0;
    };
    // this lane's NG positions of round kk of tile c; values outside the tile's nonzero range are 0
    auto load = [&](int4 c, int kk, SpmmColsLoad<NG>& d) {
      const int jA = c.y & ~7;
      const int q0 = RP * kk + NG * lane;  // tile-local position
      const int g = jA + q0;
      const int lo = c.y - jA, hi = c.w - jA;
      if (g + NG <= c.w && g + NG <= a.nnz) {
        if constexpr (NG == 4) {
          const int4 ci = ld_cs_v4(a.col + g);
          const float4 vi = ld_cs_v4(a.val + g);
          d.col[0] = ci.x; d.col[1] = ci.y; d.col[2] = ci.z; d.col[3] = ci.w;
          d.val[0] = vi.x; d.val[1] = vi.y; d.val[2] = vi.z; d.val[3] = vi.w;
        } else if constexpr (NG == 2) {
          const int2 ci = __ldcs(reinterpret_cast<const int2*>(a.col + g));
          const float2 vi = __ldcs(reinterpret_cast<const float2*>(a.val + g));
          d.col[0] = ci.x; d.col[1] = ci.y;
          d.val[0] = vi.x; d.val[1] = vi.y;
        } else {
          d.col[0] = ld_cs(a.col + g);
          d.val[0] = ld_cs(a.val + g);
        }
      } else {
#pragma unroll
        for (int e = 0; e < NG; ++e) {
          const bool ok = g + e < c.w;
          d.col[e] = ok ? ld_cs(a.col + g + e) : 0;
          d.val[e] = ok ? ld_cs(a.val + g + e) : 0.f;
        }
      }
#pragma unroll
      for (int e = 0; e < NG; ++e)
        if (q0 + e < lo || q0 + e >= hi) d.val[e] = 0.f;
    };
    // stage a loaded round into ring slot sl: position q of the round -> group q / 32, index q % 32
    auto stage = [&](const SpmmColsLoad<NG>& d, int sl) {
      const int q = NG * lane, gq = q / EG, eq = q % EG;
      int* dc = &s_col[warp][sl][gq * GS + eq];
      float* dv = &s_val[warp][sl][gq * GS + eq];
      if constexpr (NG == 4) {
        *reinterpret_cast<int4*>(dc) = make_int4(d.col[0], d.col[1], d.col[2], d.col[3]);
        *reinterpret_cast<float4*>(dv) = make_float4(d.val[0], d.val[1], d.val[2], d.val[3]);
      } else if constexpr (NG == 2) {
        *reinterpret_cast<int2*>(dc) = make_int2(d.col[0], d.col[1]);
        *reinterpret_cast<float2*>(dv) = make_float2(d.val[0], d.val[1]);
      } else {
        *dc = d.col[0];
        *dv = d.val[0];
      }
    };
    // the group's 32 gathers of the round staged in slot sl
    const int ldx = (int)a.ldx, ldy = (int)a.ldy;  // < 2^31 (checked by the launcher): one IMAD.WIDE per address
    auto gather = [&](int sl, float (&xv)[EG]) {
      const int* sc = &s_col[warp][sl][grp * GS];
#pragma unroll
      for (int e = 0; e < EG; e += 4) {
        const int4 c4 = *reinterpret_cast<const int4*>(sc + e);
        xv[e] = __ldg(Xc + (int64_t)c4.x * ldx);
        xv[e + 1] = __ldg(Xc + (int64_t)c4.y * ldx);
        xv[e + 2] = __ldg(Xc + (int64_t)c4.z * ldx);
        xv[e + 3] = __ldg(Xc + (int64_t)c4.w * ldx);
      }
    };
    auto reduce = [&](int kk, int sl, const float (&xc)[EG]) {
      const int i0 = cT.x;
      if (kk == 0 && r0e) {
        if (grp == 0) a.Y[(int64_t)i0 * a.ldy + cl] = rc + rcc;
        rc = rcc = 0.f;
      }
      const float* sv = &s_val[warp][sl][grp * GS];
      const unsigned short* tg = &tail[RP * kk + EG * grp];
      float* yt = a.Y + (int64_t)(i0 - 1) * ldy + cl;  // row r of the tile ends where rid = r + 1
      unsigned first_rid = 0u;
      float run = 0.f, first_val = 0.f;
#pragma unroll
      for (int e8 = 0; e8 < EG; e8 += 8) {
        const uint4 tq = *reinterpret_cast<const uint4*>(tg + e8);
        const float4 v0 = *reinterpret_cast<const float4*>(sv + e8);
        const float4 v1 = *reinterpret_cast<const float4*>(sv + e8 + 4);
        const float vv[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
        if ((tq.x | tq.y | tq.z | tq.w) == 0u) {  // no row ends in these 8 (group-uniform): FMAs only
#pragma unroll
          for (int e = 0; e < 8; ++e) run = fmaf(vv[e], xc[e8 + e], run);
          continue;
        }
        const unsigned w4[4] = {tq.x, tq.y, tq.z, tq.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          run = fmaf(vv[e], xc[e8 + e], run);
          const unsigned rid = (e & 1) ? (w4[e >> 1] >> 16) : (w4[e >> 1] & 0xFFFFu);
          if (rid != 0u) {  // group-uniform
            if (first_rid != 0u) __stcs(yt + (int64_t)(int)rid * ldy, run);
            else { first_val = run; first_rid = rid; }
            run = 0.f;
          }
        }
      }
      // group flags: bit j set when group j has a row end in this round
      const unsigned B = __ballot_sync(kFull, first_rid != 0u);
      unsigned GF = 0u;
#pragma unroll
      for (int j = 0; j < NG; ++j) GF |= ((B >> (j * P)) & 1u) << j;
      float v = run;
#pragma unroll
      for (int o = 1; o < NG; o <<= 1) {
        const float vo = __shfl_up_sync(kFull, v, o * P);
        const bool reset = grp >= o ? ((GF >> (grp - o + 1)) & ((1u << o) - 1u)) != 0u : true;
        if (!reset) v = vo + v;
      }
      const float lval = __shfl_up_sync(kFull, v, P % 32);
      const float agg_v = __shfl_sync(kFull, v, (NG - 1) * P + cl);
      if (first_rid != 0u) {
        const bool lf = (GF & ((1u << grp) - 1u)) != 0u;  // a row ended in an earlier group
        const float rcs = rc + rcc;
        const float carry_in = grp == 0 ? rcs : (lf ? lval : rcs + lval);
        a.Y[(int64_t)(i0 - 1 + (int)first_rid) * a.ldy + cl] = carry_in + first_val;
      }
      rc = GF ? 0.f : rc;
      rcc = GF ? 0.f : rcc;
      csum_add(rc, rcc, agg_v);
    };
    stream_prefetch_offsets<R, K>(pa, cT, lane, olo, ohi);
    r0e = row_pass(cT);
    if (t_begin + 1 < t_end) stream_prefetch_offsets<R, K>(pa, cT1, lane, olo, ohi);
    // pipeline: step st stages round st+1 (loaded during step st-1) and issues its gathers, loads
    // round st+2 into registers, and reduces round st (staged and gathered during step st-1)
    SpmmColsLoad<NG> ld;
    float X0[EG], X1[EG];
    load(cT, 0, ld);
    stage(ld, 0);
    if (1 < nsteps) load(RT > 1 ? cT : cT1, RT > 1 ? 1 : 0, ld);
    __syncwarp();
    gather(0, X0);
    int t = t_begin, k = 0, st = 0;
    auto step = [&](float (&xc)[EG], float (&xn)[EG]) {
      const int sl = st & 1;
      if (st + 1 < nsteps) {
        stage(ld, sl ^ 1);
        __syncwarp();
        gather(sl ^ 1, xn);
      }
      if (st + 2 < nsteps) {
        const int k2 = k + 2;
        const int4 c2 = k2 < RT ? cT : (k2 < 2 * RT ? cT1 : cT2);
        load(c2, k2 < RT ? k2 : (k2 < 2 * RT ? k2 - RT : k2 - 2 * RT), ld);
      }
      reduce(k, sl, xc);
      if (++k == RT) {
        k = 0;
        ++t;
        __syncwarp();
        for (int w = lane; w < kCap / 8; w += 32) reinterpret_cast<uint4*>(tail)[w] = make_uint4(0u, 0u, 0u, 0u);
        __syncwarp();
        if (t < t_end) {
          r0e = row_pass(cT1);
          if (t + 1 < t_end) stream_prefetch_offsets<R, K>(pa, cT2, lane, olo, ohi);
          cT = cT1;
          cT1 = cT2;
          if (t + 2 < t_end) cT2 = tile_coords(pa, t + 2);
        }
      }
      __syncwarp();
    };
    // one copy of the step (the code of a round is large: two rotated copies thrashed the instruction
    // cache), the gathered round moved into place with register copies
    for (; st < nsteps; ++st) {
      step(X0, X1);
#pragma unroll
      for (int e = 0; e < EG; ++e) X0[e] = X1[e];
    }
  }

  if (grp == 0) {
    if (cl == 0) a.carry_row[gw] = i_last;
    a.carry_val[(int64_t)gw * P + cl] = rc + rcc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned done = atomicAdd(a.ticket, 1u);
    s_last = done == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    const int nc = (int)gridDim.x * W;
    // one (carry, column) pair per thread: carries of equal rows are summed in warp order
    for (int u = threadIdx.x; u < nc * P; u += W * 32) {
      const int c = u / P, j = u % P;
      const int r = __ldcg(a.carry_row + c);
      if (r >= a.rows) continue;
      if (c > 0 && __ldcg(a.carry_row + c - 1) == r) continue;
      float* dst = a.Y + (int64_t)r * a.ldy + j;
      float sum = __ldcg(dst), comp = 0.f;
      for (int kk = c; kk < nc && __ldcg(a.carry_row + kk) == r; ++kk)
        csum_add(sum, comp, __ldcg(a.carry_val + (int64_t)kk * P + j));
      *dst = sum + comp;
    }
    if (threadIdx.x == 0) *a.ticket = 0u;
  }
}

}  // namespace lbk
