// k_merge.cuh -- sm_100a device code (arXiv 2212.08964).  Citations "P:L" = PAPER.md line L.
// a3 + a4: the merge-path tile processors (warp-streamed, CTA-wide, unaligned fallback) and the
// stream / stream+gather ceiling probes.
#pragma once
#include "dev_common.cuh"

namespace lbk {

// ----------------------------------------------------------------------------- merge-path tiles
template <int NT, int L, bool VEC>
struct MergeCfg {
  static constexpr int kSlots = (L + 6) / 4;                // 4-wide slots covering [j0&~3, j1)
  static constexpr int kNV = (kSlots + NT - 1) / NT;        // slots per thread
  static constexpr int kWarps = NT / 32;
  static constexpr int kChunks = kNV * kWarps;              // 128-nonzero chunks per tile
  static constexpr int kTailWords = (4 * kSlots + 31) / 32;
  static_assert(kChunks <= 32, "chunk scan uses one warp");
  struct Smem {
    unsigned tail[2][kTailWords];  // bit q set: local nonzero q (from j0&~3) ends its row
    int rowend[2][L];              // local end (exclusive) of each row ending in the tile
    float out[2][4 * kSlots];      // row sum at its last nonzero (tail positions only)
    int cflag[kChunks];
    float cval[kChunks];
  };
};

// Persistent merge-path tile processor (Alg.3, per-tile reading R3-R5).
template <int NT, int L, bool VEC>
__global__ void __launch_bounds__(NT, 3) merge_tile_kernel(TileArgs a) {
  using Cfg = MergeCfg<NT, L, VEC>;
  constexpr int NV = Cfg::kNV;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  typename Cfg::Smem& sm = *reinterpret_cast<typename Cfg::Smem*>(smem_raw);

  const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t_begin = blockIdx.x * a.tiles_per_cta;
  const int t_end = min(a.num_tiles, t_begin + a.tiles_per_cta);

  for (int w = tid; w < 2 * Cfg::kTailWords; w += NT) (&sm.tail[0][0])[w] = 0u;
  __syncthreads();

  // partial of the row open at the start of the current tile (this CTA's share), compensated
  float cta_s = 0.f, cta_c = 0.f;
  int i_last = 0;
  for (int t = t_begin; t < t_end; ++t) {
    const int b = t & 1;
    const int2 c0 = a.coords[t], c1 = a.coords[t + 1];
    const int i0 = c0.x, j0 = c0.y, i1 = c1.x, j1 = c1.y;
    const int nrows = i1 - i0;
    const int jA = j0 & ~3;
    const int nslots = (j1 - jA + 3) >> 2;
    const int lo = j0 - jA, hi = j1 - jA;  // valid local positions [lo, hi)

    // (1) stream this thread's column indices / values (evict-first)
    int cidx[NV][4];
    float vals[NV][4];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int s = v * NT + tid;
      const int g = jA + 4 * s;
      if (s < nslots) {
        if (VEC && g + 4 <= a.nnz) {
          int4 ci = ld_cs_v4(a.col + g);
          float4 vi = ld_cs_v4(a.val + g);
          cidx[v][0] = ci.x; cidx[v][1] = ci.y; cidx[v][2] = ci.z; cidx[v][3] = ci.w;
          vals[v][0] = vi.x; vals[v][1] = vi.y; vals[v][2] = vi.z; vals[v][3] = vi.w;
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const bool ok = g + e < a.nnz && 4 * s + e >= lo;
            cidx[v][e] = ok ? ld_cs(a.col + g + e) : 0;
            vals[v][e] = ok ? ld_cs(a.val + g + e) : 0.f;
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) { cidx[v][e] = 0; vals[v][e] = 0.f; }
      }
    }
    // (2) gather x for valid positions (all gathers issued before any use)
    float xv[NV][4];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int q0 = 4 * (v * NT + tid);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int q = q0 + e;
        const bool ok = q >= lo && q < hi;
        xv[v][e] = ok ? ld_x(a.x + cidx[v][e]) : 0.f;
        if (!ok) vals[v][e] = 0.f;  // masked positions contribute exactly nothing
      }
    }
    // (3) row ends of the tile -> tail bits + local ends (rows [i0, i1))
    for (int r = tid; r < nrows; r += NT) {
      const int e = __ldg(a.off + i0 + 1 + r) - jA;
      const int s = r == 0 ? lo : __ldg(a.off + i0 + r) - jA;
      sm.rowend[b][r] = e;
      if (e > s) atomicOr(&sm.tail[b][(e - 1) >> 5], 1u << ((e - 1) & 31));
    }
    __syncthreads();

    // (4) per-thread segmented sums over its 4-wide slots, then warp segmented scan
    float tv[NV][4];       // value at each tail (before the carry-in of the first tail)
    unsigned tails[NV];    // 4-bit tail mask per slot
    bool lflag[NV];        // exclusive (lane) prefix flag
    float lval[NV];        // exclusive (lane) prefix value
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int q0 = 4 * (v * NT + tid);
      const unsigned word = q0 < 4 * Cfg::kSlots ? sm.tail[b][q0 >> 5] : 0u;
      const unsigned f4 = (word >> (q0 & 31)) & 0xFu;
      tails[v] = f4;
      float run = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        run = fmaf(vals[v][e], xv[v][e], run);
        tv[v][e] = run;
        if ((f4 >> e) & 1u) run = 0.f;
      }
      bool f = f4 != 0u;
      float val = run;
      warp_segscan_incl(f, val, lane);
      // exclusive prefix for this lane
      float ev = __shfl_up_sync(kFull, val, 1);
      int ef = __shfl_up_sync(kFull, (int)f, 1);
      lflag[v] = lane ? (bool)ef : false;
      lval[v] = lane ? ev : 0.f;
      if (lane == 31) {
        sm.cflag[v * Cfg::kWarps + warp] = f;
        sm.cval[v * Cfg::kWarps + warp] = val;
      }
    }
    __syncthreads();

    // (5) chunk-level scan (chunk c = v*warps + warp covers local nonzeros [128c, 128c+128))
    bool cf = lane < (unsigned)Cfg::kChunks ? (bool)sm.cflag[lane] : false;
    float cv = lane < (unsigned)Cfg::kChunks ? sm.cval[lane] : 0.f;
    warp_segscan_incl(cf, cv, lane);
    const float agg_val = __shfl_sync(kFull, cv, Cfg::kChunks - 1);
    float ex_v = __shfl_up_sync(kFull, cv, 1);
    int ex_f = __shfl_up_sync(kFull, (int)cf, 1);
    if (lane == 0) { ex_v = 0.f; ex_f = 0; }
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const float chunk_in = __shfl_sync(kFull, ex_v, v * Cfg::kWarps + warp);
      const float carry_in = lflag[v] ? lval[v] : chunk_in + lval[v];
      const int q0 = 4 * (v * NT + tid);
      bool first = true;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if ((tails[v] >> e) & 1u) {
          sm.out[b][q0 + e] = first ? carry_in + tv[v][e] : tv[v][e];
          first = false;
        }
      }
    }
    (void)ex_f;
    // this buffer's tail bits are no longer read: clear them for tile t+2
    for (int w = tid; w < Cfg::kTailWords; w += NT) sm.tail[b][w] = 0u;
    __syncthreads();

    // (6) rows ending in this tile: y[r] = row sum within the tile (+ this CTA's carry for
    //     the first row); coalesced stores (Alg.3 P:321 "y[row] <- running_total")
    for (int r = tid; r < nrows; r += NT) {
      const int e = sm.rowend[b][r];
      const int s = r == 0 ? lo : sm.rowend[b][r - 1];
      float yv = e > s ? sm.out[b][e - 1] : 0.f;
      if (r == 0) {
        float cs = cta_s, cc = cta_c;
        csum_add(cs, cc, yv);
        yv = cs + cc;
      }
      a.y[i0 + r] = yv;
    }
    // (7) carry the open row (i1) to the next tile of this CTA (Alg.3)
    if (nrows > 0) { cta_s = agg_val; cta_c = 0.f; }
    else csum_add(cta_s, cta_c, agg_val);
    i_last = i1;
  }
  if (tid == 0 && t_begin < t_end) {
    a.carry_row[blockIdx.x] = i_last;
    a.carry_val[blockIdx.x] = cta_s + cta_c;
  }
}

// Fix-up (Alg.3) of merge_tile_kernel: y[row] += the carries of the CTAs whose runs ended
// inside `row`, in CTA order, compensated (fixup_carries); one thread per carry.
__global__ void fixup_kernel(TileArgs a, int n) {
  fixup_carries(a, n, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

// ----------------------------------------------------------------------------- merge-path tiles, wide
// CTA tiles: each thread owns E = 8 or 16 contiguous nonzeros of the tile, read
// with 256-bit loads (sm_100a LDG.256, L1 no-allocate, L2 evict-first): the per-tile scans and
// barriers are amortised over 2-4x more nonzeros, and a warp still reads whole 32-byte sectors.
// Tile length L = NT*E - 8: the 32-byte-aligned nonzero range [j0&~7, j1) spans <= L + 7.

template <int E>
struct WideTile {
  int i0, j0, i1, j1;
  int col[E];
  float val[E];
  int off_lo, off_hi;
};

template <int NT, int E>
__device__ __forceinline__ void wide_load(const TileArgs& a, int4 c, int tid, WideTile<E>& d, uint64_t spol) {
  d.i0 = c.x; d.j0 = c.y; d.i1 = c.z; d.j1 = c.w;  // coords prefetched one tile earlier
  const int g = (d.j0 & ~7) + E * tid;
  if (g < d.j1 && g + E <= a.nnz) {
#pragma unroll
    for (int k = 0; k < E / 8; ++k) {
      int ci[8];
      float vi[8];
      ld_stream_v8(a.col + g + 8 * k, ci, spol);
      ld_stream_v8(a.val + g + 8 * k, vi, spol);
#pragma unroll
      for (int e = 0; e < 8; ++e) { d.col[8 * k + e] = ci[e]; d.val[8 * k + e] = vi[e]; }
    }
  } else {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const bool ok = g + e < d.j1;
      d.col[e] = ok ? ld_cs(a.col + g + e) : 0;
      d.val[e] = ok ? ld_cs(a.val + g + e) : 0.f;
    }
  }
  if (tid < d.i1 - d.i0) {
    d.off_lo = __ldg(a.off + d.i0 + tid);
    d.off_hi = __ldg(a.off + d.i0 + tid + 1);
  }
}


// x gathers for valid positions; the gathered value replaces col (as float bits) to save registers
template <int E>
__device__ __forceinline__ void wide_gather(const TileArgs& a, WideTile<E>& d, int tid, float (&xv)[E]) {
  const int q0 = E * tid, lo = d.j0 & 7, hi = d.j1 - (d.j0 & ~7);
  if (q0 >= lo && q0 + E <= hi) {  // interior thread: no masking
#pragma unroll
    for (int e = 0; e < E; ++e) xv[e] = ld_x(a.x + d.col[e]);
  } else {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const bool ok = q0 + e >= lo && q0 + e < hi;
      xv[e] = ok ? ld_x(a.x + d.col[e]) : 0.f;
      if (!ok) d.val[e] = 0.f;
    }
  }
}

template <int NT, int E, int MINB>
__global__ void __launch_bounds__(NT, MINB) merge_wide_kernel(TileArgs a) {
  constexpr int kW = NT / 32;
  constexpr int kCap = E * NT;
  static_assert(E == 8 || E == 16, "E");
  __shared__ __align__(16) unsigned short s_tailrow[2][kCap];
  __shared__ int s_cflag[kW];
  __shared__ float s_cval[kW];
  __shared__ int s_last;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t_begin = blockIdx.x * a.tiles_per_cta;
  const int t_end = min(a.num_tiles, t_begin + a.tiles_per_cta);
  const uint64_t spol = policy_evict_first();
  for (int w = tid; w < 2 * kCap; w += NT) (&s_tailrow[0][0])[w] = 0;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: coords are read below
  __syncthreads();

  WideTile<E> cur, nxt;
  float xv[E];
  int4 c_next = make_int4(0, 0, 0, 0);  // coords of tile t+1 (prefetched during tile t-1)
  if (t_begin < t_end) {
    wide_load<NT, E>(a, tile_coords(a, t_begin), tid, cur, spol);
    if (t_begin + 1 < t_end) c_next = tile_coords(a, t_begin + 1);
    wide_gather<E>(a, cur, tid, xv);
  }
  float cta_s = 0.f, cta_c = 0.f;  // partial of the open row over this CTA's tiles, compensated
  int i_last = 0;
  // reduce tile t (`cur`, gathers in xv) while tile t+1 (`nxt`) streams in and gets gathered
  for (int t = t_begin; t < t_end; ++t) {
    const int b = (t - t_begin) & 1;
    const int i0 = cur.i0, nrows = cur.i1 - cur.i0;
    const int jA = cur.j0 & ~7, lo = cur.j0 - jA;
    for (int r = tid; r < nrows; r += NT) {
      const int ob = r == tid ? cur.off_lo : __ldg(a.off + i0 + r);
      const int oe = r == tid ? cur.off_hi : __ldg(a.off + i0 + r + 1);
      const int e = oe - jA;
      const int s = r == 0 ? lo : ob - jA;
      if (e > s) s_tailrow[b][e - 1] = (unsigned short)(r + 1);
      else a.y[i0 + r] = r == 0 ? cta_s + cta_c : 0.f;
    }
    const bool has_next = t + 1 < t_end;
    if (has_next) wide_load<NT, E>(a, c_next, tid, nxt, spol);
    if (t + 2 < t_end) c_next = tile_coords(a, t + 2);
    __syncthreads();

    unsigned tr[E / 2];
#pragma unroll
    for (int k = 0; k < E / 8; ++k) {
      const uint4 q = *reinterpret_cast<const uint4*>(&s_tailrow[b][E * tid + 8 * k]);
      tr[4 * k] = q.x; tr[4 * k + 1] = q.y; tr[4 * k + 2] = q.z; tr[4 * k + 3] = q.w;
    }
    unsigned any = 0u;
#pragma unroll
    for (int k = 0; k < E / 2; ++k) any |= tr[k];
    float run = 0.f, first_val = 0.f;
    int first_r = -1;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      run = fmaf(cur.val[e], xv[e], run);
      const unsigned rid = (e & 1) ? (tr[e >> 1] >> 16) : (tr[e >> 1] & 0xFFFFu);
      if (rid) {
        const int r = (int)rid - 1;
        if (first_r < 0) { first_r = r; first_val = run; }
        else a.y[i0 + r] = run;
        run = 0.f;
      }
    }
    bool f = first_r >= 0;
    float val = run;
    warp_segscan_incl(f, val, (unsigned)lane);
    float lval = __shfl_up_sync(kFull, val, 1);
    const int lf = __shfl_up_sync(kFull, (int)f, 1);
    const bool lflag = lane ? (bool)lf : false;
    if (lane == 0) lval = 0.f;
    if (lane == 31) { s_cflag[warp] = f; s_cval[warp] = val; }
    if (has_next) wide_gather<E>(a, nxt, tid, xv);  // next tile's gathers out before the barrier
    __syncthreads();

    bool cf = lane < kW ? (bool)s_cflag[lane] : false;
    float cv = lane < kW ? s_cval[lane] : 0.f;
    warp_segscan_incl_n<kW>(cf, cv, (unsigned)lane);
    const float agg_val = __shfl_sync(kFull, cv, kW - 1);
    float ex_v = __shfl_up_sync(kFull, cv, 1);
    if (lane == 0) ex_v = 0.f;
    const float chunk_in = __shfl_sync(kFull, ex_v, warp);
    if (first_r >= 0) {
      float yv = (lflag ? lval : chunk_in + lval) + first_val;
      if (first_r == 0) {
        float cs = cta_s, cc = cta_c;
        csum_add(cs, cc, yv);
        yv = cs + cc;
      }
      a.y[i0 + first_r] = yv;
    }
    if (any) {
#pragma unroll
      for (int k = 0; k < E / 8; ++k)
        *reinterpret_cast<uint4*>(&s_tailrow[b][E * tid + 8 * k]) = make_uint4(0u, 0u, 0u, 0u);
    }
    if (nrows > 0) { cta_s = agg_val; cta_c = 0.f; }
    else csum_add(cta_s, cta_c, agg_val);
    i_last = cur.i1;
    cur = nxt;
  }

  if (tid == 0) {
    if (t_begin < t_end) {
      a.carry_row[blockIdx.x] = i_last;
      a.carry_val[blockIdx.x] = cta_s + cta_c;
    }
    __threadfence();
    const unsigned done = atomicAdd(a.ticket, 1u);
    s_last = done == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    fixup_carries_blocked(a, (int)gridDim.x, tid, NT);
    if (tid == 0) *a.ticket = 0u;
  }
}

// ----------------------------------------------------------------------------- merge-path tiles, short rows
// CTA tiles of L = 8*NT - 8 merge items ("first splitting the work across blocks, and then to threads
// within a block") with the tile's products staged in shared memory:
//  1. thread t owns the 8 contiguous nonzero positions [8t, 8t+8) of the tile's 32-byte-aligned range
//     (one 256-bit load each of col_idx / values, evict-first), gathers x and stores the 8 products;
//  2. thread t then sums rows i0 + t, i0 + t + NT, ... of the tile over the staged products -- every
//     row end is one thread's, y stores are coalesced, and there is no segmented scan at all;
//  3. rows holding more than kSeq products in the tile are queued and summed by one warp each (lanes
//     stride the row, fixed xor tree), so a long row never serialises a thread.
// Row "nrows" of a tile is the open row (i1): its partial becomes the carry into the CTA's next tile
// (shared memory, compensated 2Sum pair), and the CTA's last carry goes to the last-CTA fix-up
// (Alg.3, fixup_carries).  The products and the long-row queue are double-buffered, so a
// tile costs two CTA barriers.  Accuracy: a row's part in one tile is <= kSeq sequential terms or
// <= 2L/32 per lane + a 5-level tree; parts of a row across tiles / CTAs are 2Sum-compensated.
// For matrices with short rows (C2 stencil: 5 products per row) this replaces the position-split
// segmented scans of merge_wide_kernel, whose row ends cost most of its instructions.
template <int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) merge_rows_kernel(TileArgs a) {
  constexpr int kCap = 8 * NT, kW = NT / 32, kSeq = 32, kLongMax = kCap / (kSeq + 1) + 2;
  __shared__ __align__(16) float s_prod[2][kCap];
  __shared__ int s_long[2][kLongMax];
  __shared__ int s_nlong[2];
  __shared__ float s_carry[2][2];  // [tile parity][sum, compensation] of the open row
  __shared__ int s_last;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t_begin = blockIdx.x * a.tiles_per_cta;
  const int t_end = min(a.num_tiles, t_begin + a.tiles_per_cta);
  const uint64_t spol = policy_evict_first();
  const uint64_t opol = a.off_keep ? policy_evict_last() : spol;
  if (tid < 2) {
    s_nlong[tid] = 0;
    s_carry[tid][0] = 0.f;
    s_carry[tid][1] = 0.f;
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: coords are read below

  // this thread's 8 positions of the tile's col/val, loaded one tile ahead
  int col[8];
  float val[8];
  auto load = [&](int4 c) {
    const int g = (c.y & ~7) + 8 * tid;
    if (g < c.w && g + 8 <= a.nnz) {
      ld_stream_v8(a.col + g, col, spol);
      ld_stream_v8(a.val + g, val, spol);
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const bool ok = g + e < c.w;
        col[e] = ok ? ld_cs(a.col + g + e) : 0;
        val[e] = ok ? ld_cs(a.val + g + e) : 0.f;
      }
    }
  };

  int4 cur = make_int4(0, 0, 0, 0), nxt = cur;
  if (t_begin < t_end) {
    cur = tile_coords(a, t_begin);
    load(cur);
    if (t_begin + 1 < t_end) nxt = tile_coords(a, t_begin + 1);
  }
  int i_last = cur.z;
  for (int t = t_begin; t < t_end; ++t) {
    const int b = (t - t_begin) & 1;
    const int i0 = cur.x, nrows = cur.z - cur.x, jA = cur.y & ~7, lo = cur.y - jA, hi = cur.w - jA;
    // (1) products of this thread's 8 positions (outside [lo, hi): exactly 0)
    float p[8];
    {
      const int q0 = 8 * tid;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const bool ok = q0 + e >= lo && q0 + e < hi;
        p[e] = ok ? val[e] * ld_x(a.x + col[e]) : 0.f;
      }
    }
    // the next tile's col/val stream in while this tile is reduced
    const int i_end = cur.z;
    if (t + 1 < t_end) {
      cur = nxt;
      load(cur);
      if (t + 2 < t_end) nxt = tile_coords(a, t + 2);
    }
    float4* sp = reinterpret_cast<float4*>(&s_prod[b][8 * tid]);
    sp[0] = make_float4(p[0], p[1], p[2], p[3]);
    sp[1] = make_float4(p[4], p[5], p[6], p[7]);
    __syncthreads();  // (A) products (and the previous tile's carry) visible
    if (tid == 0) s_nlong[b ^ 1] = 0;  // the previous tile's queue count was read before (A)

    // (2) rows of the tile, one thread each; r == nrows is the open row (its partial is the carry)
    const float* pr = s_prod[b];
    auto bounds = [&](int r, int& s, int& e) {
      s = r == 0 ? lo : ld_off(a.off + i0 + r, opol) - jA;
      e = r < nrows ? ld_off(a.off + i0 + r + 1, opol) - jA : hi;
    };
    auto finish = [&](int r, float v) {
      float cs = v, cc = 0.f;
      if (r == 0) {  // carry of the row open at the tile start (previous tile of this CTA)
        cs = s_carry[b ^ 1][0];
        cc = s_carry[b ^ 1][1];
        csum_add(cs, cc, v);
      }
      if (r < nrows) {
        a.y[i0 + r] = cs + cc;
      } else {
        s_carry[b][0] = cs;
        s_carry[b][1] = cc;
      }
    };
    for (int r = tid; r <= nrows; r += NT) {
      int s, e;
      bounds(r, s, e);
      if (e - s > kSeq) {
        s_long[b][atomicAdd(&s_nlong[b], 1)] = r;
        continue;
      }
      float v = 0.f;
      for (int q = s; q < e; ++q) v += pr[q];
      finish(r, v);
    }
    // (3) long rows: one warp each
    __syncthreads();  // (B) the queue is complete
    const int nl = s_nlong[b];
    if (nl > 0) {
      for (int k = warp; k < nl; k += kW) {
        const int r = s_long[b][k];
        int s, e;
        bounds(r, s, e);
        float v = 0.f;
        for (int q = s + lane; q < e; q += 32) v += pr[q];
        v = warp_sum(v);
        if (lane == 0) finish(r, v);
      }
    }
    i_last = i_end;
  }
  __syncthreads();  // the last tile's carry is written

  if (tid == 0) {
    if (t_begin < t_end) {
      const int bl = (t_end - 1 - t_begin) & 1;
      a.carry_row[blockIdx.x] = i_last;
      a.carry_val[blockIdx.x] = s_carry[bl][0] + s_carry[bl][1];
    }
    __threadfence();
    const unsigned done = atomicAdd(a.ticket, 1u);
    s_last = done == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    fixup_carries_blocked(a, (int)gridDim.x, tid, NT);
    if (tid == 0) *a.ticket = 0u;
  }
}

// ----------------------------------------------------------------------------- merge-path tiles, warp-streamed
// Each WARP owns a contiguous run of merge-path tiles (tile length L = 256*R - 8) and streams
// them as rounds of 256 nonzeros (8 contiguous per lane, 256-bit loads).  A 3-deep register
// pipeline keeps round r+2 loading and round r+1's x gathers in flight while round r is
// reduced; the partial sum of the open row flows from round to round (and tile to tile) in a
// warp-uniform register, so there is no CTA barrier in the main loop and one warp segmented scan
// per 256 nonzeros.  The row pass of tile t+1 runs at the end of tile t from prefetched offsets
// and marks each row's last nonzero in a per-warp shared buffer.
// Measured choices: the first-row store and the tail clear are predicated, not
// branched (C3 291.5 -> 294.5 GNZ/s); __syncwarp only after a tile's row pass, not after every round
// (lanes touch only their own tail[] entries inside a tile; C3 286.7 -> 291.4 GNZ/s).

template <int R>
struct StreamCfg {
  static constexpr int kCap = 256 * R;  // local nonzero positions per tile
  static constexpr int L = kCap - 8;    // merge items per tile
  static constexpr int K = 2;           // rows per lane whose offsets are prefetched (64 rows / tile)
};

struct StreamRound {  // one round's data for one lane
  int col[8];
  float val[8];
};

__device__ __forceinline__ void stream_load(const TileArgs& a, int4 c, int k, int lane, StreamRound& d,
                                            uint64_t spol) {
  const int g = (c.y & ~7) + 256 * k + 8 * lane;
  if (g < c.w && g + 8 <= a.nnz) {
    ld_stream_v8(a.col + g, d.col, spol);
    ld_stream_v8(a.val + g, d.val, spol);
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const bool ok = g + e < c.w;
      d.col[e] = ok ? ld_cs(a.col + g + e) : 0;
      d.val[e] = ok ? ld_cs(a.val + g + e) : 0.f;
    }
  }
}

// One x value.  TIER 0: x[c].  With an x-reuse plan the column stream holds ~slot (< 0) for hot
// columns, whose x values sit in shared memory at byte address sxb + 4*slot (TIER >= 1), and
// cols + w for warm columns, read from the dense copy x_warm[w] with an L2 evict_last policy while
// the remaining (cold) columns are read from x with evict_first (TIER 2).  Predicated loads, no
// branch.
template <int TIER>
__device__ __forceinline__ float gx(const float* __restrict__ x, const float* __restrict__ xw, int cols, uint32_t sxb,
                                    int c, uint64_t xpol, uint64_t cpol) {
  float v;
  if (TIER == 2) {
    asm("{\n\t.reg .pred p, q, r;\n\tsetp.lt.s32 p, %1, 0;\n\tsetp.ge.s32 q, %1, %4;\n\tor.pred r, p, q;\n\t"
        "@p ld.shared.f32 %0, [%2];\n\t"
        "@q ld.global.nc.L2::cache_hint.f32 %0, [%3], %6;\n\t"
        "@!r ld.global.nc.L2::cache_hint.f32 %0, [%5], %7;\n\t}"
        : "=f"(v)
        : "r"(c), "r"(sxb + ((unsigned)~c << 2)), "l"(xw + (c - cols)), "r"(cols), "l"(x + c), "l"(xpol), "l"(cpol));
    return v;
  }
  if (TIER == 1) {
    asm("{\n\t.reg .pred p;\n\tsetp.lt.s32 p, %1, 0;\n\t@p ld.shared.f32 %0, [%2];\n\t"
        "@!p ld.global.nc.f32 %0, [%3];\n\t}"
        : "=f"(v)
        : "r"(c), "r"(sxb + ((unsigned)~c << 2)), "l"(x + c));
    return v;
  }
  return ld_x(x + c);
}

// the 8 gathers of a lane's round (every loaded column index is valid; positions outside the tile
// are masked later by zeroing their values)
template <int TIER>
__device__ __forceinline__ void gx8(const float* __restrict__ x, const float* __restrict__ xw, int cols, uint32_t sxb,
                                    const StreamRound& d, float (&xv)[8], uint64_t xpol, uint64_t cpol) {
#pragma unroll
  for (int e = 0; e < 8; ++e) xv[e] = gx<TIER>(x, xw, cols, sxb, d.col[e], xpol, cpol);
}

// y store predicated on `p` (no branch)
__device__ __forceinline__ void st_cs_if(float* ptr, float v, bool p) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.global.cs.f32 [%0], %1;\n\t}"
               :: "l"(ptr), "f"(v), "r"((unsigned)p) : "memory");
}


// y stores of the warp-streamed kernel.  With PEERS (the fix-up of the fused multi-GPU epilogue,
// DESIGN.md 7b) the value also goes to every other rank's copy of y over NVLink; `peers` = false for a
// partial value, which stays local.
template <bool PEERS>
__device__ __forceinline__ void put_y(const TileArgs& a, int idx, float v, bool peers = true) {
  __stcs(a.y + idx, v);
  if (PEERS && peers) {
#pragma unroll
    for (int p = 0; p < kMaxPeers; ++p)
      if (p < a.npeers) __stcg(a.peer_y[p] + idx, v);
  }
}

// Row pass of tile c into tail[]: tail[q] = r + 1 when local nonzero q ends row r (r >= 0);
// rows r > 0 with no nonzero in the tile get y = 0; returns (warp-uniform) whether row 0 has no
// nonzero in the tile (its value is then the carry entering the tile).
template <int R, int K, typename TailT>
__device__ __forceinline__ bool stream_row_pass(const TileArgs& a, int4 c, int lane, const int (&lo_)[K],
                                                const int (&hi_)[K], TailT* tail) {
  const int i0 = c.x, nrows = c.z - c.x, jA = c.y & ~7, lo = c.y - jA;
  bool row0_empty = false;
  if (LB_ABL & 4) return false;
  for (int j = 0; 32 * j < nrows; ++j) {
    const int r = lane + 32 * j;
    if (r < nrows) {
      int ob, oe;
      if (j < K) {
#pragma unroll
        for (int q = 0; q < K; ++q)
          if (q == j) { ob = lo_[q]; oe = hi_[q]; }
      } else {
        ob = __ldcs(a.off + i0 + r);
        oe = __ldcs(a.off + i0 + r + 1);
      }
      const int e = oe - jA;
      const int s = r == 0 ? lo : ob - jA;
      if (e > s) tail[e - 1] = (TailT)(r + 1);
      else if (r > 0) put_y<false>(a, i0 + r, 0.f);
      else row0_empty = true;
    }
  }
  return __shfl_sync(kFull, (int)row0_empty, 0) != 0;
}

// 8 row ids of a lane's round from the warp's tail buffer (16- or 32-bit entries)
__device__ __forceinline__ void tail_read8(const unsigned short* p, unsigned (&rid)[8]) {
  const uint4 q = *reinterpret_cast<const uint4*>(p);
  const unsigned w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int e = 0; e < 8; ++e) rid[e] = (e & 1) ? (w[e >> 1] >> 16) : (w[e >> 1] & 0xFFFFu);
}
__device__ __forceinline__ void tail_read8(const unsigned* p, unsigned (&rid)[8]) {
  const uint4 q0 = *reinterpret_cast<const uint4*>(p), q1 = *reinterpret_cast<const uint4*>(p + 4);
  rid[0] = q0.x; rid[1] = q0.y; rid[2] = q0.z; rid[3] = q0.w;
  rid[4] = q1.x; rid[5] = q1.y; rid[6] = q1.z; rid[7] = q1.w;
}

// Fused multi-GPU epilogue (PEERS): when a tile is done, its final rows [i0, i1) -- every row that ends
// in the tile, written to the local y by this warp (the row pass, the rounds) -- are copied to every
// other rank's y with coalesced stores over NVLink.  The warp's first row is excluded when it started
// before the warp's run (`open_row`, partial: the fix-up completes it and sends it).  One coalesced
// pass per tile instead of a peer store per row end keeps the epilogue off the rounds' critical path
// (measured: a software-pipelined variant of this copy was no faster).
__device__ __forceinline__ void stream_peer_copy(const TileArgs& a, int4 c, int open_row, int lane) {
  const int r0 = c.x == open_row ? c.x + 1 : c.x;
  for (int r = r0 + lane; r < c.z; r += 32) {
    const float v = __ldcg(a.y + r);  // this warp's own stores, ordered by the __syncwarp before the call
#pragma unroll
    for (int p = 0; p < kMaxPeers; ++p)
      if (p < a.npeers) __stcg(a.peer_y[p] + r, v);
  }
}

// Reduce one round (256 nonzeros) of tile c: products val*x summed per lane, rows that end after
// the lane's first row end are stored directly, the ballot-based segmented scan gives each lane's
// first row its carry-in, and `rc` (warp-uniform) carries the open row's partial to the next round.
template <typename TailT>
__device__ __forceinline__ void stream_reduce_round(const TileArgs& a, int4 cT, int k, int lane, bool r0e,
                                                    float (&val)[8], const float (&xc)[8], TailT* tail, float& rc,
                                                    float& rcc) {
  // (b) the row open at the tile start has no nonzero here: it ends now with the carry
  const int i0 = cT.x;
  if (k == 0 && r0e) {
    if (lane == 0) put_y<false>(a, i0, rc + rcc);
    rc = 0.f;
    rcc = 0.f;
  }
  // (c) positions outside the tile's nonzero range [lo, hi) add exactly zero (warp-uniform test)
  {
    const int lo = cT.y & 7, hi = cT.w - (cT.y & ~7);
    if ((k == 0 && lo) || 256 * k + 256 > hi) {
      const int q0 = 256 * k + 8 * lane;
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (q0 + e < lo || q0 + e >= hi) val[e] = 0.f;
    }
  }
  // (d) reduce this round: rows that end inside the lane's 8 nonzeros after its first row end
  // are complete; the first one waits for the carry-in from the lanes before
  unsigned rids[8];
  if (LB_ABL & 4) {
#pragma unroll
    for (int e = 0; e < 8; ++e) rids[e] = (lane == 31 && e == 7) ? 1u : 0u;
  } else {
    tail_read8(&tail[256 * k + 8 * lane], rids);
  }
  float* yt = a.y + i0 - 1;  // row r of the tile ends where rid = r + 1
  unsigned any = 0u, first_rid = 0u;
  float run = 0.f, first_val = 0.f;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    run = fmaf(val[e], xc[e], run);
    const unsigned rid = rids[e];
    any |= rid;
    if (!(LB_ABL & 1)) st_cs_if(yt + rid, run, rid != 0u && first_rid != 0u);
    const bool take = rid != 0u && first_rid == 0u;
    first_val = take ? run : first_val;
    first_rid = take ? rid : first_rid;
    run = rid != 0u ? 0.f : run;
  }
  // segmented inclusive scan over the lanes (Kogge-Stone; a lane with a row end starts a new
  // segment): lane l adds the partial of lane l-o unless a lane in (l-o, l] has a row end
  const unsigned B = __ballot_sync(kFull, first_rid != 0u);
  float v = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    if (LB_ABL & 2) break;
    const float vo = __shfl_up_sync(kFull, v, o);
    const bool reset = lane >= o ? ((B >> (lane - o + 1)) & ((1u << o) - 1u)) != 0u : true;
    if (!reset) v = vo + v;
  }
  const float lval = __shfl_up_sync(kFull, v, 1);
  const float agg_v = __shfl_sync(kFull, v, 31);
  {  // branch-free: predicated store of the first row end, predicated clear of the lane's tail entries
    const bool lf = (B & ((1u << lane) - 1u)) != 0u;  // a row ended in an earlier lane
    const float rcs = rc + rcc;
    const float carry_in = lane == 0 ? rcs : (lf ? lval : rcs + lval);
    if (!(LB_ABL & 1) || (LB_ABL & 4)) st_cs_if(a.y + (i0 - 1) + (int)first_rid, carry_in + first_val, first_rid != 0u);
    if (!(LB_ABL & 4)) {
      const unsigned ta = (unsigned)__cvta_generic_to_shared(&tail[256 * k + 8 * lane]);
      asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t@q st.shared.v4.u32 [%0], {0, 0, 0, 0};\n\t}"
                   :: "r"(ta), "r"(any) : "memory");
      if (sizeof(TailT) == 4)  // 32-bit row ids: 8 entries are 32 bytes
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t@q st.shared.v4.u32 [%0], {0, 0, 0, 0};\n\t}"
                     :: "r"(ta + 16u), "r"(any) : "memory");
    }
  }
  // the open row's partial: restarts at a row end in this round, else accumulates -- compensated
  // (rc + rcc), so a row spanning thousands of rounds keeps ~2u relative error;
  // branch-free and warp-uniform
  rc = B ? 0.f : rc;
  rcc = B ? 0.f : rcc;
  csum_add(rc, rcc, agg_v);
}

// One carry per warp (rows == a.rows for warps without tiles: skipped by the fix-up), then the
// last CTA to finish applies all carries in warp order (Alg.3 fix-up P:332-337, deterministic,
// compensated).
template <bool PEERS>
__device__ __forceinline__ void stream_carries_fixup(const TileArgs& a, int gw, int lane, int W, int i_last, float rc,
                                                     int& s_last) {
  if (lane == 0) {
    a.carry_row[gw] = i_last;
    a.carry_val[gw] = rc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // the CTA's peer stores (ordered before this thread by the barrier) are performed system-wide
    // before the kernel ends (fence cumulativity); then the carries are released at GPU scope
    if (PEERS) __threadfence_system();
    __threadfence();
    const unsigned done = atomicAdd(a.ticket, 1u);
    s_last = done == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    fixup_carries_blocked(a, (int)gridDim.x * W, threadIdx.x, W * 32,
                          [&](int r, float v) { put_y<PEERS>(a, r, v); });
    if (threadIdx.x == 0) *a.ticket = 0u;
    if (PEERS) __threadfence_system();
  }
}

// TailT: unsigned short for merge-path tiles (<= L rows), unsigned for nonzero-split tiles (any
// number of rows per tile).
// TIER >= 1: the column stream is an x-reuse plan's remapped copy (lb_csr_plan_hot_x); the CTA
// stages the x values of the hot columns (a.x_hot, a.hot_n4 float4s) in dynamic shared memory and
// serves those gathers from it -- one CTA per SM so the staged copy is shared by all of its warps.
// TIER 2 adds the warm columns, read from the dense L2-resident copy a.x_warm.
template <int W, int R, int MINB, typename TailT = unsigned short, int TIER = 0, bool PEERS = false>
__global__ void __launch_bounds__(W * 32, MINB) merge_stream_kernel(TileArgs a) {
  constexpr bool HOT = TIER >= 1;
  using Cfg = StreamCfg<R>;
  constexpr int K = Cfg::K;
  __shared__ __align__(16) TailT s_tail[W][Cfg::kCap];
  __shared__ int s_last;
  extern __shared__ __align__(16) float s_xhot[];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = blockIdx.x * W + warp;  // global warp id: owns tiles [t_begin, t_end)
  const int t_begin = min(a.num_tiles, gw * a.tiles_per_cta);
  const int t_end = min(a.num_tiles, t_begin + a.tiles_per_cta);
  const uint64_t spol = policy_evict_first();
  const uint64_t xpol = TIER == 2 ? policy_evict_last() : 0ull;
  TailT* tail = s_tail[warp];
  for (int w = lane; w < Cfg::kCap * (int)sizeof(TailT) / 16; w += 32)
    reinterpret_cast<uint4*>(tail)[w] = make_uint4(0u, 0u, 0u, 0u);
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: coords (and x_hot) are read below
  if (HOT) {
    for (int i = threadIdx.x; i < a.hot_n4; i += W * 32)
      reinterpret_cast<float4*>(s_xhot)[i] = __ldcg(reinterpret_cast<const float4*>(a.x_hot) + i);
    __syncthreads();
  }
  __syncwarp();

  // partial sum of the row open at the current stream position, compensated (warp-uniform)
  float rc = 0.f, rcc = 0.f;
  int i_last = t_begin < t_end ? __ldg(&a.coords[t_end].x) : a.rows;
  if (t_begin < t_end) {
    const float* __restrict__ xg = a.x;
    const float* __restrict__ xw = a.x_warm;
    const uint32_t sxb = HOT ? (uint32_t)__cvta_generic_to_shared(s_xhot) : 0u;
    const int nsteps = (t_end - t_begin) * R;
    // coordinates of tiles t, t+1, t+2 (int4 = i0, j0, i1, j1)
    int4 cT = tile_coords(a, t_begin);
    int4 cT1 = t_begin + 1 < t_end ? tile_coords(a, t_begin + 1) : cT;
    int4 cT2 = t_begin + 2 < t_end ? tile_coords(a, t_begin + 2) : cT1;
    int olo[K], ohi[K];
    stream_prefetch_offsets<R, K>(a, cT, lane, olo, ohi);
    // PEERS: the warp's first row is partial when it started before the warp's first tile (the
    // fix-up completes it and sends it to the peers); every other row this warp writes is final
    const int open_row = PEERS && cT.x < a.rows && cT.y > __ldg(a.off + cT.x) ? cT.x : -1;
    bool r0e = stream_row_pass<R, K, TailT>(a, cT, lane, olo, ohi, tail);
    if (t_begin + 1 < t_end) stream_prefetch_offsets<R, K>(a, cT1, lane, olo, ohi);
    __syncwarp();
    // three rounds in flight: reduced (gathered), gathering, loading -- rotated by unrolling the
    // loop three times, so no register is copied between rounds
    StreamRound D0, D1, D2;
    float X0[8], X1[8], X2[8];
    stream_load(a, cT, 0, lane, D0, spol);
    if (1 < nsteps) stream_load(a, R > 1 ? cT : cT1, R > 1 ? 1 : 0, lane, D1, spol);
    gx8<TIER>(xg, xw, a.cols, sxb, D0, X0, xpol, spol);

    int t = t_begin, k = 0, st = 0;
    auto step = [&](StreamRound& dc, float (&xc)[8], StreamRound& dn, float (&xn)[8], StreamRound& dl) {
      // (a) gathers for round st+1, loads for round st+2
      if (st + 1 < nsteps) gx8<TIER>(xg, xw, a.cols, sxb, dn, xn, xpol, spol);
      if (st + 2 < nsteps) {
        const int k2 = k + 2;
        const bool same = k2 < R;
        stream_load(a, same ? cT : cT1, same ? k2 : k2 - R, lane, dl, spol);
      }
      stream_reduce_round(a, cT, k, lane, r0e, dc.val, xc, tail, rc, rcc);
      // (e) tile t done: (PEERS) its final rows go to the other ranks, row pass of tile t+1 (offsets
      // prefetched), advance coords
      if (++k == R) {
        k = 0;
        ++t;
        __syncwarp();
        if (PEERS) stream_peer_copy(a, cT, open_row, lane);
        if (t < t_end) {
          r0e = stream_row_pass<R, K, TailT>(a, cT1, lane, olo, ohi, tail);
          if (t + 1 < t_end) stream_prefetch_offsets<R, K>(a, cT2, lane, olo, ohi);
          cT = cT1;
          cT1 = cT2;
          if (t + 2 < t_end) cT2 = tile_coords(a, t + 2);
        }
        __syncwarp();  // the row pass's tail[] writes before the next round's reads
      }
    };
    while (true) {
      step(D0, X0, D1, X1, D2);
      if (++st == nsteps) break;
      step(D1, X1, D2, X2, D0);
      if (++st == nsteps) break;
      step(D2, X2, D0, X0, D1);
      if (++st == nsteps) break;
    }
  }

  stream_carries_fixup<PEERS>(a, gw, lane, W, i_last, rc + rcc, s_last);
}

// ----------------------------------------------------------------------------- ceiling probe
// Diagnostic: stream col/val with the tile kernels' 256-bit loads and gather x[col] with no row
// structure (no scans, no y) -- the stream+gather ceiling of this matrix on this GPU, against which
// bench.py reports the tile processor.  `flag` is 0 at run time (keeps the sum live).
// TIER >= 1: the column stream is an x-reuse plan's (hot slots ~s, warm cols + w) and the CTA stages
// x_hot in dynamic shared memory exactly as merge_stream_kernel does -- the ceiling of the plan.
template <int TIER>
__global__ void __launch_bounds__(512) probe_stream_gather_kernel(int nnz, const int* __restrict__ col,
                                                                  const float* __restrict__ val,
                                                                  const float* __restrict__ x,
                                                                  const float* __restrict__ x_hot, int hot_n4,
                                                                  const float* __restrict__ x_warm, int cols,
                                                                  int flag, float* sink) {
  extern __shared__ __align__(16) float s_xhot[];
  const uint64_t pol = policy_evict_first();
  const uint64_t xpol = TIER == 2 ? policy_evict_last() : 0ull;
  if (TIER >= 1) {
    for (int i = threadIdx.x; i < hot_n4; i += blockDim.x)
      reinterpret_cast<float4*>(s_xhot)[i] = __ldcg(reinterpret_cast<const float4*>(x_hot) + i);
    __syncthreads();
  }
  const uint32_t sxb = TIER >= 1 ? (uint32_t)__cvta_generic_to_shared(s_xhot) : 0u;
  float s = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 8;
  int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
  for (; i + 8 <= nnz; i += stride) {
    StreamRound d;
    float xv[8];
    ld_stream_v8(col + i, d.col, pol);
    ld_stream_v8(val + i, d.val, pol);
    gx8<TIER>(x, x_warm, cols, sxb, d, xv, xpol, pol);
#pragma unroll
    for (int e = 0; e < 8; ++e) s = fmaf(d.val[e], xv[e], s);
  }
  for (; i < nnz; ++i) s = fmaf(val[i], gx<TIER>(x, x_warm, cols, sxb, col[i], xpol, pol), s);
  if (flag) sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Diagnostic: the stream+gather probe with the hot tier spread over a thread-block
// cluster of C CTAs (C SMs): slot s lives in the shared memory of cluster rank s % C at index s / C, and
// a gather of a hot column reads it through distributed shared memory (mapa + ld.shared::cluster), so
// the cluster holds C times the hot columns one SM can.  Measures whether remote shared-memory reads
// relieve the L1->L2 request path that the cold gathers saturate.
template <int C>
__global__ void __launch_bounds__(512) probe_cluster_gather_kernel(int nnz, const int* __restrict__ col,
                                                                   const float* __restrict__ val,
                                                                   const float* __restrict__ x,
                                                                   const float* __restrict__ x_hot, int hot_n,
                                                                   int flag, float* sink) {
  extern __shared__ __align__(16) float s_xhot[];
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int per = (hot_n + C - 1) / C;
  for (int i = threadIdx.x; i < per; i += blockDim.x) {
    const int sl = i * C + (int)rank;
    s_xhot[i] = sl < hot_n ? __ldcg(x_hot + sl) : 0.f;
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  const uint64_t pol = policy_evict_first();
  const uint32_t sxb = (uint32_t)__cvta_generic_to_shared(s_xhot);
  constexpr int kLog = C == 1 ? 0 : C == 2 ? 1 : C == 4 ? 2 : 3;
  float s = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 8;
  int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
  for (; i + 8 <= nnz; i += stride) {
    int c[8];
    float v[8], xv[8];
    ld_stream_v8(col + i, c, pol);
    ld_stream_v8(val + i, v, pol);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const unsigned sl = (unsigned)~c[e];
      asm("{\n\t.reg .pred p;\n\t.reg .u32 ra;\n\tsetp.lt.s32 p, %1, 0;\n\t"
          "@p mapa.shared::cluster.u32 ra, %2, %3;\n\t"
          "@p ld.shared::cluster.f32 %0, [ra];\n\t"
          "@!p ld.global.nc.f32 %0, [%4];\n\t}"
          : "=f"(xv[e])
          : "r"(c[e]), "r"(sxb + ((sl >> kLog) << 2)), "r"(sl & (C - 1)), "l"(x + c[e]));
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) s = fmaf(v[e], xv[e], s);
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (flag) sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Diagnostic: the read-only stream ceiling -- col_idx and values streamed with the same 256-bit
// evict-first loads and no x gathers (8 B per nonzero).  bench.py reports the tile kernel's
// algorithmic bytes against this as well as against the copy peak.
__global__ void __launch_bounds__(512) probe_stream_kernel(int nnz, const int* __restrict__ col,
                                                           const float* __restrict__ val, int flag, float* sink) {
  const uint64_t pol = policy_evict_first();
  float s = 0.f;
  int acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 8;
  int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
  for (; i + 8 <= nnz; i += stride) {
    int c[8];
    float v[8];
    ld_stream_v8(col + i, c, pol);
    ld_stream_v8(val + i, v, pol);
#pragma unroll
    for (int e = 0; e < 8; ++e) { s += v[e]; acc ^= c[e]; }
  }
  for (; i < nnz; ++i) { s += val[i]; acc ^= col[i]; }
  if (flag) sink[blockIdx.x * blockDim.x + threadIdx.x] = s + (float)acc;
}

}  // namespace lbk
