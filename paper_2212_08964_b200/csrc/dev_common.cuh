// dev_common.cuh -- device helpers shared by every kernel header of liblb (arXiv 2212.08964, Ch.3-4).
// Citations "P:L" = PAPER.md line L.
//
// The path is bandwidth/gather bound (2 flops per >= 8 bytes); no tensor cores.
//  * x[col] gathers use plain LDG (L1-allocating): on B200 random 4-byte gathers are bound by
//    ~1 L1TEX wavefront per clock per SM (profiles/r01_microbench_l2_capacity.txt); TMA gather4 /
//    bulk copies measured ~60 G/s, so they are not used for x.
//  * col_idx / values are streamed with 256-bit loads that do not allocate in L1 and are evicted
//    first from L2 (`ld_stream_v8`).
//  * Every sum that can run over an unbounded number of partials (the open row carried across
//    rounds and tiles, the fix-up over carries, long rows in the row-granular schedules) is
//    compensated (2Sum, `csum_add`): fp32 sequential sums of same-sign terms break the 1e-5
//    relative tolerance after ~1e3 terms, compensated ones stay at ~2u.
#pragma once
#include <cstdint>
#include <climits>
#include <cuda_runtime.h>

namespace lbk {

constexpr unsigned kFull = 0xffffffffu;

// Diagnostic ablations of merge_stream_kernel (tools/ablate.sh builds separate libraries with
// -DLB_ABL=mask; results are WRONG by construction, timings only).  0 in every product build.
//   1: no y stores in the main loop   2: no segmented scan   4: no row pass / tail reads
#ifndef LB_ABL
#define LB_ABL 0
#endif

// ----------------------------------------------------------------------------- loads
__device__ __forceinline__ int4 ld_cs_v4(const int* p) { return __ldcs(reinterpret_cast<const int4*>(p)); }
__device__ __forceinline__ float4 ld_cs_v4(const float* p) { return __ldcs(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ int ld_cs(const int* p) { return __ldcs(p); }
__device__ __forceinline__ float ld_cs(const float* p) { return __ldcs(p); }
__device__ __forceinline__ float ld_x(const float* p) { return __ldg(p); }

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// 8 consecutive 32-bit elements with one 256-bit load (sm_100a LDG.E.256; 32-byte aligned p),
// L1 no-allocate, L2 policy `pol` (evict-first for the col/val stream)
__device__ __forceinline__ void ld_stream_v8(const int* p, int (&r)[8], uint64_t pol) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "l"(p), "l"(pol));
}
__device__ __forceinline__ void ld_stream_v8(const float* p, float (&r)[8], uint64_t pol) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
               : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
               : "l"(p), "l"(pol));
}

// ----------------------------------------------------------------------------- compensated sums
// 2Sum (Knuth): t = fl(s + v) and the exact rounding error e = (s + v) - t; the error is kept in c,
// so the value of the pair is s + c.  Branch-free, six flops, exact for any s, v (no overflow).
// Explicit _rn intrinsics: nothing may contract or reassociate these.
__device__ __forceinline__ void csum_add(float& s, float& c, float v) {
  const float t = __fadd_rn(s, v);
  const float bp = __fsub_rn(t, s);
  const float e = __fadd_rn(__fsub_rn(s, __fsub_rn(t, bp)), __fsub_rn(v, bp));
  s = t;
  c = __fadd_rn(c, e);
}

// ----------------------------------------------------------------------------- warp scans
// Segmented inclusive scan across a warp.  Pairs (f, v); combine(left, right) =
// (left.f | right.f, right.f ? right.v : left.v + right.v).  With f = "a segment ended at or
// after this element" it propagates the partial sum of the open segment; with f = "segment
// head" it is a classic head-flag segmented scan.  Kogge-Stone: every result is a tree sum.
__device__ __forceinline__ void warp_segscan_incl(bool& f, float& v, unsigned lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    float vo = __shfl_up_sync(kFull, v, o);
    int fo = __shfl_up_sync(kFull, (int)f, o);
    if (lane >= (unsigned)o) {
      if (!f) v = vo + v;
      f = f || fo;
    }
  }
}

// The same over the first N lanes only (N a power of two <= 32).
template <int N>
__device__ __forceinline__ void warp_segscan_incl_n(bool& f, float& v, unsigned lane) {
#pragma unroll
  for (int o = 1; o < N; o <<= 1) {
    float vo = __shfl_up_sync(kFull, v, o);
    int fo = __shfl_up_sync(kFull, (int)f, o);
    if (lane >= (unsigned)o) {
      if (!f) v = vo + v;
      f = f || fo;
    }
  }
}

__device__ __forceinline__ int warp_incl_scan_int(int v, unsigned lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(kFull, v, o);
    if (lane >= (unsigned)o) v += t;
  }
  return v;
}

__device__ __forceinline__ int4 block_excl_scan3(int4 v, int4* total) {
  __shared__ int4 ws[32];
  __shared__ int4 wtot;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int a = v.x, b = v.y, c = v.z;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int ta = __shfl_up_sync(kFull, a, o), tb = __shfl_up_sync(kFull, b, o), tc = __shfl_up_sync(kFull, c, o);
    if (lane >= o) { a += ta; b += tb; c += tc; }
  }
  if (lane == 31) ws[warp] = make_int4(a, b, c, 0);
  __syncthreads();
  if (warp == 0) {
    const int4 w = lane < nw ? ws[lane] : make_int4(0, 0, 0, 0);
    int wa = w.x, wb = w.y, wc = w.z;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int ta = __shfl_up_sync(kFull, wa, o), tb = __shfl_up_sync(kFull, wb, o), tc = __shfl_up_sync(kFull, wc, o);
      if (lane >= o) { wa += ta; wb += tb; wc += tc; }
    }
    if (lane < nw) ws[lane] = make_int4(wa - w.x, wb - w.y, wc - w.z, 0);  // exclusive warp offsets
    if (lane == nw - 1) wtot = make_int4(wa, wb, wc, 0);
  }
  __syncthreads();
  const int4 base = ws[warp];
  if (total) *total = wtot;
  const int4 r = make_int4(base.x + a - v.x, base.y + b - v.y, base.z + c - v.z, 0);
  __syncthreads();
  return r;
}

// Fixed xor-shuffle tree over the 32 lanes (deterministic; every lane gets the total).
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// ----------------------------------------------------------------------------- tile-kernel arguments
constexpr int kMaxPeers = 7;  // other GPUs of one 8-GPU node

struct TileArgs {
  const int* off;
  const int* col;
  const float* val;
  const float* x;
  float* y;
  const int2* coords;  // [T+1] merge-path (or nonzero-split) coordinates (row, nz)
  int rows, nnz;
  int num_tiles;
  int tiles_per_cta;   // tiles per CTA (CTA-tile kernels) or per warp (warp-streamed kernels)
  int* carry_row;
  float* carry_val;
  unsigned* ticket;    // zero before launch; the last CTA resets it
  const float* x_hot;  // x-reuse plan: x of the planned hot columns, gathered this call
  int hot_n4;          // number of float4s of x_hot staged in shared memory (0: no plan)
  const float* x_warm; // x-reuse plan: x of the warm columns (column stream value cols + w)
  int cols;
  float* peer_y[kMaxPeers];  // fused multi-GPU epilogue: the other ranks' y at this rank's rows
  int npeers;
  int off_keep;        // 1: row offsets small enough to keep in L2 across calls (evict_last loads)
};

// one row offset with an explicit L2 policy (evict_last keeps a small offsets array resident in L2
// across calls, so the next call's partition search hits L2; evict_first streams a large one)
__device__ __forceinline__ int ld_off(const int* p, uint64_t pol) {
  int v;
  asm("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}

// tile t's coordinates (i0, j0, i1, j1)
__device__ __forceinline__ int4 tile_coords(const TileArgs& a, int t) {
  const int2 c0 = a.coords[t], c1 = a.coords[t + 1];
  return make_int4(c0.x, c0.y, c1.x, c1.y);
}

// offsets of the first 32*K rows of tile c (row r = lane + 32 j), prefetched one tile ahead
template <int R, int K>
__device__ __forceinline__ void stream_prefetch_offsets(const TileArgs& a, int4 c, int lane, int (&lo_)[K],
                                                        int (&hi_)[K]) {
  const int nrows = c.z - c.x;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const int r = lane + 32 * j;
    if (r < nrows) {
      lo_[j] = __ldcs(a.off + c.x + r);
      hi_[j] = __ldcs(a.off + c.x + r + 1);
    }
  }
}

// The fix-up of the tile kernels (Alg.3, run by the last CTA to finish): y[r] += the
// carries of the runs that ended inside row r, in run order, compensated (carries are sorted by row;
// a giant row split over thousands of runs keeps ~2u relative error).  `nc` carries, thread `tid` of
// `nthreads`.  rows == a.rows marks the terminal corner (skipped, reading R5).
__device__ __forceinline__ void fixup_carries(const TileArgs& a, int nc, int tid, int nthreads) {
  for (int c = tid; c < nc; c += nthreads) {
    const int r = __ldcg(a.carry_row + c);
    if (r >= a.rows) continue;
    if (c > 0 && __ldcg(a.carry_row + c - 1) == r) continue;
    float s = __ldcg(a.y + r), cc = 0.f;
    for (int k = c; k < nc && __ldcg(a.carry_row + k) == r; ++k) csum_add(s, cc, __ldcg(a.carry_val + k));
    a.y[r] = s + cc;
  }
}

// The same fix-up with the carries split into contiguous blocks, one per thread, read 8 at a time:
// the run heads of a batch (carries whose row differs from the previous carry's) load their y and
// carry values together, so a fix-up over thousands of carries costs a few dependent L2 round trips
// per thread instead of several per carry.  Same order and arithmetic as fixup_carries (bitwise equal).
struct StoreY {
  const TileArgs& a;
  __device__ void operator()(int r, float v) const { a.y[r] = v; }
};
template <typename Store>
__device__ __forceinline__ void fixup_carries_blocked(const TileArgs& a, int nc, int tid, int nthreads, Store store) {
  const int per = (nc + nthreads - 1) / nthreads;
  const int c0 = tid * per, c1 = min(nc, c0 + per);
  for (int base = c0; base < c1; base += 8) {
    int rr[8];
    float vv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int c = base + u;
      rr[u] = c < c1 ? __ldcg(a.carry_row + c) : INT_MAX;
      vv[u] = c < c1 ? __ldcg(a.carry_val + c) : 0.f;
    }
    int prev = base > 0 ? __ldcg(a.carry_row + base - 1) : INT_MIN;
    float yy[8];
    bool head[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      head[u] = rr[u] < a.rows && rr[u] != prev;
      prev = rr[u];
      yy[u] = head[u] ? __ldcg(a.y + rr[u]) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (!head[u]) continue;
      float sum = yy[u], comp = 0.f;
      int k = u;
      for (; k < 8 && rr[k] == rr[u]; ++k) csum_add(sum, comp, vv[k]);
      if (k == 8 || base + k >= c1)  // the run may continue past this batch / block: finish it in order
        for (int c = base + k; c < nc && __ldcg(a.carry_row + c) == rr[u]; ++c)
          csum_add(sum, comp, __ldcg(a.carry_val + c));
      store(rr[u], sum + comp);
    }
  }
}
__device__ __forceinline__ void fixup_carries_blocked(const TileArgs& a, int nc, int tid, int nthreads) {
  fixup_carries_blocked(a, nc, tid, nthreads, StoreY{a});
}

}  // namespace lbk
