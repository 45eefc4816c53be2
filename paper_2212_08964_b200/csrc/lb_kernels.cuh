// lb_kernels.cuh -- sm_100a device code for CSR SpMV under three load-balancing schedules
// (arXiv 2212.08964, Ch.3-4).  Citations "P:L" = PAPER.md line L.
//
// The path is bandwidth/gather bound (2 flops per >= 8 bytes); no tensor cores.
// Design notes:
//  * Merge-path tiles (L merge items each) are computed by lb_partition (Alg.3 2DSearch).
//  * The tile processor is a persistent kernel: CTA c owns a contiguous run of tiles, so the
//    partial row that crosses a tile boundary is carried in registers from tile to tile and
//    only one carry per CTA reaches the fix-up ("first splitting the work across
//    blocks, and then to threads within a block").
//  * Inside a tile the nonzeros [j_t, j_{t+1}) are streamed with 128-bit loads aligned down to
//    a 16-byte boundary (reverse-offset alignment) and summed per row with a
//    warp-shuffle segmented scan; the rows [i_t, i_{t+1}) are written by a second, coalesced
//    pass.  Both passes are strided across the CTA, so every thread does an even share of the
//    tile's nonzeros and of its row ends.
//  * x[col] gathers use plain LDG (L1-allocating): on B200 random 4-byte gathers are bound by
//    ~1 L1tex line per clock per SM (~286 G/s measured, profiles/r01_microbench_gather.txt);
//    TMA gather4 / bulk copies measured ~60 G/s, so they are not used for x.
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
// x gather with an L2 evict_last policy (keeps x resident against the col/val stream)
__device__ __forceinline__ float ld_x_keep(const float* p, uint64_t pol) {
  float v;
  asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

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

__device__ __forceinline__ int warp_incl_scan_int(int v, unsigned lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(kFull, v, o);
    if (lane >= (unsigned)o) v += t;
  }
  return v;
}

// ----------------------------------------------------------------------------- validation
// flags[0]: off[0] != 0; flags[1]: first row r with off[r] > off[r+1] (INT_MAX if none);
// flags[2]: off[rows] != nnz; flags[3]: first k with col[k] outside [0, cols) (INT_MAX if none).
__global__ void validate_kernel(int rows, int cols, int nnz, const int* __restrict__ off,
                                const int* __restrict__ col, int* flags) {
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (tid == 0) {
    flags[0] = off[0] != 0;
    flags[2] = off[rows] != nnz;
  }
  for (int64_t r = tid; r < rows; r += stride)
    if (off[r] > off[r + 1]) atomicMin(&flags[1], (int)r);
  for (int64_t k = tid; k < nnz; k += stride) {
    int c = col[k];
    if (c < 0 || c >= cols) atomicMin(&flags[3], (int)k);
  }
}

// max row length (for LB_SCHED_AUTO): grid-stride max over off[r+1]-off[r], one atomicMax per warp
__global__ void max_row_kernel(int rows, const int* __restrict__ off, int* out) {
  int m = 0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
    m = max(m, __ldg(off + r + 1) - __ldg(off + r));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(kFull, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// ----------------------------------------------------------------------------- partition
// Alg.3 P:306-311 (2DSearch) for every tile boundary t = 0..T:
//   d = min(t*L, rows+nnz);  i = #{k < rows : k + off[k+1] < d};  j = d - i.
// k + off[k+1] is the merge position of row end k (row end before nonzero off[k+1], reading
// R1); it is strictly increasing in k, so i is a lower-bound binary search on
// [max(0, d-nnz), min(d, rows)] (below d-nnz every row end precedes d).
__device__ __forceinline__ int2 merge_path_search(int rows, int nnz, const int* __restrict__ off, int64_t t,
                                                  int64_t L) {
  const int64_t total = (int64_t)rows + nnz;
  const int64_t d = t * L < total ? t * L : total;
  int lo = (int)(d - nnz > 0 ? d - nnz : 0);
  int hi = (int)(d < rows ? d : rows);
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if ((int64_t)mid + __ldg(off + mid + 1) < d) lo = mid + 1;
    else hi = mid;
  }
  return make_int2(lo, (int)(d - lo));
}

__global__ void partition_kernel(int rows, int nnz, const int* __restrict__ off, int64_t L, int64_t T,
                                 int2* __restrict__ coords) {
  // PDL: let the dependent tile kernel start its prologue now (it waits for our completion)
  asm volatile("griddepcontrol.launch_dependents;");
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t > T) return;
  coords[t] = merge_path_search(rows, nnz, off, t, L);
}

// The same partition (threads 0..T; T = -1 skips it) fused with the per-call gathers of an x-reuse
// plan (lb_csr_plan_hot_x): x_hot[h] = x[hot_cols[h]] (staged in shared memory by the tile kernel)
// and x_warm[w] = x[warm_cols[w]] (a dense copy of the warm columns that stays in L2).
__global__ void partition_xhot_kernel(int rows, int nnz, const int* __restrict__ off, int64_t L, int64_t T,
                                      int2* __restrict__ coords, const int* __restrict__ hot_cols, int hot_n,
                                      const int* __restrict__ warm_cols, int warm_n, const float* __restrict__ x,
                                      float* __restrict__ x_hot, float* __restrict__ x_warm,
                                      const unsigned* __restrict__ wmask = nullptr,
                                      const int* __restrict__ wbase = nullptr, int64_t nquad = 0) {
  asm volatile("griddepcontrol.launch_dependents;");
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t <= T) {
    coords[t] = merge_path_search(rows, nnz, off, t, L);
    return;
  }
  const int64_t h = t - (T + 1);
  if (h < hot_n) {
    x_hot[h] = __ldg(x + __ldg(hot_cols + h));
    return;
  }
  const int64_t w = h - hot_n;  // warm columns ascend, so these reads sweep x in address order
  if (w < warm_n) {
    x_warm[w] = __ldg(x + __ldg(warm_cols + w));
    return;
  }
  // compact plan: x_warm = the referenced non-hot entries of x in column order, by stream compaction
  // with the plan's bit mask (wmask: bit c of the warm columns; wbase: warm index of the word's first
  // one).  Thread u covers columns 4u .. 4u+3 and reads only the ones it keeps (coalesced sweep).
  const int64_t u = w - warm_n;
  if (u < nquad) {
    const unsigned m = __ldg(wmask + (u >> 3));
    const int sh = (int)(u & 7) * 4;
    unsigned bits = (m >> sh) & 0xFu;
    if (!bits) return;
    int o = __ldg(wbase + (u >> 3)) + __popc(m & ((1u << sh) - 1u));
    const float* xq = x + 4 * u;
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (bits & (1u << e)) x_warm[o++] = __ldg(xq + e);
  }
}

// Chunk boundaries for lb_spmv_host_x(LB_SPMV_CHUNKED): for k = 1 .. K-1 the first tile t >= k*step
// (scanning at most `span` tiles) whose start coordinate is clean -- j == off[i], no row split -- else
// T.  out[k] = t, out[K + k] = coords[t].x (its first row).
__global__ void clean_tiles_kernel(const int2* __restrict__ coords, const int* __restrict__ off, int64_t T, int K,
                                   int span, int64_t step, int* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x + 1;
  if (k >= K) return;
  // the scan starts at k*step: the host picks step a few tiles short of a whole number of waves (one
  // tile per warp of a launch), so a chunk whose cut is found within that slack fills its waves exactly
  int64_t t = (int64_t)k * step, found = T;
  for (int n = 0; n < span && t < T; ++n, ++t) {
    const int2 c = coords[t];
    if (c.y == __ldg(off + c.x)) { found = t; break; }
  }
  out[k] = (int)found;
  out[K + k] = coords[found].x;
}

// compact plan: bit mask and per-word base index of the warm columns (ascending list)
__global__ void plan_mask_kernel(const int* __restrict__ warm_cols, int warm_n, unsigned* __restrict__ wmask,
                                 int* __restrict__ wbase) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < warm_n; w += stride) {
    const int c = __ldg(warm_cols + w);
    atomicOr(wmask + (c >> 5), 1u << (c & 31));
    if (w == 0 || (__ldg(warm_cols + w - 1) >> 5) != (c >> 5)) wbase[c >> 5] = (int)w;
  }
}

// Nonzero-splitting partition (table; reading R19): tiles of L nonzeros, T = max(1,
// ceil(nnz/L)); boundary t: j = min(t*L, nnz), i = #{r : off[r+1] <= j} (upper bound of j in
// off[1..rows]), with (0, 0) and (rows, nnz) at the ends.  Every such (i, j) is a merge-path point,
// so the merge-path tile processors run these tiles unchanged.
__global__ void partition_nz_kernel(int rows, int nnz, const int* __restrict__ off, int64_t L, int64_t T,
                                    int2* __restrict__ coords) {
  asm volatile("griddepcontrol.launch_dependents;");
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t > T) return;
  const int j = (int)(t * L < nnz ? t * L : nnz);
  int i;
  if (t == 0) i = 0;
  else if (t == T) i = rows;
  else {
    int lo = 0, hi = rows;  // first r in [0, rows] with off[r+1] > j (r = rows if none)
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(off + mid + 1) <= j) lo = mid + 1;
      else hi = mid;
    }
    i = lo;
  }
  coords[t] = make_int2(i, j);
}

// ----------------------------------------------------------------------------- merge-path tiles
struct MergeArgs {
  const int* off;
  const int* col;
  const float* val;
  const float* x;
  float* y;
  const int2* coords;   // [T+1] tile coordinates (row, nz)
  int rows, nnz;
  int num_tiles;
  int tiles_per_cta;
  int* carry_row;       // [gridDim.x] row still open at the end of the CTA's run of tiles
  float* carry_val;     // [gridDim.x] its partial sum over the CTA's tiles
};

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
__global__ void __launch_bounds__(NT, 3) merge_tile_kernel(MergeArgs a) {
  using Cfg = MergeCfg<NT, L, VEC>;
  constexpr int NV = Cfg::kNV;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  typename Cfg::Smem& sm = *reinterpret_cast<typename Cfg::Smem*>(smem_raw);

  const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t_begin = blockIdx.x * a.tiles_per_cta;
  const int t_end = min(a.num_tiles, t_begin + a.tiles_per_cta);

  for (int w = tid; w < 2 * Cfg::kTailWords; w += NT) (&sm.tail[0][0])[w] = 0u;
  __syncthreads();

  float cta_carry = 0.f;  // partial of the row open at the start of the current tile (this CTA's share)
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
      if (r == 0) yv += cta_carry;
      a.y[i0 + r] = yv;
    }
    // (7) carry the open row (i1) to the next tile of this CTA (Alg.3)
    cta_carry = nrows > 0 ? agg_val : cta_carry + agg_val;
    i_last = i1;
  }
  if (tid == 0 && t_begin < t_end) {
    a.carry_row[blockIdx.x] = i_last;
    a.carry_val[blockIdx.x] = cta_carry;
  }
}

// Fix-up (Alg.3): y[row] += carries of the CTAs whose runs ended inside `row`
// (rows == rows means the terminal corner: skipped, reading R5).  Carries are sorted by row;
// the first carry of each row sums its run in CTA order (deterministic).
__global__ void fixup_kernel(int rows, int n, const int* __restrict__ carry_row,
                             const float* __restrict__ carry_val, float* __restrict__ y) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int r = carry_row[c];
  if (r >= rows) return;
  if (c > 0 && carry_row[c - 1] == r) return;
  float s = 0.f;
  for (int k = c; k < n && carry_row[k] == r; ++k) s += carry_val[k];
  y[r] += s;
}

// ----------------------------------------------------------------------------- merge-path tiles, TMA pipeline
// sm_100a tile processor used when row_offsets / col_idx / values are 16-byte aligned:
//  * one elected thread streams each upcoming tile's col/val/offset ranges into an S-stage
//    shared-memory ring with cp.async.bulk (TMA bulk copies, L2 evict-first), completing on an
//    mbarrier per stage, so DRAM latency is off the critical path;
//  * the row pass writes, for every nonzero that ends a row, the row's local index
//    (tailrow[q] = r + 1) -- no atomics -- and writes y = 0 (+carry) for rows with no nonzero in
//    the tile;
//  * the nonzero pass reads col/val/tailrow with 128/64-bit shared loads, gathers x, runs the
//    warp segmented scan + chunk scan, and the thread owning a row's last nonzero stores y[row];
//  * two __syncthreads per tile; the fix-up (Alg.3) runs in the last CTA to finish
//    (atomic ticket), in CTA order (deterministic).
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
// Wait for the phase with parity `parity` to complete.  Watchdog: a stage must land within
// milliseconds; after ~2^32 cycles the kernel traps (an error, never a silent hang).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  const long long t0 = clock64();
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if (clock64() - t0 > (1ll << 32)) __trap();  // ~2 s at 2 GHz
  }
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// global -> shared bulk copy (16-byte aligned, size multiple of 16), completes on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}

constexpr int kMaxPeers = 7;  // other GPUs of one 8-GPU node

struct PipeArgs {
  const int* off;
  const int* col;
  const float* val;
  const float* x;
  float* y;
  const int2* coords;
  int rows, nnz;
  int num_tiles;
  int tiles_per_cta;
  int* carry_row;
  float* carry_val;
  unsigned* ticket;  // zero before launch; the last CTA resets it
  const float* x_hot;  // x-reuse plan: x of the planned hot columns, gathered this call
  int hot_n4;          // number of float4s of x_hot staged in shared memory (0: no plan)
  const float* x_warm; // x-reuse plan: x of the warm columns (column stream value cols + w)
  int cols;
  float* peer_y[kMaxPeers];  // fused multi-GPU epilogue: the other ranks' y at this rank's rows
  int npeers;
};

// Tile length for E nonzeros per thread: the 16-byte-aligned nonzero range of a tile spans at
// most L + 6 elements, so L = NT*E - 8 fills every thread (tile quantisation).
template <int NT, int E>
constexpr int pipe_tile_len() { return NT * E - 8; }

template <int NT, int E, int S>
struct PipeCfg {
  static constexpr int L = pipe_tile_len<NT, E>();
  static constexpr int kCap = NT * E;                // staged elements per array per stage (>= L + 8)
  static constexpr int kWarps = NT / 32;
  static_assert(E % 4 == 0 && E >= 4 && E <= 16, "E: multiple of 4 in [4, 16]");
  static_assert(kWarps <= 32, "chunk scan uses one warp");
  struct Smem {
    int col[S][kCap];
    float val[S][kCap];
    int off[S][kCap];
    unsigned short tailrow[2][kCap];  // local row index + 1 of the row ending at nonzero q (0: none)
    uint64_t bar[S];
    int cflag[kWarps];
    float cval[kWarps];
    int last;
  };
};

template <int NT, int E, int S>
__device__ __forceinline__ void pipe_issue(const PipeArgs& a, typename PipeCfg<NT, E, S>::Smem& sm, int t, int stage,
                                           uint64_t pol) {
  // called by one thread: stage tile t's offsets [i0&~3, i1], col/val [j0&~3, j1)
  const int2 c0 = a.coords[t], c1 = a.coords[t + 1];
  const int oA = c0.x & ~3, oEnd = c1.x + 1;           // need off[i0 .. i1]
  const int jA = c0.y & ~3, jEnd = c1.y;
  const int oLim = (a.rows + 1) & ~3, jLim = a.nnz & ~3; // bulk copies stay inside the arrays
  const int oB = max(oA, min((oEnd + 3) & ~3, oLim));
  const int jB = max(jA, min((jEnd + 3) & ~3, jLim));
  const uint32_t ob = 4u * (oB - oA), jb = 4u * (jB - jA);
  mbar_arrive_expect_tx(&sm.bar[stage], ob + 2 * jb);
  if (ob) bulk_g2s(&sm.off[stage][0], a.off + oA, ob, &sm.bar[stage], pol);
  if (jb) {
    bulk_g2s(&sm.col[stage][0], a.col + jA, jb, &sm.bar[stage], pol);
    bulk_g2s(&sm.val[stage][0], a.val + jA, jb, &sm.bar[stage], pol);
  }
  // array-end remainders (< 4 elements): generic stores, published by a later __syncthreads
  for (int k = oB; k < oEnd; ++k) sm.off[stage][k - oA] = __ldg(a.off + k);
  for (int k = jB; k < jEnd; ++k) {
    sm.col[stage][k - jA] = __ldg(a.col + k);
    sm.val[stage][k - jA] = __ldg(a.val + k);
  }
}

template <int NT, int E, int S, int MINB>
__global__ void __launch_bounds__(NT, MINB) merge_pipe_kernel(PipeArgs a) {
  using Cfg = PipeCfg<NT, E, S>;
  constexpr int kW = Cfg::kWarps;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  typename Cfg::Smem& sm = *reinterpret_cast<typename Cfg::Smem*>(smem_raw);

  const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t_begin = blockIdx.x * a.tiles_per_cta;
  const int t_end = min(a.num_tiles, t_begin + a.tiles_per_cta);
  const uint64_t pol = policy_evict_first();
  const int q_begin = E * (int)tid;  // this thread's contiguous local nonzero positions [q_begin, q_begin+E)

  for (int w = tid; w < 2 * Cfg::kCap; w += NT) (&sm.tailrow[0][0])[w] = 0;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&sm.bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  // PDL: everything above overlapped the partition kernel; coords are read below.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (tid == 0)
    for (int s = 0; s < S && t_begin + s < t_end; ++s) pipe_issue<NT, E, S>(a, sm, t_begin + s, s, pol);
  __syncthreads();  // publishes the prologue's generic (array-end) stores

  float cta_carry = 0.f;
  int i_last = 0;
  for (int t = t_begin; t < t_end; ++t) {
    const int n = t - t_begin;
    const int st = n % S;
    const int b = n & 1;
    const int2 c0 = a.coords[t], c1 = a.coords[t + 1];
    const int i0 = c0.x, j0 = c0.y, i1 = c1.x, j1 = c1.y;
    const int nrows = i1 - i0;
    const int jA = j0 & ~3, oA = i0 & ~3;
    const int lo = j0 - jA, hi = j1 - jA;
    mbar_wait(&sm.bar[st], (uint32_t)((n / S) & 1));

    // (1) row pass: mark each row's last nonzero in the tile, or write rows without one
    {
      const int* so = &sm.off[st][i0 - oA];
      for (int r = tid; r < nrows; r += NT) {
        const int e = so[r + 1] - jA;
        const int s = r == 0 ? lo : so[r] - jA;
        if (e > s) sm.tailrow[b][e - 1] = (unsigned short)(r + 1);
        else a.y[i0 + r] = r == 0 ? cta_carry : 0.f;
      }
    }
    __syncthreads();

    // (2) nonzero pass over this thread's E contiguous positions
    float first_val = 0.f, run = 0.f;
    int first_r = -1;
    unsigned tmask = 0u;
    if (q_begin < hi) {
      int cc[E];
      float vv[E], xv[E];
      unsigned tr[E / 2];
#pragma unroll
      for (int k = 0; k < E / 4; ++k) {
        const int4 ci = *reinterpret_cast<const int4*>(&sm.col[st][q_begin + 4 * k]);
        const float4 vi = *reinterpret_cast<const float4*>(&sm.val[st][q_begin + 4 * k]);
        const uint2 ti = *reinterpret_cast<const uint2*>(&sm.tailrow[b][q_begin + 4 * k]);
        cc[4 * k] = ci.x; cc[4 * k + 1] = ci.y; cc[4 * k + 2] = ci.z; cc[4 * k + 3] = ci.w;
        vv[4 * k] = vi.x; vv[4 * k + 1] = vi.y; vv[4 * k + 2] = vi.z; vv[4 * k + 3] = vi.w;
        tr[2 * k] = ti.x; tr[2 * k + 1] = ti.y;
      }
#pragma unroll
      for (int e = 0; e < E; ++e) {  // all gathers in flight before any use
        const bool ok = q_begin + e >= lo && q_begin + e < hi;
        xv[e] = ok ? ld_x(a.x + cc[e]) : 0.f;
        if (!ok) vv[e] = 0.f;
      }
#pragma unroll
      for (int e = 0; e < E; ++e) {
        run = fmaf(vv[e], xv[e], run);
        const unsigned rid = (e & 1) ? (tr[e >> 1] >> 16) : (tr[e >> 1] & 0xFFFFu);
        if (rid) {
          const int r = (int)rid - 1;
          if (first_r < 0) {
            first_r = r;          // needs the carry-in from earlier threads: stored after the scans
            first_val = run;
          } else {
            a.y[i0 + r] = run;    // row started in this thread: final (r > 0 here)
          }
          run = 0.f;
        }
      }
#pragma unroll
      for (int k = 0; k < E / 2; ++k) tmask |= tr[k];
    }
    bool f = first_r >= 0;
    float val = run;
    warp_segscan_incl(f, val, lane);
    float lval = __shfl_up_sync(kFull, val, 1);      // every lane must execute full-mask shuffles
    const int lf = __shfl_up_sync(kFull, (int)f, 1);
    const bool lflag = lane ? (bool)lf : false;
    if (lane == 0) lval = 0.f;
    if (lane == 31) {
      sm.cflag[warp] = f;
      sm.cval[warp] = val;
    }
    __syncthreads();
    // stage st is fully consumed: refill it with tile t + S (async proxy after generic reads)
    if (tid == 0 && t + S < t_end) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      pipe_issue<NT, E, S>(a, sm, t + S, st, pol);
    }

    // (3) warp-chunk scan; the first row end of each thread gets its carry-in
    bool cf = lane < (unsigned)kW ? (bool)sm.cflag[lane] : false;
    float cv = lane < (unsigned)kW ? sm.cval[lane] : 0.f;
    warp_segscan_incl(cf, cv, lane);
    const float agg_val = __shfl_sync(kFull, cv, kW - 1);
    float ex_v = __shfl_up_sync(kFull, cv, 1);
    if (lane == 0) ex_v = 0.f;
    const float chunk_in = __shfl_sync(kFull, ex_v, warp);
    if (first_r >= 0) {
      float yv = (lflag ? lval : chunk_in + lval) + first_val;
      if (first_r == 0) yv += cta_carry;
      a.y[i0 + first_r] = yv;
    }
    if (tmask) {  // clear this thread's row marks for tile t+2
#pragma unroll
      for (int k = 0; k < E / 4; ++k) *reinterpret_cast<uint2*>(&sm.tailrow[b][q_begin + 4 * k]) = make_uint2(0u, 0u);
    }
    cta_carry = nrows > 0 ? agg_val : cta_carry + agg_val;
    i_last = i1;
  }

  // carry of this CTA's run, then the last CTA to finish applies all carries (Alg.3 fix-up)
  if (tid == 0) {
    if (t_begin < t_end) {
      a.carry_row[blockIdx.x] = i_last;
      a.carry_val[blockIdx.x] = cta_carry;
    }
    __threadfence();
    const unsigned done = atomicAdd(a.ticket, 1u);
    sm.last = done == gridDim.x - 1;
  }
  __syncthreads();
  if (sm.last) {
    __threadfence();
    const int nc = (int)gridDim.x;
    for (int c = tid; c < nc; c += NT) {
      const int r = __ldcg(a.carry_row + c);
      if (r >= a.rows) continue;
      if (c > 0 && __ldcg(a.carry_row + c - 1) == r) continue;
      float s = 0.f;
      for (int k = c; k < nc && __ldcg(a.carry_row + k) == r; ++k) s += __ldcg(a.carry_val + k);
      a.y[r] = __ldcg(a.y + r) + s;
    }
    if (tid == 0) *a.ticket = 0u;
  }
}

// ----------------------------------------------------------------------------- merge-path tiles, direct (default)
// The default tile processor.  On B200 every in-flight x[col] gather miss holds a 128-byte L1
// line, so the gather rate follows the L1 capacity left over by shared memory
// (profiles/r01_microbench_l1.txt: ~75 GNZ/s with 30 KB of L1, ~270 with 250 KB).  This kernel
// therefore keeps shared memory to ~4 KB per CTA and streams the tile's col/val with coalesced
// 128-bit loads straight into registers (thread t owns local nonzeros [4t, 4t+4), which makes
// the per-thread contiguous layout and the coalesced layout the same thing), prefetching the
// next tile's col/val/offsets while the current tile is reduced, and issuing the next tile's
// gathers before the second barrier of the current one.
struct DirectTile {
  int i0, j0, i1, j1;   // tile coordinates
  int4 col;             // this thread's 4 column indices (positions 4t..4t+3 from j0&~3)
  float4 val;           // and values (0 outside [j0, j1))
  int off_lo, off_hi;   // off[i0 + t], off[i0 + t + 1] for the row pass (t < rows of the tile)
};

template <int NT>
__device__ __forceinline__ void direct_load(const PipeArgs& a, int t, int tid, DirectTile& d) {
  const int2 c0 = a.coords[t], c1 = a.coords[t + 1];
  d.i0 = c0.x; d.j0 = c0.y; d.i1 = c1.x; d.j1 = c1.y;
  const int jA = d.j0 & ~3;
  const int g = jA + 4 * tid;
  if (g < d.j1 && g + 4 <= a.nnz) {
    d.col = ld_cs_v4(a.col + g);
    d.val = ld_cs_v4(a.val + g);
  } else {
    int c[4] = {0, 0, 0, 0};
    float v[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (g + e < d.j1) { c[e] = ld_cs(a.col + g + e); v[e] = ld_cs(a.val + g + e); }
    d.col = make_int4(c[0], c[1], c[2], c[3]);
    d.val = make_float4(v[0], v[1], v[2], v[3]);
  }
  const int nrows = d.i1 - d.i0;
  if (tid < nrows) {
    d.off_lo = __ldg(a.off + d.i0 + tid);
    d.off_hi = __ldg(a.off + d.i0 + tid + 1);
  }
}

// gathers for positions [lo, hi) of the tile (others contribute exactly 0)
template <bool XKEEP>
__device__ __forceinline__ void direct_gather(const PipeArgs& a, const DirectTile& d, int tid, float4& xv, float4& vv,
                                              uint64_t xpol) {
  const int jA = d.j0 & ~3;
  const int q0 = 4 * tid, lo = d.j0 - jA, hi = d.j1 - jA;
  const int cc[4] = {d.col.x, d.col.y, d.col.z, d.col.w};
  const float vl[4] = {d.val.x, d.val.y, d.val.z, d.val.w};
  float xr[4], vr[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const bool ok = q0 + e >= lo && q0 + e < hi;
    xr[e] = ok ? (XKEEP ? ld_x_keep(a.x + cc[e], xpol) : ld_x(a.x + cc[e])) : 0.f;
    vr[e] = ok ? vl[e] : 0.f;
  }
  xv = make_float4(xr[0], xr[1], xr[2], xr[3]);
  vv = make_float4(vr[0], vr[1], vr[2], vr[3]);
}

template <int NT, int MINB, bool XKEEP>
__global__ void __launch_bounds__(NT, MINB) merge_direct_kernel(PipeArgs a) {
  constexpr int kW = NT / 32;
  constexpr int kCap = 4 * NT;  // local nonzero positions per tile (L = kCap - 8)
  __shared__ __align__(16) unsigned short s_tailrow[2][kCap];
  __shared__ int s_cflag[kW];
  __shared__ float s_cval[kW];
  __shared__ int s_last;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t_begin = blockIdx.x * a.tiles_per_cta;
  const int t_end = min(a.num_tiles, t_begin + a.tiles_per_cta);
  const uint64_t xpol = XKEEP ? policy_evict_last() : 0ull;
  for (int w = tid; w < 2 * kCap; w += NT) (&s_tailrow[0][0])[w] = 0;
  // PDL: the prologue above overlapped the partition kernel; coords are read below.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();

  // Three-stage software pipeline per thread: while tile t is reduced, tile t+1's gathers are
  // in flight and tile t+2's col/val/offsets stream in from DRAM.
  DirectTile cur, mid, nxt;         // tile t (gathered), t+1 (loaded, being gathered), t+2 (loading)
  float4 xv_cur = make_float4(0.f, 0.f, 0.f, 0.f), vv_cur = xv_cur, xv_mid = xv_cur, vv_mid = xv_cur;
  if (t_begin < t_end) direct_load<NT>(a, t_begin, tid, cur);
  if (t_begin + 1 < t_end) direct_load<NT>(a, t_begin + 1, tid, mid);
  if (t_begin < t_end) direct_gather<XKEEP>(a, cur, tid, xv_cur, vv_cur, xpol);

  float cta_carry = 0.f;
  int i_last = 0;
  for (int t = t_begin; t < t_end; ++t) {
    const int b = (t - t_begin) & 1;
    const int i0 = cur.i0, nrows = cur.i1 - cur.i0;
    const int jA = cur.j0 & ~3, lo = cur.j0 - jA;
    // (1) row pass: mark each row's last nonzero, or write rows without a nonzero in the tile
    for (int r = tid; r < nrows; r += NT) {
      const int ob = r == tid ? cur.off_lo : __ldg(a.off + i0 + r);
      const int oe = r == tid ? cur.off_hi : __ldg(a.off + i0 + r + 1);
      const int e = oe - jA;
      const int s = r == 0 ? lo : ob - jA;
      if (e > s) s_tailrow[b][e - 1] = (unsigned short)(r + 1);
      else a.y[i0 + r] = r == 0 ? cta_carry : 0.f;
    }
    // (2) gathers of tile t+1 (its col arrived during the previous tile), loads of tile t+2
    if (t + 1 < t_end) direct_gather<XKEEP>(a, mid, tid, xv_mid, vv_mid, xpol);
    if (t + 2 < t_end) direct_load<NT>(a, t + 2, tid, nxt);
    __syncthreads();

    // (3) this thread's 4 nonzeros: row sums, non-first row ends stored directly
    const uint2 tr = *reinterpret_cast<const uint2*>(&s_tailrow[b][4 * tid]);
    const unsigned rid[4] = {tr.x & 0xFFFFu, tr.x >> 16, tr.y & 0xFFFFu, tr.y >> 16};
    const float xa[4] = {xv_cur.x, xv_cur.y, xv_cur.z, xv_cur.w};
    const float va[4] = {vv_cur.x, vv_cur.y, vv_cur.z, vv_cur.w};
    float run = 0.f, first_val = 0.f;
    int first_r = -1;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      run = fmaf(va[e], xa[e], run);
      if (rid[e]) {
        const int r = (int)rid[e] - 1;
        if (first_r < 0) { first_r = r; first_val = run; }
        else a.y[i0 + r] = run;  // row started inside this thread (r > 0)
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
    __syncthreads();

    // (4) warp-chunk scan; the first row end of each thread gets its carry-in
    bool cf = lane < kW ? (bool)s_cflag[lane] : false;
    float cv = lane < kW ? s_cval[lane] : 0.f;
    warp_segscan_incl(cf, cv, (unsigned)lane);
    const float agg_val = __shfl_sync(kFull, cv, kW - 1);
    float ex_v = __shfl_up_sync(kFull, cv, 1);
    if (lane == 0) ex_v = 0.f;
    const float chunk_in = __shfl_sync(kFull, ex_v, warp);
    if (first_r >= 0) {
      float yv = (lflag ? lval : chunk_in + lval) + first_val;
      if (first_r == 0) yv += cta_carry;
      a.y[i0 + first_r] = yv;
    }
    if (tr.x | tr.y) *reinterpret_cast<uint2*>(&s_tailrow[b][4 * tid]) = make_uint2(0u, 0u);
    cta_carry = nrows > 0 ? agg_val : cta_carry + agg_val;
    i_last = cur.i1;
    cur = mid;
    xv_cur = xv_mid;
    vv_cur = vv_mid;
    mid = nxt;
  }

  // carry of this CTA's run; the last CTA to finish applies all carries (Alg.3 fix-up)
  if (tid == 0) {
    if (t_begin < t_end) {
      a.carry_row[blockIdx.x] = i_last;
      a.carry_val[blockIdx.x] = cta_carry;
    }
    __threadfence();
    const unsigned done = atomicAdd(a.ticket, 1u);
    s_last = done == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    const int nc = (int)gridDim.x;
    for (int c = tid; c < nc; c += NT) {
      const int r = __ldcg(a.carry_row + c);
      if (r >= a.rows) continue;
      if (c > 0 && __ldcg(a.carry_row + c - 1) == r) continue;
      float sum = 0.f;
      for (int k = c; k < nc && __ldcg(a.carry_row + k) == r; ++k) sum += __ldcg(a.carry_val + k);
      a.y[r] = __ldcg(a.y + r) + sum;
    }
    if (tid == 0) *a.ticket = 0u;
  }
}

// ----------------------------------------------------------------------------- merge-path tiles, wide
// Like merge_direct_kernel but each thread owns E = 8 or 16 contiguous nonzeros of the tile, read
// with 256-bit loads (sm_100a LDG.256, L1 no-allocate, L2 evict-first): the per-tile scans and
// barriers are amortised over 2-4x more nonzeros, and a warp still reads whole 32-byte sectors.
// Tile length L = NT*E - 8: the 32-byte-aligned nonzero range [j0&~7, j1) spans <= L + 7.
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

template <int E>
struct WideTile {
  int i0, j0, i1, j1;
  int col[E];
  float val[E];
  int off_lo, off_hi;
};

template <int NT, int E>
__device__ __forceinline__ void wide_load(const PipeArgs& a, int4 c, int tid, WideTile<E>& d, uint64_t spol) {
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

// tile t's coordinates (i0, j0, i1, j1)
__device__ __forceinline__ int4 tile_coords(const PipeArgs& a, int t) {
  const int2 c0 = a.coords[t], c1 = a.coords[t + 1];
  return make_int4(c0.x, c0.y, c1.x, c1.y);
}

// x gathers for valid positions; the gathered value replaces col (as float bits) to save registers
template <int E>
__device__ __forceinline__ void wide_gather(const PipeArgs& a, WideTile<E>& d, int tid, float (&xv)[E]) {
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

// Segmented inclusive scan over the first N lanes only (N a power of two <= 32).
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

template <int NT, int E, int MINB>
__global__ void __launch_bounds__(NT, MINB) merge_wide_kernel(PipeArgs a) {
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
  float cta_carry = 0.f;
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
      else a.y[i0 + r] = r == 0 ? cta_carry : 0.f;
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
      if (first_r == 0) yv += cta_carry;
      a.y[i0 + first_r] = yv;
    }
    if (any) {
#pragma unroll
      for (int k = 0; k < E / 8; ++k)
        *reinterpret_cast<uint4*>(&s_tailrow[b][E * tid + 8 * k]) = make_uint4(0u, 0u, 0u, 0u);
    }
    cta_carry = nrows > 0 ? agg_val : cta_carry + agg_val;
    i_last = cur.i1;
    cur = nxt;
  }

  if (tid == 0) {
    if (t_begin < t_end) {
      a.carry_row[blockIdx.x] = i_last;
      a.carry_val[blockIdx.x] = cta_carry;
    }
    __threadfence();
    const unsigned done = atomicAdd(a.ticket, 1u);
    s_last = done == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    const int nc = (int)gridDim.x;
    for (int c = tid; c < nc; c += NT) {
      const int r = __ldcg(a.carry_row + c);
      if (r >= a.rows) continue;
      if (c > 0 && __ldcg(a.carry_row + c - 1) == r) continue;
      float sum = 0.f;
      for (int k = c; k < nc && __ldcg(a.carry_row + k) == r; ++k) sum += __ldcg(a.carry_val + k);
      a.y[r] = __ldcg(a.y + r) + sum;
    }
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
#ifndef LB_PRED_TAIL
#define LB_PRED_TAIL 1  // stream_reduce_round: predicated first-row store and tail clear, no branches
                        // (C3 291.5 -> 294.5 GNZ/s, C4 253.1 -> 255.5; 0 = the branchy form)
#endif
#ifndef LB_STEP_SYNC
#define LB_STEP_SYNC 0  // merge_stream_kernel: 1 = __syncwarp after every round; 0 = only after a tile's row pass
                        // (lanes touch only their own tail[] entries inside a tile): C3 286.7 -> 291.4 GNZ/s
#endif

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

__device__ __forceinline__ void stream_load(const PipeArgs& a, int4 c, int k, int lane, StreamRound& d,
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
template <bool XKEEP, int TIER>
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
  return XKEEP ? ld_x_keep(x + c, xpol) : ld_x(x + c);
}

// the 8 gathers of a lane's round (every loaded column index is valid; positions outside the tile
// are masked later by zeroing their values)
template <bool XKEEP, int TIER>
__device__ __forceinline__ void gx8(const float* __restrict__ x, const float* __restrict__ xw, int cols, uint32_t sxb,
                                    const StreamRound& d, float (&xv)[8], uint64_t xpol, uint64_t cpol) {
#pragma unroll
  for (int e = 0; e < 8; ++e) xv[e] = gx<XKEEP, TIER>(x, xw, cols, sxb, d.col[e], xpol, cpol);
}

// y store predicated on `p` (no branch)
__device__ __forceinline__ void st_cs_if(float* ptr, float v, bool p) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.global.cs.f32 [%0], %1;\n\t}"
               :: "l"(ptr), "f"(v), "r"((unsigned)p) : "memory");
}

template <int R, int K>
__device__ __forceinline__ void stream_prefetch_offsets(const PipeArgs& a, int4 c, int lane, int (&lo_)[K],
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

// y stores of the warp-streamed kernel.  With PEERS (the fix-up of the fused multi-GPU epilogue,
// DESIGN.md 7b) the value also goes to every other rank's copy of y over NVLink; `peers` = false for a
// partial value, which stays local.
template <bool PEERS>
__device__ __forceinline__ void put_y(const PipeArgs& a, int idx, float v, bool peers = true) {
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
__device__ __forceinline__ bool stream_row_pass(const PipeArgs& a, int4 c, int lane, const int (&lo_)[K],
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
__device__ __forceinline__ void tail_clear8(unsigned short* p) { *reinterpret_cast<uint4*>(p) = make_uint4(0u, 0u, 0u, 0u); }
__device__ __forceinline__ void tail_clear8(unsigned* p) {
  *reinterpret_cast<uint4*>(p) = make_uint4(0u, 0u, 0u, 0u);
  *reinterpret_cast<uint4*>(p + 4) = make_uint4(0u, 0u, 0u, 0u);
}

// Fused multi-GPU epilogue (PEERS): when a tile is done, its final rows [i0, i1) -- every row that ends
// in the tile, written to the local y by this warp (the row pass, the rounds) -- are copied to every
// other rank's y with coalesced stores over NVLink.  The warp's first row is excluded when it started
// before the warp's run (`open_row`, partial: the fix-up completes it and sends it).  One coalesced
// pass per tile instead of a peer store per row end keeps the epilogue off the rounds' critical path
// (measured: a software-pipelined variant of this copy was no faster).
__device__ __forceinline__ void stream_peer_copy(const PipeArgs& a, int4 c, int open_row, int lane) {
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
__device__ __forceinline__ void stream_reduce_round(const PipeArgs& a, int4 cT, int k, int lane, bool r0e,
                                                    float (&val)[8], const float (&xc)[8], TailT* tail, float& rc) {
  // (b) the row open at the tile start has no nonzero here: it ends now with the carry
  const int i0 = cT.x;
  if (k == 0 && r0e) {
    if (lane == 0) put_y<false>(a, i0, rc);
    rc = 0.f;
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
#if LB_PRED_TAIL
  {  // branch-free: predicated store of the first row end, predicated clear of the lane's tail entries
    const bool lf = (B & ((1u << lane) - 1u)) != 0u;  // a row ended in an earlier lane
    const float carry_in = lane == 0 ? rc : (lf ? lval : rc + lval);
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
#else
  if (first_rid != 0u) {
    const bool lf = (B & ((1u << lane) - 1u)) != 0u;  // a row ended in an earlier lane
    const float carry_in = lane == 0 ? rc : (lf ? lval : rc + lval);
    const int row = i0 - 1 + (int)first_rid;
    if (!(LB_ABL & 1) || (LB_ABL & 4)) put_y<false>(a, row, carry_in + first_val);
  }
  if (any && !(LB_ABL & 4)) tail_clear8(&tail[256 * k + 8 * lane]);
#endif
  rc = B ? agg_v : rc + agg_v;
}

// One carry per warp (rows == a.rows for warps without tiles: skipped by the fix-up), then the
// last CTA to finish applies all carries in warp order (Alg.3 fix-up P:332-337, deterministic).
template <bool PEERS>
__device__ __forceinline__ void stream_carries_fixup(const PipeArgs& a, int gw, int lane, int W, int i_last, float rc,
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
    const int nc = (int)gridDim.x * W;
    for (int c = threadIdx.x; c < nc; c += W * 32) {
      const int r = __ldcg(a.carry_row + c);
      if (r >= a.rows) continue;
      if (c > 0 && __ldcg(a.carry_row + c - 1) == r) continue;
      float sum = 0.f;
      for (int kk = c; kk < nc && __ldcg(a.carry_row + kk) == r; ++kk) sum += __ldcg(a.carry_val + kk);
      put_y<PEERS>(a, r, __ldcg(a.y + r) + sum);
    }
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
template <int W, int R, int MINB, bool XKEEP, typename TailT = unsigned short, int TIER = 0, bool PEERS = false>
__global__ void __launch_bounds__(W * 32, MINB) merge_stream_kernel(PipeArgs a) {
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
  const uint64_t xpol = (XKEEP || TIER == 2) ? policy_evict_last() : 0ull;
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

  float rc = 0.f;  // partial sum of the row open at the current stream position (warp-uniform)
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
    gx8<XKEEP, TIER>(xg, xw, a.cols, sxb, D0, X0, xpol, spol);

    int t = t_begin, k = 0, st = 0;
    auto step = [&](StreamRound& dc, float (&xc)[8], StreamRound& dn, float (&xn)[8], StreamRound& dl) {
      // (a) gathers for round st+1, loads for round st+2
      if (st + 1 < nsteps) gx8<XKEEP, TIER>(xg, xw, a.cols, sxb, dn, xn, xpol, spol);
      if (st + 2 < nsteps) {
        const int k2 = k + 2;
        const bool same = k2 < R;
        stream_load(a, same ? cT : cT1, same ? k2 : k2 - R, lane, dl, spol);
      }
      stream_reduce_round(a, cT, k, lane, r0e, dc.val, xc, tail, rc);
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
#if LB_STEP_SYNC == 0
        __syncwarp();  // the row pass's tail[] writes before the next round's reads
#endif
      }
#if LB_STEP_SYNC
      __syncwarp();
#endif
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

  stream_carries_fixup<PEERS>(a, gw, lane, W, i_last, rc, s_last);
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
    gx8<false, TIER>(x, x_warm, cols, sxb, d, xv, xpol, pol);
#pragma unroll
    for (int e = 0; e < 8; ++e) s = fmaf(d.val[e], xv[e], s);
  }
  for (; i < nnz; ++i) s = fmaf(val[i], gx<false, TIER>(x, x_warm, cols, sxb, col[i], xpol, pol), s);
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

// ----------------------------------------------------------------------------- hot-column plan
// B200 extension (not in the paper).  On random-column matrices the tile
// processor is bound by x[col] gathers that miss L1 (~1 L1TEX line per clock per SM), while shared
// memory serves random 4-byte reads several times faster.  A plan picks the `slots` columns with
// the most stored entries (ties: lower column id first; only columns with >= 2 entries), assigns
// them shared-memory slots, and rewrites a private copy of col_idx with ~slot for those entries.
// Every call gathers x of the hot columns once (partition_xhot_kernel) and each CTA stages them in
// shared memory.  Products and summation order are unchanged, so results are bitwise identical.

// deg[c] = number of stored entries in column c (deg zeroed by the caller)
__global__ void col_degree_kernel(int64_t nnz, const int* __restrict__ col, int* __restrict__ deg) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += stride)
    atomicAdd(deg + __ldcs(col + k), 1);
}

// bins[b] += #{c : lo <= deg[c] < hi, (deg[c] - lo) / w == b}; block-private shared histogram
constexpr int kDegBins = 8192;
__global__ void __launch_bounds__(256) degree_hist_kernel(int cols, const int* __restrict__ deg, int64_t lo,
                                                          int64_t hi, int64_t w, int* __restrict__ bins) {
  __shared__ int h[kDegBins];
  for (int i = threadIdx.x; i < kDegBins; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < cols; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = __ldg(deg + c);
    if (d >= lo && d < hi) atomicAdd(&h[(d - lo) / w], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kDegBins; i += blockDim.x)
    if (h[i]) atomicAdd(bins + i, h[i]);
}

// Tier assignment in column order.  Column c is HOT if deg[c] >= t1_hi, or deg[c] == t1_tie and it
// is among the first b1 such columns; WARM if it is not hot and deg[c] >= t2.  256 threads x 16
// columns per block; plan_count_kernel counts (above, tie, >= t2) per block, plan_scan_kernel turns
// the counts into exclusive offsets (one block), plan_assign_kernel writes the tier map.
constexpr int kHotPer = 16;
constexpr int kHotChunk = 256 * kHotPer;

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

__global__ void __launch_bounds__(256) plan_count_kernel(int cols, const int* __restrict__ deg, int t1_hi, int t1_tie,
                                                         int t2, int4* __restrict__ blk) {
  const int64_t c0 = (int64_t)blockIdx.x * kHotChunk + (int64_t)threadIdx.x * kHotPer;
  int a = 0, b = 0, c = 0;
#pragma unroll
  for (int i = 0; i < kHotPer; ++i) {
    if (c0 + i < cols) {
      const int d = __ldg(deg + c0 + i);
      a += d >= t1_hi;
      b += d == t1_tie;
      c += d >= t2;
    }
  }
  int4 tot;
  block_excl_scan3(make_int4(a, b, c, 0), &tot);
  if (threadIdx.x == 0) blk[blockIdx.x] = tot;
}

// one block: per-block counts -> exclusive offsets (x: above t1, y: t1 ties, z: warm); a block's
// warm count is (>= t2) - above - (ties admitted as hot: clamp(b1 - tie offset, 0, ties)), valid
// because the host only enables the warm tier (warm_on) with t2 <= t1_tie (every hot column >= t2).
// totals = (above, ties, >= t2, warm)
__global__ void __launch_bounds__(1024) plan_scan_kernel(int n, int b1, int warm_on, int4* __restrict__ blk,
                                                         int* __restrict__ totals) {
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int b0 = threadIdx.x * per;
  int a = 0, b = 0, c = 0;
  for (int i = 0; i < per; ++i)
    if (b0 + i < n) { a += blk[b0 + i].x; b += blk[b0 + i].y; c += blk[b0 + i].z; }
  int4 tot;
  const int4 ex = block_excl_scan3(make_int4(a, b, c, 0), &tot);
  // pass 2 needs each block's tie offset: recompute sequentially per thread, then scan warm counts
  int ra = ex.x, rb = ex.y;
  int wsum = 0;
  for (int i = 0; i < per; ++i)
    if (b0 + i < n) {
      const int4 v = blk[b0 + i];
      const int admitted = min(max(b1 - rb, 0), v.y);
      wsum += warm_on ? v.z - v.x - admitted : 0;
      ra += v.x;
      rb += v.y;
    }
  int4 wtot;
  const int4 wex = block_excl_scan3(make_int4(wsum, 0, 0, 0), &wtot);
  ra = ex.x;
  rb = ex.y;
  int rw = wex.x;
  for (int i = 0; i < per; ++i)
    if (b0 + i < n) {
      const int4 v = blk[b0 + i];
      const int admitted = min(max(b1 - rb, 0), v.y);
      blk[b0 + i] = make_int4(ra, rb, rw, 0);
      rw += warm_on ? v.z - v.x - admitted : 0;
      ra += v.x;
      rb += v.y;
    }
  if (threadIdx.x == 0) { totals[0] = tot.x; totals[1] = tot.y; totals[2] = tot.z; totals[3] = wtot.x; }
}

// deg_smap: in deg[c]; out -1 (cold), slot s < n_hot (hot), n_hot + w (warm w); hot_cols[s] = c,
// warm_cols[w] = c; sums[0] += degrees of hot columns, sums[1] += degrees of warm columns
__global__ void __launch_bounds__(256) plan_assign_kernel(int cols, int* __restrict__ deg_smap, int t1_hi, int t1_tie,
                                                          int t2, int n_above, int b1, int n_hot,
                                                          const int4* __restrict__ blk, int* __restrict__ hot_cols,
                                                          int* __restrict__ warm_cols,
                                                          unsigned long long* __restrict__ sums) {
  const int64_t c0 = (int64_t)blockIdx.x * kHotChunk + (int64_t)threadIdx.x * kHotPer;
  int d[kHotPer];
  int a = 0, b = 0;
#pragma unroll
  for (int i = 0; i < kHotPer; ++i) {
    d[i] = c0 + i < cols ? deg_smap[c0 + i] : 0;
    a += d[i] >= t1_hi;
    b += d[i] == t1_tie;
  }
  // warm count of this thread depends on its tie ranks: computed in the walk below, so the block
  // scan of warm counts is done on the walk's result
  const int4 ex = block_excl_scan3(make_int4(a, b, 0, 0), nullptr);
  int ra = blk[blockIdx.x].x + ex.x, rb = blk[blockIdx.x].y + ex.y;
  int slot[kHotPer];
  int nw = 0;
#pragma unroll
  for (int i = 0; i < kHotPer; ++i) {
    int sl = -1;
    if (c0 + i < cols) {
      if (d[i] >= t1_hi) sl = ra++;
      else if (d[i] == t1_tie) {
        if (rb < b1) sl = n_above + rb;
        ++rb;
      }
      if (sl < 0 && d[i] >= t2) { sl = -2; ++nw; }  // warm, numbered below
    }
    slot[i] = sl;
  }
  const int4 wex = block_excl_scan3(make_int4(nw, 0, 0, 0), nullptr);
  int rw = blk[blockIdx.x].z + wex.x;
  unsigned long long hs = 0, wsum = 0;
#pragma unroll
  for (int i = 0; i < kHotPer; ++i) {
    if (c0 + i >= cols) break;
    int v = slot[i];
    if (v >= 0) {
      hot_cols[v] = (int)(c0 + i);
      hs += (unsigned)d[i];
    } else if (v == -2) {
      warm_cols[rw] = (int)(c0 + i);
      wsum += (unsigned)d[i];
      v = n_hot + rw++;
    }
    deg_smap[c0 + i] = v;
  }
  for (int o = 16; o > 0; o >>= 1) {
    hs += __shfl_xor_sync(kFull, hs, o);
    wsum += __shfl_xor_sync(kFull, wsum, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (hs) atomicAdd(sums, hs);
    if (wsum) atomicAdd(sums + 1, wsum);
  }
}

// hcol[k] = ~slot (hot), cols + w (warm) or col[k] (cold)
__global__ void plan_remap_kernel(int64_t nnz, int cols, int n_hot, const int* __restrict__ col,
                                  const int* __restrict__ smap, int* __restrict__ hcol) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += stride) {
    const int c = __ldcs(col + k);
    const int v = __ldg(smap + c);
    hcol[k] = v < 0 ? c : (v < n_hot ? ~v : cols + (v - n_hot));
  }
}

// ----------------------------------------------------------------------------- SSSP (NEXT-4)
// Listing 5: each round relaxes the out-edges of the frontier vertices,
//   dist[v] = atomicMin(dist[v], dist[u] + w(u, v)),  v joins the next frontier if it improved,
// until the frontier is empty.  Distances are fp32 >= 0 (or +inf), whose bit patterns order like
// int32, so atomicMin on the int view is the float minimum.  The frontier is a vertex list; a vertex
// is pushed at most once per round (stamp[v] = round of its last push).  The edges of a round are
// balanced by the chosen schedule: thread-mapped (a thread per frontier vertex), group-mapped (a warp
// takes 32 frontier vertices and strides their edge pool, Alg.2) or merge-path (frontier vertices +
// edges split evenly into per-thread diagonal ranges, each found by the 2-D search, Alg.3).

// Relax edge (u -> v) with candidate distance nd = dist[u] + w.  A plain read of dist[v] first
// skips the atomic when nd cannot improve it (distances only decrease, so a stale read is never
// smaller than the current value); the vertices pushed to the next frontier are counted with one
// atomicAdd per group of lanes that push together (warp-aggregated).
__device__ __forceinline__ void sssp_relax(int v, float nd, float* __restrict__ dist, int* __restrict__ stamp,
                                           int round, int* __restrict__ q_out, int* __restrict__ n_out) {
  bool push = false;
  if (__float_as_int(nd) < __ldcg(reinterpret_cast<const int*>(dist) + v)) {
    const int old = atomicMin(reinterpret_cast<int*>(dist) + v, __float_as_int(nd));
    push = __float_as_int(nd) < old && atomicExch(stamp + v, round) != round;
  }
  const unsigned active = __activemask();
  const unsigned m = __ballot_sync(active, push);
  if (push) {
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(n_out, __popc(m));
    base = __shfl_sync(m, base, leader);
    q_out[base + __popc(m & ((1u << lane) - 1u))] = v;
  }
}

__global__ void sssp_init_kernel(int n, int source, float* __restrict__ dist, int* __restrict__ stamp,
                                 int* __restrict__ q_in, int* __restrict__ counts) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += stride) {
    dist[v] = v == source ? 0.f : __int_as_float(0x7f800000);
    stamp[v] = -1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    q_in[0] = source;
    counts[0] = 1;  // frontier size
    counts[1] = 0;  // next frontier size
    counts[2] = 0;  // negative-weight flag
  }
}

// any weight < 0 (or NaN) sets flag
__global__ void sssp_check_weights_kernel(int64_t nnz, const float* __restrict__ w, int* flag) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += stride)
    if (!(__ldg(w + k) >= 0.f)) { atomicExch(flag, 1); return; }
}

__global__ void sssp_thread_kernel(int F, const int* __restrict__ q_in, const int* __restrict__ off,
                                   const int* __restrict__ col, const float* __restrict__ w, float* __restrict__ dist,
                                   int* __restrict__ stamp, int round, int* __restrict__ q_out,
                                   int* __restrict__ n_out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= F) return;
  const int u = q_in[i];
  const float du = __ldcg(dist + u);
  for (int e = __ldg(off + u); e < __ldg(off + u + 1); ++e)
    sssp_relax(__ldg(col + e), du + __ldg(w + e), dist, stamp, round, q_out, n_out);
}

// group-mapped (G = 32): a warp takes 32 frontier vertices, scans their degrees and strides the pool
__global__ void sssp_warp_kernel(int F, const int* __restrict__ q_in, const int* __restrict__ off,
                                 const int* __restrict__ col, const float* __restrict__ w, float* __restrict__ dist,
                                 int* __restrict__ stamp, int round, int* __restrict__ q_out, int* __restrict__ n_out) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = gw * 32; base < F; base += nw * 32) {
    const int64_t i = base + lane;
    int u = 0, b = 0, cnt = 0;
    float du = 0.f;
    if (i < F) {
      u = q_in[i];
      b = __ldg(off + u);
      cnt = __ldg(off + u + 1) - b;
      du = __ldcg(dist + u);
    }
    const int incl = warp_incl_scan_int(cnt, lane);
    const int total = __shfl_sync(kFull, incl, 31);
    // uniform trip count so every lane takes part in the shuffles
    const int rounds_k = (total + 31) / 32;
    for (int rk = 0; rk < rounds_k; ++rk) {
      const int k = rk * 32 + lane;
      int lo = 0;  // first lane whose inclusive prefix exceeds k (binary lifting over the 32 prefixes)
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const int cand = lo + step;
        const int pv = __shfl_sync(kFull, incl, cand - 1);
        if (pv <= k) lo = cand;
      }
      const int src_lane = lo;
      const int pe = __shfl_sync(kFull, incl, src_lane > 0 ? src_lane - 1 : 0);  // every lane shuffles
      const int excl = src_lane ? pe : 0;
      const int bb = __shfl_sync(kFull, b, src_lane);
      const float dd = __shfl_sync(kFull, du, src_lane);
      if (k < total) {
        const int e = bb + (k - excl);
        sssp_relax(__ldg(col + e), dd + __ldg(w + e), dist, stamp, round, q_out, n_out);
      }
    }
  }
}

// Merge-path relaxation over CTA tiles (Listing 5 P:1076-1107 with Alg.3's split): the merge items of a
// round are the frontier vertices' ends and their out-edges (edge k of the round belongs to frontier
// vertex i with fo[i] <= k < fo[i+1]); CTA tile t takes items [t*kSsspTile, (t+1)*kSsspTile).  Thread
// 0 finds the tile's (vertex, edge) start and end by the 2-D search; the tile's frontier vertices are
// staged in shared memory (fo[i], off[u] - fo[i], dist[u]); each thread then takes 8 consecutive edges
// of the tile -- one shared-memory binary search for its first edge's vertex, then a forward walk --
// so a warp reads 256 consecutive edges' col/w (coalesced within each adjacency list) and issues the
// 8 edges' loads before relaxing them.  A stale (larger) dist[u] snapshot is harmless: a vertex whose
// distance drops during the round is pushed and re-relaxes its edges next round.
constexpr int kSsspTile = 2048;  // merge items per CTA tile (256 threads x 8)
#ifndef LB_SSSP_STAMP_PREFETCH
#define LB_SSSP_STAMP_PREFETCH 1  // read every edge's stamp up front: skips the exchange for pushed vertices (28.7 vs 35.0 ms, R-MAT-24)
#endif

__device__ __forceinline__ int sssp_diag(int F, int Ef, const int* __restrict__ fo, int64_t d) {
  // i = #{k < F : k + fo[k+1] < d}
  int lo = (int)(d - Ef > 0 ? d - Ef : 0), hi = (int)(d < F ? d : F);
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if ((int64_t)mid + __ldcg(fo + mid + 1) < d) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// tile boundaries of a round: tc[t] = frontier index of diagonal min(t kSsspTile, F + E_f), t = 0..T
// (one thread per boundary, all searches in parallel)
__global__ void __launch_bounds__(256) sssp_tile_coords_kernel(int F, const int* __restrict__ fo, int T,
                                                               int* __restrict__ tc) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > T) return;
  const int Ef = __ldcg(fo + F);
  const int64_t total = (int64_t)F + Ef;
  const int64_t d = (int64_t)t * kSsspTile < total ? (int64_t)t * kSsspTile : total;
  tc[t] = sssp_diag(F, Ef, fo, d);
}

__global__ void __launch_bounds__(256) sssp_merge_kernel(int F, const int* __restrict__ q_in,
                                                         const int* __restrict__ fo, const int* __restrict__ off,
                                                         const int* __restrict__ col, const float* __restrict__ w,
                                                         float* __restrict__ dist, int* __restrict__ stamp, int round,
                                                         int* __restrict__ q_out, int* __restrict__ n_out,
                                                         const int* __restrict__ tc) {
  __shared__ int s_fo[kSsspTile + 2];
  __shared__ int s_base[kSsspTile + 1];
  __shared__ float s_du[kSsspTile + 1];
  __shared__ int s_q[kSsspTile];  // this tile's pushes (<= its edges), flushed with one global atomic
  __shared__ int s_qn, s_qbase;
  const int tid = threadIdx.x;
  const int Ef = __ldcg(fo + F);
  const int64_t total = (int64_t)F + Ef;
  if (tid == 0) s_qn = 0;
  for (int64_t t = blockIdx.x; t * kSsspTile < total; t += gridDim.x) {
    const int64_t d0 = t * kSsspTile, d1 = d0 + kSsspTile < total ? d0 + kSsspTile : total;
    const int i0 = __ldcg(tc + t), i1 = __ldcg(tc + t + 1);
    const int j0 = (int)(d0 - i0), j1 = (int)(d1 - i1);
    const int nv = (i1 < F ? i1 : F - 1) - i0 + 1;  // frontier vertices touched: i0 .. min(i1, F-1)
    for (int q = tid; q < nv; q += 256) {
      const int i = i0 + q, u = q_in[i], f = __ldcg(fo + i);
      s_fo[q] = f;
      s_base[q] = __ldg(off + u) - f;
      s_du[q] = __ldcg(dist + u);
    }
    if (tid == 0) s_fo[nv > 0 ? nv : 0] = i0 + nv <= F - 1 ? __ldcg(fo + i0 + nv) : Ef;
    __syncthreads();
    const int k0 = j0 + 8 * tid;
    if (nv > 0 && k0 < j1) {
      // vertex of edge k0: the last q with s_fo[q] <= k0
      int lo = 0, hi = nv;  // answer in [0, nv)
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (s_fo[mid] <= k0) lo = mid; else hi = mid;
      }
      int q = lo;
      int ev[8];
      float dv[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int k = k0 + e;
        if (k < j1) {
          while (s_fo[q + 1] <= k) ++q;
          ev[e] = s_base[q] + k;
          dv[e] = s_du[q];
        } else {
          ev[e] = -1;
        }
      }
      int cv[8];
      float wv[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        cv[e] = ev[e] >= 0 ? __ldg(col + ev[e]) : 0;
        wv[e] = ev[e] >= 0 ? __ldg(w + ev[e]) : 0.f;
      }
      // relaxation: the stamps are read up front so that a vertex already pushed this round skips the
      // exchange; the atomicExch still decides, so every vertex is pushed at most once per round (the
      // frontier arrays hold n entries); pushes go to the tile's shared queue
#if LB_SSSP_STAMP_PREFETCH
      int sv[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) sv[e] = ev[e] >= 0 ? __ldcg(stamp + cv[e]) : round;
#endif
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (ev[e] < 0) continue;
        const int v = cv[e];
        const float nd = dv[e] + wv[e];
        if (__float_as_int(nd) < __ldcg(reinterpret_cast<const int*>(dist) + v)) {
          const int old = atomicMin(reinterpret_cast<int*>(dist) + v, __float_as_int(nd));
#if LB_SSSP_STAMP_PREFETCH
          if (__float_as_int(nd) < old && sv[e] != round && atomicExch(stamp + v, round) != round)
#else
          if (__float_as_int(nd) < old && atomicExch(stamp + v, round) != round)
#endif
            s_q[atomicAdd(&s_qn, 1)] = v;
        }
      }
    }
    __syncthreads();
    // flush the tile's pushes: one global reservation, coalesced stores
    const int qn = s_qn;
    if (qn > 0) {
      if (tid == 0) s_qbase = atomicAdd(n_out, qn);
      __syncthreads();
      const int qb = s_qbase;
      for (int q = tid; q < qn; q += 256) q_out[qb + q] = s_q[q];
    }
    __syncthreads();
    if (tid == 0) s_qn = 0;
  }
}

// exclusive scan of the frontier degrees: fo[i] = sum_{k<i} deg(q_in[k]), fo[F] = total.
// Three phases: per-block sums (kScanChunk items per block), one-block scan of the block sums, then
// per-block local scans plus the block offset.
constexpr int kScanChunk = 2048;  // 256 threads x 8
__global__ void __launch_bounds__(256) frontier_deg_sum_kernel(int F, const int* __restrict__ q_in,
                                                               const int* __restrict__ off, int* __restrict__ bsum) {
  const int b0 = blockIdx.x * kScanChunk + threadIdx.x * 8;
  int s = 0;
#pragma unroll
  for (int e = 0; e < 8; ++e)
    if (b0 + e < F) { const int u = q_in[b0 + e]; s += __ldg(off + u + 1) - __ldg(off + u); }
  int4 tot;
  block_excl_scan3(make_int4(s, 0, 0, 0), &tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot.x;
}
__global__ void __launch_bounds__(1024) frontier_bsum_scan_kernel(int nb, int* __restrict__ bsum) {
  const int per = (nb + blockDim.x - 1) / blockDim.x;
  const int b0 = threadIdx.x * per;
  int s = 0;
  for (int i = 0; i < per; ++i) if (b0 + i < nb) s += bsum[b0 + i];
  int4 tot;
  const int4 ex = block_excl_scan3(make_int4(s, 0, 0, 0), &tot);
  int r = ex.x;
  for (int i = 0; i < per; ++i)
    if (b0 + i < nb) { const int v = bsum[b0 + i]; bsum[b0 + i] = r; r += v; }
  if (threadIdx.x == 0) bsum[nb] = tot.x;
}
__global__ void __launch_bounds__(256) frontier_deg_scan_kernel(int F, const int* __restrict__ q_in,
                                                                const int* __restrict__ off,
                                                                const int* __restrict__ bsum, int nb,
                                                                int* __restrict__ fo) {
  const int b0 = blockIdx.x * kScanChunk + threadIdx.x * 8;
  int d[8], s = 0;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    d[e] = 0;
    if (b0 + e < F) { const int u = q_in[b0 + e]; d[e] = __ldg(off + u + 1) - __ldg(off + u); }
    s += d[e];
  }
  const int4 ex = block_excl_scan3(make_int4(s, 0, 0, 0), nullptr);
  int r = bsum[blockIdx.x] + ex.x;
#pragma unroll
  for (int e = 0; e < 8; ++e)
    if (b0 + e < F) { fo[b0 + e] = r; r += d[e]; }
  if (blockIdx.x == 0 && threadIdx.x == 0) fo[F] = bsum[nb];
}

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
  // empty rows are written here instead, so give it a PipeArgs whose y is unused (nullptr never hit
  // because we handle empty rows ourselves below)
  PipeArgs pa;
  pa.off = a.off; pa.coords = a.coords; pa.rows = a.rows; pa.nnz = a.nnz;
  float rc[P];
#pragma unroll
  for (int j = 0; j < P; ++j) rc[j] = 0.f;
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
        if (lane == 0) spmm_store<P>(a, i0, rc);
#pragma unroll
        for (int j = 0; j < P; ++j) rc[j] = 0.f;
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
        for (int j = 0; j < P; ++j) yv[j] = (lane == 0 ? rc[j] : (lf ? lval[j] : rc[j] + lval[j])) + first_val[j];
        spmm_store<P>(a, i0 + first_r, yv);
      }
      if (tq.x | tq.y) {
        if constexpr (E == 4) *reinterpret_cast<uint2*>(&tail[128 * k + 4 * lane]) = make_uint2(0u, 0u);
        else *reinterpret_cast<unsigned*>(&tail[64 * k + 2 * lane]) = 0u;
      }
#pragma unroll
      for (int j = 0; j < P; ++j) rc[j] = agg_f ? agg_v[j] : rc[j] + agg_v[j];
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
    for (int j = 0; j < P; ++j) a.carry_val[(int64_t)gw * P + j] = rc[j];
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
      float sum[P];
#pragma unroll
      for (int j = 0; j < P; ++j) sum[j] = 0.f;
      for (int kk = c; kk < nc && __ldcg(a.carry_row + kk) == r; ++kk)
#pragma unroll
        for (int j = 0; j < P; ++j) sum[j] += __ldcg(a.carry_val + (int64_t)kk * P + j);
      float* dst = a.Y + (int64_t)r * a.ldy;
#pragma unroll
      for (int j = 0; j < P; ++j) dst[j] = __ldcg(dst + j) + sum[j];
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

#ifndef LB_SPMM_ROTATE
#define LB_SPMM_ROTATE 0  // merge_spmm_cols_kernel: 1 = two rotated copies of the step (no register copies)
#endif
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

  PipeArgs pa;
  pa.off = a.off; pa.coords = a.coords; pa.rows = a.rows; pa.nnz = a.nnz;
  float rc = 0.f;  // partial of the open row, column cl (the same in every group)
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
        if (grp == 0) a.Y[(int64_t)i0 * a.ldy + cl] = rc;
        rc = 0.f;
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
        const float carry_in = grp == 0 ? rc : (lf ? lval : rc + lval);
        a.Y[(int64_t)(i0 - 1 + (int)first_rid) * a.ldy + cl] = carry_in + first_val;
      }
      rc = GF ? agg_v : rc + agg_v;
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
#if LB_SPMM_ROTATE
    while (true) {
      step(X0, X1);
      if (++st == nsteps) break;
      step(X1, X0);
      if (++st == nsteps) break;
    }
#else
    // one copy of the step (the code of a round is large: two rotated copies thrash the instruction
    // cache), the gathered round moved into place with register copies
    for (; st < nsteps; ++st) {
      step(X0, X1);
#pragma unroll
      for (int e = 0; e < EG; ++e) X0[e] = X1[e];
    }
#endif
  }

  if (grp == 0) {
    if (cl == 0) a.carry_row[gw] = i_last;
    a.carry_val[(int64_t)gw * P + cl] = rc;
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
      float sum = 0.f;
      for (int kk = c; kk < nc && __ldcg(a.carry_row + kk) == r; ++kk) sum += __ldcg(a.carry_val + (int64_t)kk * P + j);
      float* dst = a.Y + (int64_t)r * a.ldy + j;
      *dst = __ldcg(dst) + sum;
    }
    if (threadIdx.x == 0) *a.ticket = 0u;
  }
}

// ----------------------------------------------------------------------------- thread-mapped
// Listing 3: for row in tiles() (grid-stride, Listing 2), for nz in
// atoms(row): sum += values[nz] * x[indices[nz]]; y[row] = sum.  Four independent partial
// sums (reading R12) for ILP.
__global__ void __launch_bounds__(256) thread_mapped_kernel(int rows, const int* __restrict__ off,
                                                            const int* __restrict__ col,
                                                            const float* __restrict__ val,
                                                            const float* __restrict__ x, float* __restrict__ y) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    const int b = __ldg(off + r), e = __ldg(off + r + 1);
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    int k = b;
    for (; k + 4 <= e; k += 4) {
      s0 = fmaf(__ldg(val + k), ld_x(x + __ldg(col + k)), s0);
      s1 = fmaf(__ldg(val + k + 1), ld_x(x + __ldg(col + k + 1)), s1);
      s2 = fmaf(__ldg(val + k + 2), ld_x(x + __ldg(col + k + 2)), s2);
      s3 = fmaf(__ldg(val + k + 3), ld_x(x + __ldg(col + k + 3)), s3);
    }
    for (; k < e; ++k) s0 = fmaf(__ldg(val + k), ld_x(x + __ldg(col + k)), s0);
    y[r] = (s0 + s1) + (s2 + s3);
  }
}

// ----------------------------------------------------------------------------- group-mapped
// Alg.2 P:255-281 / P:1036-1041 with reading R8-R10: a group of G lanes takes G consecutive
// rows per round; lane l loads its row's atom count, the group builds the inclusive prefix
// sum, lanes stride the group's atom pool by G and find each atom's row with
// a binary search in the prefix sum (get_tile); products are summed per row with a
// warp segmented scan and accumulated in a per-warp, per-row shared-memory slot (no
// atomics, deterministic); y[row] = sum over the group's warps in fixed order.
template <int G>
__global__ void __launch_bounds__(256) group_mapped_kernel(int rows, const int* __restrict__ off,
                                                           const int* __restrict__ col,
                                                           const float* __restrict__ val,
                                                           const float* __restrict__ x, float* __restrict__ y) {
  constexpr int NT = 256;
  constexpr int kGroups = NT / G;
  constexpr int kWpg = G / 32;  // warps per group
  __shared__ int s_incl[kGroups][G];
  __shared__ int s_start[kGroups][G];
  __shared__ float s_acc[NT / 32][G];
  __shared__ int s_wsum[NT / 32];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = tid / G, gl = tid % G, wig = gl >> 5;  // group, lane in group, warp in group
  const int64_t n_groups = (int64_t)gridDim.x * kGroups;

  for (int64_t base = (blockIdx.x * (int64_t)kGroups + grp) * G; base < rows; base += n_groups * G) {
    // all groups of the CTA run the same number of rounds (uniform loop for __syncthreads)
    const int64_t r = base + gl;
    const int b = r < rows ? __ldg(off + r) : 0;
    const int cnt = r < rows ? __ldg(off + r + 1) - b : 0;
    int incl = warp_incl_scan_int(cnt, lane);
    if (kWpg > 1) {
      if (lane == 31) s_wsum[warp] = incl;
      __syncthreads();
      int add = 0;
      for (int w = 0; w < wig; ++w) add += s_wsum[grp * kWpg + w];
      incl += add;
    }
    s_incl[grp][gl] = incl;
    s_start[grp][gl] = b;
    for (int q = lane; q < G; q += 32) s_acc[warp][q] = 0.f;
    if (kWpg > 1) __syncthreads(); else __syncwarp();
    const int total = s_incl[grp][G - 1];

    // this warp takes atoms k = k0 + 32*wig + lane, k0 += G
    for (int k0 = 0; k0 < total; k0 += G) {
      const int k = k0 + 32 * wig + lane;
      const bool ok = k < total;
      int rl = 0;
      float p = 0.f;
      if (ok) {
        int lo = 0, hi = G - 1;  // first rl with incl[rl] > k
        while (lo < hi) {
          int mid = (lo + hi) >> 1;
          if (s_incl[grp][mid] > k) hi = mid; else lo = mid + 1;
        }
        rl = lo;
        const int excl = rl ? s_incl[grp][rl - 1] : 0;
        const int nz = s_start[grp][rl] + (k - excl);
        p = __ldg(val + nz) * ld_x(x + __ldg(col + nz));
      }
      const int prev = __shfl_up_sync(kFull, rl, 1);
      const int next = __shfl_down_sync(kFull, rl, 1);
      const bool next_ok = __shfl_down_sync(kFull, (int)ok, 1);
      bool head = lane == 0 || prev != rl;
      float v = p;
      warp_segscan_incl(head, v, lane);
      const bool tail = ok && (lane == 31 || !next_ok || next != rl);
      if (tail) s_acc[warp][rl] += v;
      __syncwarp();
    }
    if (kWpg > 1) __syncthreads(); else __syncwarp();
    if (r < rows) {
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < kWpg; ++w) s += s_acc[grp * kWpg + w][gl];
      y[r] = s;
    }
    if (kWpg > 1) __syncthreads(); else __syncwarp();
  }
}

// ----------------------------------------------------------------------------- warp-mapped
// Warp-level load balancing (P:1031-1034 [Sec. Warp- and block-level load balancing]): every warp
// takes an equal share of tiles (rows) -- a contiguous run of ceil(rows / warps) rows -- and
// processes them one at a time; the atoms of a row are processed in parallel by the 32 lanes, each
// striding by the warp size ("CSR-vector").  Lane l sums k = b+l, b+l+32, ... in order; the row
// sum is a fixed xor-shuffle tree over the lanes (deterministic).
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

__device__ __forceinline__ float row_dot_lanes(int b, int e, int lane, int stride, const int* __restrict__ col,
                                               const float* __restrict__ val, const float* __restrict__ x) {
  float s0 = 0.f, s1 = 0.f;
  int k = b + lane;
  for (; k + stride < e; k += 2 * stride) {
    s0 = fmaf(__ldg(val + k), ld_x(x + __ldg(col + k)), s0);
    s1 = fmaf(__ldg(val + k + stride), ld_x(x + __ldg(col + k + stride)), s1);
  }
  if (k < e) s0 = fmaf(__ldg(val + k), ld_x(x + __ldg(col + k)), s0);
  return s0 + s1;
}

__global__ void __launch_bounds__(256) warp_mapped_kernel(int rows, int rows_per_warp, const int* __restrict__ off,
                                                          const int* __restrict__ col, const float* __restrict__ val,
                                                          const float* __restrict__ x, float* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t r0 = w * rows_per_warp;
  const int64_t r1 = (r0 + rows_per_warp < rows ? r0 + rows_per_warp : (int64_t)rows);
  for (int64_t r = r0; r < r1; ++r) {
    const float s = warp_sum(row_dot_lanes(__ldg(off + r), __ldg(off + r + 1), lane, 32, col, val, x));
    if (lane == 0) y[r] = s;
  }
}

// ----------------------------------------------------------------------------- binning
// Three-bin schedule (Alg.4 P:341-397 [Sec. Binning and Reordering]; three kernels): rows
// with >= kBinCta nonzeros go to the CTA bin, >= kBinWarp to the warp bin, the rest to the thread
// bin.  The bins are built by a stable compaction (count per block of
// kBinRows rows -> one-block scan -> scatter), so each bin lists its rows in ascending order
// (reading R21; Alg.4's atomic bin_size++ leaves the order unspecified).  Layout of `ids`:
// [CTA bin | warp bin | thread bin], sizes in sizes[0..2].  The three processing kernels are
// persistent and read the bin sizes on the device, so the whole schedule needs no host sync.
constexpr int kBinCta = 256;   // block_size (threads per CTA of the CTA-bin kernel)
constexpr int kBinWarp = 32;   // warp_size
constexpr int kBinRows = 1024; // rows per compaction block (256 threads x 4)

__device__ __forceinline__ int bin_of(int n) { return n >= kBinCta ? 0 : n >= kBinWarp ? 1 : 2; }

// counts[bin * nb + blk] = rows of block blk in `bin`
__global__ void __launch_bounds__(256) bin_count_kernel(int rows, const int* __restrict__ off, int nb,
                                                        int* __restrict__ counts) {
  __shared__ int s_c[3];
  if (threadIdx.x < 3) s_c[threadIdx.x] = 0;
  __syncthreads();
  int c[3] = {0, 0, 0};
  const int64_t r0 = (int64_t)blockIdx.x * kBinRows;
  for (int i = threadIdx.x; i < kBinRows; i += 256) {
    const int64_t r = r0 + i;
    if (r < rows) {
      const int b = bin_of(__ldg(off + r + 1) - __ldg(off + r));
      c[0] += b == 0; c[1] += b == 1; c[2] += b == 2;
    }
  }
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    int v = c[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&s_c[q], v);
  }
  __syncthreads();
  if (threadIdx.x < 3) counts[threadIdx.x * nb + blockIdx.x] = s_c[threadIdx.x];
}

// exclusive scan of counts (in place, bin-major so that bin q's blocks follow bin q-1's: the
// result is each block's write offset into `ids`), sizes[q] = rows in bin q
__global__ void __launch_bounds__(1024) bin_scan_kernel(int nb, int* __restrict__ counts, int* __restrict__ sizes) {
  __shared__ int s_w[32];
  __shared__ int s_carry;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  const int n = 3 * nb;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int base = 0; base < n; base += 1024) {
    const int i = base + threadIdx.x;
    const int v = i < n ? counts[i] : 0;
    int incl = warp_incl_scan_int(v, lane);
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const int t = s_w[lane];
      s_w[lane] = warp_incl_scan_int(t, lane) - t;
    }
    __syncthreads();
    const int excl = s_carry + s_w[warp] + incl - v;
    if (i < n) counts[i] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    // sizes from the offsets of each bin's first block and the total
    const int o1 = nb > 0 ? counts[nb] : 0, o2 = nb > 0 ? counts[2 * nb] : 0;
    sizes[0] = o1;
    sizes[1] = o2 - o1;
    sizes[2] = s_carry - o2;
  }
}

// ids[offset of (bin, block) + rank of the row among the block's rows of that bin] = row
__global__ void __launch_bounds__(256) bin_scatter_kernel(int rows, const int* __restrict__ off, int nb,
                                                          const int* __restrict__ offsets, int* __restrict__ ids) {
  __shared__ int s_w[3][8];
  __shared__ int s_base[3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < 3) s_base[threadIdx.x] = offsets[threadIdx.x * nb + blockIdx.x];
  __syncthreads();
  // 4 rounds of 256 consecutive rows; within a round rows are ranked in thread order
  for (int rd = 0; rd < kBinRows / 256; ++rd) {
    const int64_t r = (int64_t)blockIdx.x * kBinRows + rd * 256 + threadIdx.x;
    const int b = r < rows ? bin_of(__ldg(off + r + 1) - __ldg(off + r)) : 3;
    int rank = 0;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const unsigned m = __ballot_sync(kFull, b == q);
      if (lane == 0) s_w[q][warp] = __popc(m);
      if (b == q) rank = __popc(m & ((1u << lane) - 1u));
    }
    __syncthreads();
    if (b < 3) {
      int before = 0;
      for (int w = 0; w < warp; ++w) before += s_w[b][w];
      ids[s_base[b] + before + rank] = (int)r;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
      int t = 0;
      for (int w = 0; w < 8; ++w) t += s_w[threadIdx.x][w];
      s_base[threadIdx.x] += t;
    }
    __syncthreads();
  }
}

// CTA bin: one CTA (256 threads) per row, threads stride the row by 256, fixed-order block sum
__global__ void __launch_bounds__(256) bin_cta_kernel(const int* __restrict__ ids, const int* __restrict__ sizes,
                                                      const int* __restrict__ off, const int* __restrict__ col,
                                                      const float* __restrict__ val, const float* __restrict__ x,
                                                      float* __restrict__ y) {
  __shared__ float s_w[8];
  const int n = __ldg(sizes + 0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const int r = __ldg(ids + i);
    const float v = warp_sum(row_dot_lanes(__ldg(off + r), __ldg(off + r + 1), threadIdx.x, 256, col, val, x));
    if (lane == 0) s_w[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) s += s_w[w];
      y[r] = s;
    }
    __syncthreads();
  }
}

// warp bin: one warp per row, lanes stride by 32
__global__ void __launch_bounds__(256) bin_warp_kernel(const int* __restrict__ ids, const int* __restrict__ sizes,
                                                       const int* __restrict__ off, const int* __restrict__ col,
                                                       const float* __restrict__ val, const float* __restrict__ x,
                                                       float* __restrict__ y) {
  const int n0 = __ldg(sizes + 0), n = __ldg(sizes + 1);
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n; i += nw) {
    const int r = __ldg(ids + n0 + i);
    const float s = warp_sum(row_dot_lanes(__ldg(off + r), __ldg(off + r + 1), lane, 32, col, val, x));
    if (lane == 0) y[r] = s;
  }
}

// thread bin: one thread per row, atoms summed sequentially (Alg.4 THREAD_BIN; reading R21 for
// its y[A.indices[k]] garble: the row's own y[row] is written)
__global__ void __launch_bounds__(256) bin_thread_kernel(const int* __restrict__ ids, const int* __restrict__ sizes,
                                                         const int* __restrict__ off, const int* __restrict__ col,
                                                         const float* __restrict__ val, const float* __restrict__ x,
                                                         float* __restrict__ y) {
  const int base = __ldg(sizes + 0) + __ldg(sizes + 1), n = __ldg(sizes + 2);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = __ldg(ids + base + i);
    const int b = __ldg(off + r), e = __ldg(off + r + 1);
    float s = 0.f;
    for (int k = b; k < e; ++k) s = fmaf(__ldg(val + k), ld_x(x + __ldg(col + k)), s);
    y[r] = s;
  }
}

}  // namespace lbk
