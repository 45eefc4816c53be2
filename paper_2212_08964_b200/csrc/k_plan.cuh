// k_plan.cuh -- sm_100a device code (arXiv 2212.08964).  Citations "P:L" = PAPER.md line L.
// x-reuse plan build kernels (B200 extension).
#pragma once
#include "dev_common.cuh"

namespace lbk {

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

}  // namespace lbk
