// k_partition.cuh -- sm_100a device code (arXiv 2212.08964).  Citations "P:L" = PAPER.md line L.
// a1 validation, a2 merge-path / nonzero-split partitions, the x-reuse plan's per-call gathers.
#pragma once
#include "dev_common.cuh"

namespace lbk {

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

// The same search by a group of G lanes per boundary, (G+1)-ary: each step the G lanes test G evenly
// spaced rows of the bracket at once (one load each, independent) and a ballot of the monotone
// predicate k + off[k+1] < d narrows the bracket ~(G+1)x; the last <= G candidates are tested
// directly.  ~6 dependent steps instead of ~22 for 4M rows: a partition of few boundaries is
// latency-bound (every dependent step is an L2 or DRAM round trip), so this costs fewer microseconds
// at G times the loads.  G = 16 keeps 32K boundaries within one wave of resident warps.  Same result
// as merge_path_search (the count of true predicates).
template <int G>
__device__ __forceinline__ int2 merge_path_search_group(int rows, int nnz, const int* __restrict__ off, int64_t t,
                                                        int64_t L, int g, unsigned gmask, int gbase, uint64_t pol) {
  const int64_t total = (int64_t)rows + nnz;
  const int64_t d = t * L < total ? t * L : total;
  int lo = (int)(d - nnz > 0 ? d - nnz : 0);
  int hi = (int)(d < rows ? d : rows);  // the answer i lies in [lo, hi]
  while (hi - lo > G) {
    const int k = lo + (int)(((int64_t)(hi - lo) * (g + 1)) / (G + 1));  // strictly increasing in g
    const bool p = (int64_t)k + ld_off(off + k + 1, pol) < d;
    const int c = __popc(__ballot_sync(gmask, p) & gmask);  // p holds exactly on lanes 0 .. c-1
    const int klo = __shfl_sync(gmask, k, gbase + (c > 0 ? c - 1 : 0));
    const int khi = __shfl_sync(gmask, k, gbase + (c < G ? c : G - 1));
    if (c > 0) lo = klo + 1;
    if (c < G) hi = khi;
  }
  const int k = lo + g;
  const bool p = k < hi && (int64_t)k + ld_off(off + k + 1, pol) < d;
  const int i = lo + __popc(__ballot_sync(gmask, p) & gmask);
  return make_int2(i, (int)(d - i));
}

template <int G>
__global__ void partition_group_kernel(int rows, int nnz, const int* __restrict__ off, int64_t L, int64_t T,
                                       int2* __restrict__ coords, int off_keep) {
  static_assert(G == 8 || G == 16 || G == 32, "group size");
  asm volatile("griddepcontrol.launch_dependents;");
  const int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  if (t > T) return;  // group-uniform
  const int lane = threadIdx.x & 31, g = lane % G, gbase = lane - g;
  const unsigned gmask = (G == 32 ? kFull : ((1u << G) - 1u)) << gbase;
  const uint64_t pol = off_keep ? policy_evict_last() : policy_evict_first();
  const int2 c = merge_path_search_group<G>(rows, nnz, off, t, L, g, gmask, gbase, pol);
  if (g == 0) coords[t] = c;
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

}  // namespace lbk
