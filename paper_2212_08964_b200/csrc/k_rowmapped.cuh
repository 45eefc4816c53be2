// k_rowmapped.cuh -- sm_100a device code (arXiv 2212.08964).  Citations "P:L" = PAPER.md line L.
// Row-granular schedules: thread-mapped (a5), group-mapped (a6), warp-mapped and binning (NEXT-3).
#pragma once
#include "dev_common.cuh"

namespace lbk {

// ----------------------------------------------------------------------------- thread-mapped
// Listing 3: for row in tiles() (grid-stride, Listing 2), for nz in
// atoms(row): sum += values[nz] * x[indices[nz]]; y[row] = sum.  Four independent partial
// sums (reading R12) for ILP over chunks of kRowChunk atoms; chunk sums are accumulated with 2Sum
// (csum_add), so a row of 1e6 same-sign atoms keeps ~1e-6 relative error.  A row of <= kRowChunk
// atoms is one chunk: exactly the plain four-partial sum.
constexpr int kRowChunk = 64;
__global__ void __launch_bounds__(256) thread_mapped_kernel(int rows, const int* __restrict__ off,
                                                            const int* __restrict__ col,
                                                            const float* __restrict__ val,
                                                            const float* __restrict__ x, float* __restrict__ y) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    const int b = __ldg(off + r), e = __ldg(off + r + 1);
    float S = 0.f, C = 0.f;
    int k = b;
    do {
      const int ce = min(e, k + kRowChunk);
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
      for (; k + 4 <= ce; k += 4) {
        s0 = fmaf(__ldg(val + k), ld_x(x + __ldg(col + k)), s0);
        s1 = fmaf(__ldg(val + k + 1), ld_x(x + __ldg(col + k + 1)), s1);
        s2 = fmaf(__ldg(val + k + 2), ld_x(x + __ldg(col + k + 2)), s2);
        s3 = fmaf(__ldg(val + k + 3), ld_x(x + __ldg(col + k + 3)), s3);
      }
      for (; k < ce; ++k) s0 = fmaf(__ldg(val + k), ld_x(x + __ldg(col + k)), s0);
      csum_add(S, C, (s0 + s1) + (s2 + s3));
    } while (k < e);
    y[r] = S + C;
  }
}

// ----------------------------------------------------------------------------- group-mapped
// Alg.2 P:255-281 / P:1036-1041 with reading R8-R10: a group of G lanes takes G consecutive
// rows per round; lane l loads its row's atom count, the group builds the inclusive prefix
// sum, lanes stride the group's atom pool by G and find each atom's row with
// a binary search in the prefix sum (get_tile); products are summed per row with a
// warp segmented scan and accumulated in a per-warp, per-row shared-memory slot (no
// atomics, deterministic; compensated: a slot is a 2Sum pair, so a giant row that takes thousands
// of rounds keeps ~2u relative error); y[row] = sum over the group's warps in fixed order.
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
  __shared__ float s_cmp[NT / 32][G];
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
    for (int q = lane; q < G; q += 32) s_acc[warp][q] = s_cmp[warp][q] = 0.f;
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
      if (tail) {
        float sa = s_acc[warp][rl], sc = s_cmp[warp][rl];
        csum_add(sa, sc, v);
        s_acc[warp][rl] = sa;
        s_cmp[warp][rl] = sc;
      }
      __syncwarp();
    }
    if (kWpg > 1) __syncthreads(); else __syncwarp();
    if (r < rows) {
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < kWpg; ++w) s += s_acc[grp * kWpg + w][gl] + s_cmp[grp * kWpg + w][gl];
      y[r] = s;
    }
    if (kWpg > 1) __syncthreads(); else __syncwarp();
  }
}

// ----------------------------------------------------------------------------- warp-mapped
// Warp-level load balancing (P:1031-1034 [Sec. Warp- and block-level load balancing]): every warp
// takes an equal share of tiles (rows) -- a contiguous run of ceil(rows / warps) rows -- and
// processes them one at a time; the atoms of a row are processed in parallel by the 32 lanes, each
// striding by the warp size ("CSR-vector").  Lane l sums k = b+l, b+l+stride, ... in order (two
// partials over chunks of 32 strides, chunk sums accumulated with 2Sum); the row sum is a fixed
// xor-shuffle tree over the lanes (deterministic).
__device__ __forceinline__ float row_dot_lanes(int b, int e, int lane, int stride, const int* __restrict__ col,
                                               const float* __restrict__ val, const float* __restrict__ x) {
  float S = 0.f, C = 0.f;
  int k = b + lane;
  while (k < e) {
    const int ke = min(e, k + 32 * stride);
    float s0 = 0.f, s1 = 0.f;
    for (; k + stride < ke; k += 2 * stride) {
      s0 = fmaf(__ldg(val + k), ld_x(x + __ldg(col + k)), s0);
      s1 = fmaf(__ldg(val + k + stride), ld_x(x + __ldg(col + k + stride)), s1);
    }
    if (k < ke) {
      s0 = fmaf(__ldg(val + k), ld_x(x + __ldg(col + k)), s0);
      k += stride;
    }
    csum_add(S, C, s0 + s1);
  }
  return S + C;
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
