// k_sssp.cuh -- sm_100a device code (arXiv 2212.08964).  Citations "P:L" = PAPER.md line L.
// SSSP frontier rounds (NEXT-4, Listing 5).
#pragma once
#include "dev_common.cuh"

namespace lbk {

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

}  // namespace lbk
