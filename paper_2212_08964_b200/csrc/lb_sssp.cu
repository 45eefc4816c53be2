// lb_sssp.cu -- single-source shortest paths on the load-balancing schedules (NEXT-4; Listing 5
// P:1076-1107).  C ABI in include/lb.h.
#include "k_sssp.cuh"
#include "lb_internal.h"

#include <algorithm>
#include <utility>

namespace lbi {
namespace {

// ----------------------------------------------------------------------------- SSSP (NEXT-4)
lb_status_t sssp_impl(lb_csr_s* A, int64_t source, lb_schedule_t sched, float* dist, stream_t s, int32_t* rounds_out) {
  if (!A) return fail(LB_ERR_INVALID_ARG, "null handle");
  if (A->rows != A->cols) return fail(LB_ERR_INVALID_ARG, "SSSP needs a square adjacency matrix (rows %lld, cols %lld)",
                                      (long long)A->rows, (long long)A->cols);
  if (A->rows == 0) { if (rounds_out) *rounds_out = 0; return LB_OK; }
  if (source < 0 || source >= A->rows) return fail(LB_ERR_INVALID_ARG, "source %lld out of range", (long long)source);
  if (!dist) return fail(LB_ERR_INVALID_ARG, "null dist");
  if (sched == LB_SCHED_AUTO || sched == LB_SCHED_NONZERO_SPLIT) sched = LB_SCHED_MERGE_PATH;
  if (sched == LB_SCHED_BLOCK_MAPPED) sched = LB_SCHED_GROUP_MAPPED;
  if (sched != LB_SCHED_MERGE_PATH && sched != LB_SCHED_THREAD_MAPPED && sched != LB_SCHED_GROUP_MAPPED)
    return fail(LB_ERR_INVALID_ARG, "unknown schedule id %d", (int)sched);
  const int n = (int)A->rows;
  const int nb_max = n / lbk::kScanChunk + 2;
  if (!A->sssp.mem) {
    const size_t ntc = (size_t)((n + A->nnz) / lbk::kSsspTile + 2);  // tile boundaries of the largest round
    const size_t bytes = 3 * align256((size_t)n * 4) + align256(((size_t)n + 1) * 4) + align256((size_t)nb_max * 4 + 4) +
                         align256(16) + align256(ntc * 4);
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) { cudaGetLastError(); return fail(LB_ERR_OOM, "SSSP workspace"); }
    char* q = static_cast<char*>(p);
    A->sssp.mem = p;
    A->sssp.q_a = reinterpret_cast<int*>(q); q += align256((size_t)n * 4);
    A->sssp.q_b = reinterpret_cast<int*>(q); q += align256((size_t)n * 4);
    A->sssp.stamp = reinterpret_cast<int*>(q); q += align256((size_t)n * 4);
    A->sssp.fo = reinterpret_cast<int*>(q); q += align256(((size_t)n + 1) * 4);
    A->sssp.bsum = reinterpret_cast<int*>(q); q += align256((size_t)nb_max * 4 + 4);
    A->sssp.counts = reinterpret_cast<int*>(q); q += align256(16);
    A->sssp.tc = reinterpret_cast<int*>(q);
  }
  const int sms = A->dev->sm_count;
  lbk::sssp_init_kernel<<<sms * 8, kNT, 0, s>>>(n, (int)source, dist, A->sssp.stamp, A->sssp.q_a, A->sssp.counts);
  LB_LAUNCHED();
  if (A->nnz > 0) {
    lbk::sssp_check_weights_kernel<<<sms * 8, kNT, 0, s>>>(A->nnz, A->val, A->sssp.counts + 2);
    LB_LAUNCHED();
  }
  int h[3];
  LB_CUDA(cudaMemcpyAsync(h, A->sssp.counts, sizeof h, cudaMemcpyDeviceToHost, s));
  LB_CUDA(cudaStreamSynchronize(s));
  if (h[2]) return fail(LB_ERR_INVALID_ARG, "negative (or NaN) edge weight");
  int F = 1, round = 0;
  int* qi = A->sssp.q_a;
  int* qo = A->sssp.q_b;
  while (F > 0) {
    LB_CUDA(cudaMemsetAsync(A->sssp.counts + 1, 0, sizeof(int), s));
    if (sched == LB_SCHED_THREAD_MAPPED) {
      lbk::sssp_thread_kernel<<<(F + kNT - 1) / kNT, kNT, 0, s>>>(F, qi, A->off, A->col, A->val, dist, A->sssp.stamp, round,
                                                                   qo, A->sssp.counts + 1);
      LB_LAUNCHED();
    } else if (sched == LB_SCHED_GROUP_MAPPED) {
      const int64_t warps = (F + 31) / 32;
      const int grid = (int)std::min<int64_t>((warps * 32 + kNT - 1) / kNT, (int64_t)sms * 16);
      lbk::sssp_warp_kernel<<<grid, kNT, 0, s>>>(F, qi, A->off, A->col, A->val, dist, A->sssp.stamp, round, qo,
                                                 A->sssp.counts + 1);
      LB_LAUNCHED();
    } else {
      const int nb = (F + lbk::kScanChunk - 1) / lbk::kScanChunk;
      lbk::frontier_deg_sum_kernel<<<nb, 256, 0, s>>>(F, qi, A->off, A->sssp.bsum);
      LB_LAUNCHED();
      lbk::frontier_bsum_scan_kernel<<<1, 1024, 0, s>>>(nb, A->sssp.bsum);
      LB_LAUNCHED();
      lbk::frontier_deg_scan_kernel<<<nb, 256, 0, s>>>(F, qi, A->off, A->sssp.bsum, nb, A->sssp.fo);
      LB_LAUNCHED();
      // the round's CTA tiles: boundaries in parallel (host-side tile count from F + E_f is not known
      // without a sync, so the boundary kernel covers the largest possible count and each tile kernel
      // CTA stops at F + E_f)
      const int T = (int)((F + A->nnz + lbk::kSsspTile - 1) / lbk::kSsspTile);
      lbk::sssp_tile_coords_kernel<<<(T + 1 + 255) / 256, 256, 0, s>>>(F, A->sssp.fo, T, A->sssp.tc);
      LB_LAUNCHED();
      const int grid = sms * 8;  // persistent over the round's CTA tiles
      lbk::sssp_merge_kernel<<<grid, kNT, 0, s>>>(F, qi, A->sssp.fo, A->off, A->col, A->val, dist, A->sssp.stamp, round, qo,
                                                  A->sssp.counts + 1, A->sssp.tc);
      LB_LAUNCHED();
    }
    LB_CUDA(cudaMemcpyAsync(&F, A->sssp.counts + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
    LB_CUDA(cudaStreamSynchronize(s));
    std::swap(qi, qo);
    ++round;
  }
  if (rounds_out) *rounds_out = round;
  return LB_OK;
}

}  // namespace
}  // namespace lbi

using namespace lbi;

extern "C" {

lb_status_t lb_sssp(lb_csr_t A, int64_t source, lb_schedule_t sched, float* d_dist, void* stream, int32_t* rounds_out) {
  LB_NVTX("lb_sssp");
  g_err.clear();
  return sssp_impl(A, source, sched, d_dist, S(stream), rounds_out);
}

}  // extern "C"
