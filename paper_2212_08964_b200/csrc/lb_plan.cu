// lb_plan.cu -- the x-reuse plan (lb_csr_plan_hot_x; B200 extension, not in the paper):
// a per-matrix data-placement decision made once, like the partition -- hot columns' x staged in
// shared memory, warm columns' x in a dense L2-resident copy -- with the y arithmetic untouched.
#include "k_plan.cuh"
#include "lb_internal.h"

#include <algorithm>
#include <climits>
#include <vector>

namespace lbi {

namespace {
constexpr int kHotSlotsDefault = 16384;  // 64 KB of shared memory per SM (best measured on C3)
constexpr int kHotSlotsMax = 45056;      // 176 KB
constexpr int64_t kWarmCompact = -2;     // lb_csr_plan_hot_x warm_cols: compact x (all referenced columns)
constexpr int64_t kWarmDefaultBytes = 48ll << 20;  // warm tier budget when x exceeds the L2
}  // namespace

void drop_plan(lb_csr_s* A) {
  ++A->plan.gen;
  A->chunks.L = 0;  // chunk cuts are cut for the plan's tile kernel: recompute after a plan change
  if (A->plan.mem) cudaFree(A->plan.mem);
  A->plan.mem = nullptr;
  A->plan.hcol = A->plan.hot_cols = A->plan.warm_cols = nullptr;
  A->plan.x_hot = A->plan.x_warm = nullptr;
  A->plan.hot_n = A->plan.hot_n4 = A->plan.warm_n = 0;
  A->plan.hot_nnz = A->plan.warm_nnz = 0;
  A->plan.compact = false;
  A->plan.wmask = nullptr;
  A->plan.wbase = nullptr;
}

// Degree level of the K-th most referenced column (candidates: deg >= 2), by successive equal-width
// histograms of deg over the candidate range.  found = false: fewer than K candidates.  Otherwise
// tau = the level, above = #{deg > tau} (< K), at = #{deg == tau} (above + at >= K).
struct Level {
  bool found = false;
  int64_t tau = 0, above = 0, at = 0;
};

lb_status_t find_level(lb_csr_s* A, const int* deg, int* bins, int64_t K, stream_t s, Level* out) {
  const int cols = (int)A->cols;
  int64_t lo = 2, hi = A->nnz + 1, above = 0;  // above = #columns with deg >= hi
  std::vector<int> hb(lbk::kDegBins);
  const int hgrid = std::max(1, std::min(A->dev->sm_count * 4, (cols + kNT - 1) / kNT));
  *out = Level();
  while (hi > lo) {
    const int64_t w = (hi - lo + lbk::kDegBins - 1) / lbk::kDegBins;
    LB_CUDA(cudaMemsetAsync(bins, 0, lbk::kDegBins * 4, s));
    lbk::degree_hist_kernel<<<hgrid, kNT, 0, s>>>(cols, deg, lo, hi, w, bins);
    LB_LAUNCHED();
    LB_CUDA(cudaMemcpyAsync(hb.data(), bins, lbk::kDegBins * 4, cudaMemcpyDeviceToHost, s));
    LB_CUDA(cudaStreamSynchronize(s));
    int64_t cum = above;
    int found = -1;
    for (int b = lbk::kDegBins - 1; b >= 0; --b) {
      if (lo + (int64_t)b * w >= hi) continue;
      if (cum + hb[b] >= K) { found = b; break; }
      cum += hb[b];
    }
    if (found < 0) return LB_OK;  // fewer than K candidates
    const int64_t nlo = lo + (int64_t)found * w, nhi = std::min(hi, nlo + w);
    above = cum;
    if (w == 1) {
      out->found = true;
      out->tau = nlo;
      out->above = above;
      out->at = hb[found];
      return LB_OK;
    }
    lo = nlo;
    hi = nhi;
  }
  return LB_OK;
}

// Builds the plan (see lb.h lb_csr_plan_hot_x).  Synchronises `s` a few times (setup call).
lb_status_t build_plan(lb_csr_s* A, int slots, int64_t warm, stream_t s) {
  drop_plan(A);
  const bool compact = warm == kWarmCompact;
  const int cols = (int)A->cols;
  const int64_t nnz = A->nnz;
  const int nblk = (int)((A->cols + lbk::kHotChunk - 1) / lbk::kHotChunk);
  // temporaries: deg/smap [cols], bins [kDegBins], block offsets [nblk], totals, degree sums
  const size_t tmp_bytes = align256((size_t)cols * 4) + align256(lbk::kDegBins * 4) + align256((size_t)nblk * 16) +
                           align256(16) + align256(16);
  char* tmp = nullptr;
  if (cudaMalloc(&tmp, tmp_bytes) != cudaSuccess) { cudaGetLastError(); return fail(LB_ERR_OOM, "plan temporaries"); }
  struct Free { char* p; ~Free() { cudaFree(p); } } free_tmp{tmp};
  int* deg = reinterpret_cast<int*>(tmp);
  int* bins = reinterpret_cast<int*>(tmp + align256((size_t)cols * 4));
  int4* blk = reinterpret_cast<int4*>(reinterpret_cast<char*>(bins) + align256(lbk::kDegBins * 4));
  int* totals = reinterpret_cast<int*>(reinterpret_cast<char*>(blk) + align256((size_t)nblk * 16));
  unsigned long long* d_sums = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(totals) + align256(16));

  const int sms = A->dev->sm_count;
  LB_CUDA(cudaMemsetAsync(deg, 0, (size_t)cols * 4, s));
  lbk::col_degree_kernel<<<sms * 8, kNT, 0, s>>>(nnz, A->col, deg);
  LB_LAUNCHED();

  // hot tier: the `slots` most referenced columns (ties at level tau1 in column order)
  Level l1;
  lb_status_t st = find_level(A, deg, bins, slots, s, &l1);
  if (st != LB_OK) return st;
  int t1_hi = 2, t1_tie = -1, b1 = 0;
  if (l1.found) { t1_hi = (int)(l1.tau + 1); t1_tie = (int)l1.tau; b1 = (int)(slots - l1.above); }
  // warm tier: whole degree levels below the hot set, at most `warm` more columns
  int t2 = INT_MAX, warm_on = 0;
  if (compact && l1.found) {
    t2 = 1;  // every referenced column below the hot set
    warm_on = 1;
  } else if (warm > 0 && l1.found) {
    Level l2;
    if ((st = find_level(A, deg, bins, (int64_t)slots + warm, s, &l2)) != LB_OK) return st;
    const int64_t tau2 = !l2.found ? 2 : (l2.above + l2.at == (int64_t)slots + warm ? l2.tau : l2.tau + 1);
    if (tau2 <= l1.tau) { t2 = (int)tau2; warm_on = 1; }
  }

  lbk::plan_count_kernel<<<nblk, 256, 0, s>>>(cols, deg, t1_hi, t1_tie, t2, blk);
  LB_LAUNCHED();
  lbk::plan_scan_kernel<<<1, 1024, 0, s>>>(nblk, b1, warm_on, blk, totals);
  LB_LAUNCHED();
  int tot[4];
  LB_CUDA(cudaMemcpyAsync(tot, totals, sizeof tot, cudaMemcpyDeviceToHost, s));
  LB_CUDA(cudaStreamSynchronize(s));
  const int n_above = tot[0];
  const int hot_n = n_above + std::min(b1, tot[1]);
  const int warm_n = warm_on ? tot[3] : 0;
  if (hot_n == 0) return LB_OK;  // nothing worth caching: no plan

  const int hot_n4 = (hot_n + 3) / 4;
  const bool cmp = compact && warm_n > 0;
  const size_t nwords = ((size_t)cols + 31) / 32;
  const size_t plan_bytes = align256((size_t)nnz * 4) + align256((size_t)hot_n * 4) + align256((size_t)hot_n4 * 16) +
                            2 * align256((size_t)std::max(warm_n, 1) * 4) + (cmp ? 2 * align256(nwords * 4) : 0);
  void* pm = nullptr;
  if (cudaMalloc(&pm, plan_bytes) != cudaSuccess) { cudaGetLastError(); return fail(LB_ERR_OOM, "plan (%zu bytes)", plan_bytes); }
  char* q = static_cast<char*>(pm);
  int32_t* hcol = reinterpret_cast<int32_t*>(q);
  q += align256((size_t)nnz * 4);
  int32_t* hot_cols = reinterpret_cast<int32_t*>(q);
  q += align256((size_t)hot_n * 4);
  float* x_hot = reinterpret_cast<float*>(q);
  q += align256((size_t)hot_n4 * 16);
  int32_t* warm_cols = reinterpret_cast<int32_t*>(q);
  q += align256((size_t)std::max(warm_n, 1) * 4);
  float* x_warm = reinterpret_cast<float*>(q);
  q += align256((size_t)std::max(warm_n, 1) * 4);
  unsigned* wmask = cmp ? reinterpret_cast<unsigned*>(q) : nullptr;
  int* wbase = cmp ? reinterpret_cast<int*>(q + align256(nwords * 4)) : nullptr;
  LB_CUDA(cudaMemsetAsync(x_hot, 0, (size_t)hot_n4 * 16, s));
  LB_CUDA(cudaMemsetAsync(d_sums, 0, 16, s));
  lbk::plan_assign_kernel<<<nblk, 256, 0, s>>>(cols, deg, t1_hi, t1_tie, t2, n_above, b1, hot_n, blk, hot_cols,
                                               warm_cols, d_sums);
  LB_LAUNCHED();
  lbk::plan_remap_kernel<<<sms * 8, kNT, 0, s>>>(nnz, cmp ? 0 : cols, hot_n, A->col, deg, hcol);
  LB_LAUNCHED();
  if (cmp) {
    LB_CUDA(cudaMemsetAsync(wmask, 0, nwords * 4, s));
    lbk::plan_mask_kernel<<<sms * 8, kNT, 0, s>>>(warm_cols, warm_n, wmask, wbase);
    LB_LAUNCHED();
  }
  unsigned long long sums[2] = {0, 0};
  LB_CUDA(cudaMemcpyAsync(sums, d_sums, sizeof sums, cudaMemcpyDeviceToHost, s));
  LB_CUDA(cudaStreamSynchronize(s));
  A->plan.mem = pm;
  A->plan.hcol = hcol;
  A->plan.hot_cols = hot_cols;
  A->plan.x_hot = x_hot;
  A->plan.hot_n = hot_n;
  A->plan.hot_n4 = hot_n4;
  A->plan.hot_nnz = (int64_t)sums[0];
  A->plan.warm_cols = warm_cols;
  A->plan.x_warm = x_warm;
  A->plan.warm_n = warm_n;
  A->plan.compact = cmp;
  A->plan.wmask = wmask;
  A->plan.wbase = wbase;
  A->plan.warm_nnz = (int64_t)sums[1];
  return LB_OK;
}

}  // namespace lbi

using namespace lbi;

extern "C" {

lb_status_t lb_csr_plan_hot_x(lb_csr_t A, int32_t slots, int64_t warm_cols, void* stream, int32_t* hot_cols_out,
                              int64_t* hot_nnz_out) {
  LB_NVTX("lb_csr_plan_hot_x");
  g_err.clear();
  if (!A) return fail(LB_ERR_INVALID_ARG, "null handle");
  if (slots < 0) {
    drop_plan(A);
  } else {
    const bool auto_plan = slots == 0;
    if (auto_plan && A->L != 1016 && A->L != 504) {  // no plan kernel at this tile length: nothing to gain
      drop_plan(A);
      if (hot_cols_out) *hot_cols_out = 0;
      if (hot_nnz_out) *hot_nnz_out = 0;
      return LB_OK;
    }
    if (slots == 0) slots = kHotSlotsDefault;
    if (slots > kHotSlotsMax) return fail(LB_ERR_INVALID_ARG, "slots %d > %d", slots, kHotSlotsMax);
    if (warm_cols < -2) return fail(LB_ERR_INVALID_ARG, "warm_cols %lld < -2", (long long)warm_cols);
    if (!A->vec32) return fail(LB_ERR_UNSUPPORTED, "x-reuse plan needs 32-byte aligned col_idx/values");
    if (warm_cols == -1) {  // auto: only when x is larger than the L2 (measured: C5 2.2x, C3 -10%)
      int l2 = 0;
      LB_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, A->device));
      warm_cols = 4 * A->cols > (int64_t)l2 ? std::min<int64_t>(A->cols, kWarmDefaultBytes / 4) : 0;
    }
    if (A->nnz == 0 || A->cols == 0) {
      drop_plan(A);
    } else {
      lb_status_t st = build_plan(A, slots, warm_cols, S(stream));
      if (st != LB_OK) { drop_plan(A); return st; }
      // auto: keep the plan only where it pays -- a warm tier (x larger than the L2) or
      // hot columns holding >= 0.5% of the stored entries (C2 stencil 0.4% at L = 1016: the plan's
      // one-CTA-per-SM kernel was 20% slower there; C4 0.57%: +4%)
      if (auto_plan && A->plan.warm_n == 0 && 200 * A->plan.hot_nnz < A->nnz) drop_plan(A);
    }
  }
  if (hot_cols_out) *hot_cols_out = A->plan.hot_n;
  if (hot_nnz_out) *hot_nnz_out = A->plan.hot_nnz;
  return LB_OK;
}

lb_status_t lb_csr_hot_plan(lb_csr_t A, int32_t* hot_n, int64_t* hot_nnz, int64_t* warm_n, int64_t* warm_nnz,
                            int32_t* d_hot_cols_out, int32_t* d_warm_cols_out, int32_t* d_col_out, void* stream) {
  g_err.clear();
  if (!A) return fail(LB_ERR_INVALID_ARG, "null handle");
  if (hot_n) *hot_n = A->plan.hot_n;
  if (hot_nnz) *hot_nnz = A->plan.hot_nnz;
  if (warm_n) *warm_n = A->plan.warm_n;
  if (warm_nnz) *warm_nnz = A->plan.warm_nnz;
  if (A->plan.hot_n > 0) {
    if (d_hot_cols_out)
      LB_CUDA(cudaMemcpyAsync(d_hot_cols_out, A->plan.hot_cols, (size_t)A->plan.hot_n * 4, cudaMemcpyDeviceToDevice, S(stream)));
    if (d_warm_cols_out && A->plan.warm_n > 0)
      LB_CUDA(cudaMemcpyAsync(d_warm_cols_out, A->plan.warm_cols, (size_t)A->plan.warm_n * 4, cudaMemcpyDeviceToDevice, S(stream)));
    if (d_col_out)
      LB_CUDA(cudaMemcpyAsync(d_col_out, A->plan.hcol, (size_t)A->nnz * 4, cudaMemcpyDeviceToDevice, S(stream)));
  }
  return LB_OK;
}

}  // extern "C"
