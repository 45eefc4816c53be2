// lb_spmm.cu -- SpMM Y = A X on the merge-path tiles of SpMV (NEXT-2; Listing 4).
// C ABI in include/lb.h.
#include "k_spmm.cuh"
#include "lb_internal.h"

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>

namespace lbi {
namespace {

constexpr int kSpmmW = 8, kSpmmMinB = 2, kSpmmL = 1016;

// P columns per panel; E nonzeros per lane per round (P = 8 panels use E = 2 to fit the registers)
template <int P, int E = 4>
lb_status_t spmm_panel(lb_csr_s* A, const float* X, int64_t ldx, float* Y, int64_t ldy, stream_t s) {
  auto k = lbk::merge_spmm_kernel<kSpmmW, P, kSpmmMinB, E>;
  static int blocks_cache[64][3] = {{0}};
  int& blocks = blocks_cache[A->device][P == 8 ? 2 : P == 4];
  if (blocks == 0) {
    cudaFuncAttributes fa;
    LB_CUDA(cudaFuncGetAttributes(&fa, k));
    LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k, kSpmmW * 32, 0));
    const double need = (double)blocks * (fa.sharedSizeBytes + 1024);
    int pct = std::min(100, std::max(1, (int)(100.0 * need / (228.0 * 1024.0)) + 1));
    LB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
    LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k, kSpmmW * 32, 0));
    blocks = std::max(1, blocks);
  }
  const int T = (int)num_tiles(A->rows, A->nnz, kSpmmL);
  // carry_val holds kCarryVals floats: P values per warp
  const int warps_max = std::min(A->dev->sm_count * blocks * kSpmmW, std::min(kMaxCtas, kCarryVals / P));
  const int tpw = (T + warps_max - 1) / warps_max;
  const int warps = (T + tpw - 1) / tpw;
  const int grid = (warps + kSpmmW - 1) / kSpmmW;
  lbk::SpmmArgs a;
  a.off = A->off; a.col = A->col; a.val = A->val; a.X = X; a.Y = Y; a.ldx = ldx; a.ldy = ldy;
  a.coords = A->coords; a.rows = (int)A->rows; a.nnz = (int)A->nnz; a.num_tiles = T; a.tiles_per_warp = tpw;
  a.carry_row = A->carry_row; a.carry_val = A->carry_val; a.ticket = A->ticket; a.vec = A->vec ? 1 : 0;
  k<<<grid, kSpmmW * 32, 0, s>>>(a);
  LB_LAUNCHED();
  return LB_OK;
}

// lanes-over-columns SpMM panel of P = 16/32 columns (merge_spmm_cols_kernel): one CTA of 16 warps per SM
constexpr int kSpmmColsW = 16;
template <int P>
lb_status_t spmm_cols_panel(lb_csr_s* A, const float* X, int64_t ldx, float* Y, int64_t ldy, stream_t s) {
  auto k = lbk::merge_spmm_cols_kernel<kSpmmColsW, 4, P>;
  constexpr int dyn = lbk::spmm_cols_dyn_bytes(kSpmmColsW, P);
  static int blocks_cache[64][3] = {{0}};
  int& blocks = blocks_cache[A->device][P == 8 ? 0 : P == 16 ? 1 : 2];
  if (blocks == 0) {
    cudaFuncAttributes fa;
    LB_CUDA(cudaFuncGetAttributes(&fa, k));
    LB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
    LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k, kSpmmColsW * 32, dyn));
    const double need = (double)blocks * (fa.sharedSizeBytes + dyn + 1024);
    int pct = std::min(100, std::max(1, (int)(100.0 * need / (228.0 * 1024.0)) + 1));
    LB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
    LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k, kSpmmColsW * 32, dyn));
    if (blocks < 1) return fail(LB_ERR_UNSUPPORTED, "SpMM column-panel kernel does not fit");
  }
  const int T = (int)num_tiles(A->rows, A->nnz, kSpmmL);
  const int warps_max = std::min(A->dev->sm_count * blocks * kSpmmColsW, std::min(kMaxCtas, kCarryVals / P));
  const int tpw = (T + warps_max - 1) / warps_max;
  const int warps = (T + tpw - 1) / tpw;
  const int grid = (warps + kSpmmColsW - 1) / kSpmmColsW;
  lbk::SpmmArgs a;
  a.off = A->off; a.col = A->col; a.val = A->val; a.X = X; a.Y = Y; a.ldx = ldx; a.ldy = ldy;
  a.coords = A->coords; a.rows = (int)A->rows; a.nnz = (int)A->nnz; a.num_tiles = T; a.tiles_per_warp = tpw;
  a.carry_row = A->carry_row; a.carry_val = A->carry_val; a.ticket = A->ticket; a.vec = 1;
  k<<<grid, kSpmmColsW * 32, dyn, s>>>(a);
  LB_LAUNCHED();
  return LB_OK;
}

// LB_SPMM=lanes (tests and comparison runs only) forces the lanes-over-nonzeros kernel for every panel
#ifndef LB_SPMM_COLS_MIN
#define LB_SPMM_COLS_MIN 16  // narrowest panel the lanes-over-columns kernel takes (8 or 16)
#endif

int spmm_mode() {
  const char* env = getenv("LB_SPMM");
  return env && strcmp(env, "lanes") == 0 ? 1 : 0;
}

lb_status_t spmm_impl(lb_csr_s* A, int64_t n, const float* X, int64_t ldx, float* Y, int64_t ldy, stream_t s) {
  if (!A) return fail(LB_ERR_INVALID_ARG, "null handle");
  if (n < 0 || ldx < n || ldy < n) return fail(LB_ERR_INVALID_ARG, "need n >= 0, ldx >= n, ldy >= n");
  if (A->rows == 0 || n == 0) return LB_OK;
  if (!Y || (!X && A->nnz > 0)) return fail(LB_ERR_INVALID_ARG, "null X or Y");
  if ((const void*)X == (const void*)Y) return fail(LB_ERR_INVALID_ARG, "X and Y must not alias");
  lb_status_t st;
  if (!A->coords_valid || A->coords_kind != 0 || A->coords_L != kSpmmL) {
    if ((st = launch_partition(A, kSpmmL, A->coords, s)) != LB_OK) return st;
    A->coords_valid = true;
    A->coords_L = kSpmmL;
    A->coords_kind = 0;
  }
  const int mode = spmm_mode();
  const bool cols_ok = A->vec32 && ldy % 4 == 0 && ldx <= INT32_MAX && ldy <= INT32_MAX && mode != 1;
  for (int64_t c0 = 0; c0 < n;) {
    // lanes over columns: panels of 32 / 16 columns (Y rows 16-byte aligned for the zero-row stores);
    // measured against the lanes-over-nonzeros kernel (tools/bench_spmm.py,
    // profiles/r01_spmm_cols_vs_lanes.jsonl): 1.3-1.65x at n = 16 and 1.7-2.1x at n = 32 on C3/C4/C5,
    // but slower at n = 8 (0.7-0.83x), so 8..15 remaining columns take the 8-column panel below
    if (cols_ok && n - c0 >= LB_SPMM_COLS_MIN && reinterpret_cast<uintptr_t>(Y + c0) % 16 == 0) {
      const int64_t left = n - c0;
      const int P = left >= 32 ? 32 : left >= 16 ? 16 : 8;
      st = P == 32 ? spmm_cols_panel<32>(A, X + c0, ldx, Y + c0, ldy, s)
         : P == 16 ? spmm_cols_panel<16>(A, X + c0, ldx, Y + c0, ldy, s)
                   : spmm_cols_panel<8>(A, X + c0, ldx, Y + c0, ldy, s);
      if (st != LB_OK) return st;
      c0 += P;
      continue;
    }
    // 8-column panels gather one 32-byte sector per nonzero (X rows 32-byte aligned)
    const bool oct = n - c0 >= 8 && ldx % 8 == 0 && ldy % 4 == 0 &&
                     reinterpret_cast<uintptr_t>(X + c0) % 32 == 0 && reinterpret_cast<uintptr_t>(Y + c0) % 16 == 0;
    const bool quad = n - c0 >= 4 && ldx % 4 == 0 && ldy % 4 == 0 &&
                      reinterpret_cast<uintptr_t>(X + c0) % 16 == 0 && reinterpret_cast<uintptr_t>(Y + c0) % 16 == 0;
    if (oct) {
      if ((st = spmm_panel<8, 2>(A, X + c0, ldx, Y + c0, ldy, s)) != LB_OK) return st;
      c0 += 8;
    } else if (quad) {
      if ((st = spmm_panel<4>(A, X + c0, ldx, Y + c0, ldy, s)) != LB_OK) return st;
      c0 += 4;
    } else {
      if ((st = spmm_panel<1>(A, X + c0, ldx, Y + c0, ldy, s)) != LB_OK) return st;
      c0 += 1;
    }
  }
  return LB_OK;
}

}  // namespace
}  // namespace lbi

using namespace lbi;

extern "C" {

lb_status_t lb_spmm(lb_csr_t A, int64_t n, const float* d_X, int64_t ldx, float* d_Y, int64_t ldy, void* stream) {
  LB_NVTX("lb_spmm");
  g_err.clear();
  return spmm_impl(A, n, d_X, ldx, d_Y, ldy, S(stream));
}

}  // extern "C"
