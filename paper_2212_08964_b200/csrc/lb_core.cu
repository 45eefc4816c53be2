// lb_core.cu -- errors, device info, the CSR handle (a1: create / validate / destroy), the merge-path
// and nonzero-split partitions (a2) and the AUTO schedule rule.  C ABI in include/lb.h.
#include "k_partition.cuh"
#include "lb_internal.h"

#include <algorithm>
#include <climits>
#include <cstdarg>
#include <cstdio>
#include <mutex>

namespace lbi {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

lb_status_t fail(lb_status_t st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

namespace {
DeviceInfo g_dev[64];
std::mutex g_dev_mu;
}  // namespace

lb_status_t device_info(int dev, const DeviceInfo** out) {
  if (dev < 0 || dev >= 64) return fail(LB_ERR_INVALID_ARG, "device ordinal %d out of range", dev);
  std::lock_guard<std::mutex> g(g_dev_mu);
  DeviceInfo& d = g_dev[dev];
  if (d.sm_count == 0) {
    int sms = 0, l2 = 0;
    LB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    LB_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
    d.l2_bytes = l2;
    d.sm_count = sms;
  }
  *out = &d;
  return LB_OK;
}

size_t scratch_bytes(int64_t rows, int64_t nnz) {
  return align256((num_tiles(rows, nnz, kMinTile) + 1) * sizeof(int2)) + align256(kMaxCtas * sizeof(int)) +
         align256(kCarryVals * sizeof(float)) + align256(4 * sizeof(int)) + align256(sizeof(unsigned));
}

void carve_scratch(lb_csr_s* A, char* p) {
  A->coords = reinterpret_cast<int2*>(p);
  p += align256((num_tiles(A->rows, A->nnz, kMinTile) + 1) * sizeof(int2));
  A->carry_row = reinterpret_cast<int*>(p);
  p += align256(kMaxCtas * sizeof(int));
  A->carry_val = reinterpret_cast<float*>(p);
  p += align256(kCarryVals * sizeof(float));  // up to 32 values per carry (SpMM panels)
  A->flags = reinterpret_cast<int*>(p);
  p += align256(4 * sizeof(int));
  A->ticket = reinterpret_cast<unsigned*>(p);
}

// Default tile length from the matrix shape (measured on B200): matrices with
// short rows (< 8 nonzeros per row on average, e.g. stencils) run best on the short-row CTA-tile
// kernel (merge_rows_kernel) with L = 2040; longer / irregular rows on the warp-streamed kernel with
// L = 1016.
int auto_tile_length(int64_t rows, int64_t nnz) { return nnz < 8 * rows ? 2040 : 1016; }

lb_status_t check_shape(int64_t rows, int64_t cols, int64_t nnz) {
  if (rows < 0 || cols < 0 || nnz < 0) return fail(LB_ERR_INVALID_ARG, "negative size (rows=%lld cols=%lld nnz=%lld)",
                                                   (long long)rows, (long long)cols, (long long)nnz);
  if (rows + nnz > kMaxMergeItems || cols >= (int64_t)INT_MAX)
    return fail(LB_ERR_INVALID_ARG, "rows + nnz must be <= 2^31 - 2^16 - 1 and cols < 2^31 - 1 (int32 indices)");
  if (nnz > 0 && cols == 0) return fail(LB_ERR_INVALID_ARG, "nnz > 0 with cols == 0");
  return LB_OK;
}

lb_status_t init_handle(lb_csr_s* A, int64_t rows, int64_t cols, int64_t nnz, const int32_t* off, const int32_t* col,
                        const float* val) {
  A->rows = rows; A->cols = cols; A->nnz = nnz;
  A->off = off; A->col = col; A->val = val;
  LB_CUDA(cudaGetDevice(&A->device));
  lb_status_t st = device_info(A->device, &A->dev);
  if (st != LB_OK) return st;
  A->vec = (reinterpret_cast<uintptr_t>(col) % 16 == 0) && (reinterpret_cast<uintptr_t>(val) % 16 == 0);
  A->vec32 = (reinterpret_cast<uintptr_t>(col) % 32 == 0) && (reinterpret_cast<uintptr_t>(val) % 32 == 0);
  A->L = auto_tile_length(rows, nnz);
  return LB_OK;
}

namespace {

lb_status_t run_validate(lb_csr_s* A, stream_t s) {
  int init[4] = {0, INT_MAX, 0, INT_MAX};
  LB_CUDA(cudaMemcpyAsync(A->flags, init, sizeof init, cudaMemcpyHostToDevice, s));
  int64_t work = std::max<int64_t>(A->rows, A->nnz);
  int grid = (int)std::min<int64_t>(std::max<int64_t>(1, (work + kNT - 1) / kNT), (int64_t)A->dev->sm_count * 16);
  lbk::validate_kernel<<<grid, kNT, 0, s>>>((int)A->rows, (int)A->cols, (int)A->nnz, A->off, A->col, A->flags);
  LB_LAUNCHED();
  int got[4];
  LB_CUDA(cudaMemcpyAsync(got, A->flags, sizeof got, cudaMemcpyDeviceToHost, s));
  LB_CUDA(cudaStreamSynchronize(s));
  if (got[0]) return fail(LB_ERR_INVALID_CSR, "row_offsets[0] != 0");
  if (got[1] != INT_MAX) return fail(LB_ERR_INVALID_CSR, "row_offsets not monotone at row %d", got[1]);
  if (got[2]) return fail(LB_ERR_INVALID_CSR, "row_offsets[rows] != nnz (%lld)", (long long)A->nnz);
  if (got[3] != INT_MAX) return fail(LB_ERR_INVALID_CSR, "col_idx[%d] outside [0, %lld)", got[3], (long long)A->cols);
  return LB_OK;
}

}  // namespace

// Row offsets small enough (<= 1/4 of the L2) to keep resident across calls with evict_last loads: the
// next call's partition search then runs on L2 hits.
int offsets_l2_resident(const lb_csr_s* A) { return 4 * (A->rows + 1) <= (int64_t)A->dev->l2_bytes / 4 ? 1 : 0; }

lb_status_t launch_partition(const lb_csr_s* A, int64_t L, int2* coords, stream_t s) {
  const int64_t T = num_tiles(A->rows, A->nnz, L);
  const int64_t n = T + 1;
  if (n <= kWarpSearchMax) {  // latency-bound: 16 lanes per boundary, ~6 dependent steps
    constexpr int G = 16;
    const int grid = (int)((n * G + kNT - 1) / kNT);
    lbk::partition_group_kernel<G><<<grid, kNT, 0, s>>>((int)A->rows, (int)A->nnz, A->off, L, T, coords,
                                                        offsets_l2_resident(A));
    LB_LAUNCHED();
    return LB_OK;
  }
  const int grid = (int)((n + kNT - 1) / kNT);
  lbk::partition_kernel<<<grid, kNT, 0, s>>>((int)A->rows, (int)A->nnz, A->off, L, T, coords);
  LB_LAUNCHED();
  return LB_OK;
}

lb_status_t launch_partition_nz(const lb_csr_s* A, int64_t L, int2* coords, stream_t s) {
  const int64_t T = num_tiles_nz(A->nnz, L);
  const int grid = (int)((T + 1 + kNT - 1) / kNT);
  lbk::partition_nz_kernel<<<grid, kNT, 0, s>>>((int)A->rows, (int)A->nnz, A->off, L, T, coords);
  LB_LAUNCHED();
  return LB_OK;
}

lb_status_t launch_partition_xhot(const lb_csr_s* A, int64_t L, bool partition, const float* x, stream_t s) {
  const lb_plan_state& p = A->plan;
  const int64_t T = partition ? num_tiles(A->rows, A->nnz, L) : -1;
  const int warm_idx = p.compact ? 0 : p.warm_n;               // warm gather by index
  const int64_t nquad = p.compact ? (A->cols + 3) / 4 : 0;     // or by mask (compact plan)
  const int64_t n = T + 1 + p.hot_n + warm_idx + nquad;
  const int grid = (int)std::max<int64_t>(1, (n + kNT - 1) / kNT);
  lbk::partition_xhot_kernel<<<grid, kNT, 0, s>>>((int)A->rows, (int)A->nnz, A->off, L, T, A->coords, p.hot_cols,
                                                   p.hot_n, p.warm_cols, warm_idx, x, p.x_hot, p.x_warm, p.wmask,
                                                   p.wbase, nquad);
  LB_LAUNCHED();
  return LB_OK;
}

lb_status_t launch_clean_tiles(const lb_csr_s* A, int64_t T, int K, int span, int64_t step, int* d_out, stream_t s) {
  lbk::clean_tiles_kernel<<<1, 32, 0, s>>>(A->coords, A->off, T, K, span, step, d_out);
  LB_LAUNCHED();
  return LB_OK;
}

lb_status_t ensure_partition(lb_csr_s* A, bool force, bool with_plan_gathers, const float* x, stream_t s) {
  const bool repart = force || !A->coords_valid || A->coords_kind != 0 || A->coords_L != A->L;
  lb_status_t st;
  if (with_plan_gathers) st = launch_partition_xhot(A, A->L, repart, x, s);
  else st = repart ? launch_partition(A, A->L, A->coords, s) : LB_OK;
  if (st != LB_OK) return st;
  if (repart) {
    A->coords_valid = true;
    A->coords_L = A->L;
    A->coords_kind = 0;
  }
  return LB_OK;
}

// LB_SCHED_AUTO (reading R18): the paper's alpha/beta rule + a row-regularity test.
lb_status_t select_schedule(lb_csr_s* A, stream_t s, lb_schedule_t* out) {
  const int64_t alpha = 500, beta = 10000;
  if ((A->rows < alpha || A->cols < alpha) && A->nnz < beta) { *out = LB_SCHED_THREAD_MAPPED; return LB_OK; }
  if (A->rows == 0) { *out = LB_SCHED_MERGE_PATH; return LB_OK; }
  if (A->max_row < 0) {
    LB_CUDA(cudaMemsetAsync(A->flags, 0, sizeof(int), s));
    const int grid = (int)std::min<int64_t>((A->rows + kNT - 1) / kNT, (int64_t)A->dev->sm_count * 8);
    lbk::max_row_kernel<<<std::max(grid, 1), kNT, 0, s>>>((int)A->rows, A->off, A->flags);
    LB_LAUNCHED();
    int m = 0;
    LB_CUDA(cudaMemcpyAsync(&m, A->flags, sizeof(int), cudaMemcpyDeviceToHost, s));
    LB_CUDA(cudaStreamSynchronize(s));
    A->max_row = m;
  }
  const double mean = (double)A->nnz / (double)A->rows;
  const bool regular = A->max_row <= 2.0 * mean + 8.0 && mean <= 32.0;
  *out = regular ? LB_SCHED_THREAD_MAPPED : LB_SCHED_MERGE_PATH;
  return LB_OK;
}

}  // namespace lbi

using namespace lbi;

// ============================================================================ C ABI
extern "C" {

const char* lb_last_error(void) { return g_err.c_str(); }
uint64_t lb_launch_count(void) { return g_launches.load(); }
const char* lb_version(void) { return "liblb 0.2 (sm_100a)"; }

lb_status_t lb_select_schedule(lb_csr_t A, void* stream, lb_schedule_t* out) {
  g_err.clear();
  if (!A || !out) return fail(LB_ERR_INVALID_ARG, "null argument");
  return select_schedule(A, S(stream), out);
}

const char* lb_kernel_name(lb_csr_t A, lb_schedule_t sched) {
  thread_local char buf[96];
  if (sched == LB_SCHED_AUTO && A && A->max_row >= 0) select_schedule(A, nullptr, &sched);
  switch (sched) {
    case LB_SCHED_THREAD_MAPPED: return "thread_mapped_kernel";
    case LB_SCHED_GROUP_MAPPED: return "group_mapped_kernel<32>";
    case LB_SCHED_BLOCK_MAPPED: return "group_mapped_kernel<256>";
    case LB_SCHED_NONZERO_SPLIT: return "partition_nz_kernel + merge_stream_kernel<8,4,2,u32>";
    case LB_SCHED_WARP_MAPPED: return "warp_mapped_kernel";
    case LB_SCHED_BINNING: return "bin_{count,scan,scatter}_kernel + bin_{cta,warp,thread}_kernel";
    case LB_SCHED_MERGE_PATH: return A ? merge_kernel_name(A, buf, sizeof buf) : "";
    default: return "";
  }
}

lb_status_t lb_csr_create(int64_t rows, int64_t cols, int64_t nnz, const int32_t* d_row_offsets,
                          const int32_t* d_col_idx, const float* d_values, int32_t validate, void* stream,
                          lb_csr_t* out) {
  g_err.clear();
  if (!out) return fail(LB_ERR_INVALID_ARG, "null output handle pointer");
  *out = nullptr;
  lb_status_t st = check_shape(rows, cols, nnz);
  if (st != LB_OK) return st;
  if (!d_row_offsets) return fail(LB_ERR_INVALID_ARG, "null row_offsets");
  if (nnz > 0 && (!d_col_idx || !d_values)) return fail(LB_ERR_INVALID_ARG, "null col_idx or values with nnz > 0");
  lb_csr_s* A = new (std::nothrow) lb_csr_s();
  if (!A) return fail(LB_ERR_OOM, "host allocation failed");
  st = init_handle(A, rows, cols, nnz, d_row_offsets, d_col_idx, d_values);
  if (st != LB_OK) { delete A; return st; }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, scratch_bytes(rows, nnz));
  if (e != cudaSuccess) { delete A; return fail(LB_ERR_OOM, "cudaMalloc scratch: %s", cudaGetErrorString(e)); }
  carve_scratch(A, static_cast<char*>(p));
  e = cudaMemsetAsync(A->ticket, 0, sizeof(unsigned), S(stream));
  if (e != cudaSuccess) { cudaFree(p); delete A; return fail(LB_ERR_CUDA, "cudaMemsetAsync: %s", cudaGetErrorString(e)); }
  if (validate) {
    st = run_validate(A, S(stream));
    if (st != LB_OK) { cudaFree(p); delete A; return st; }
  }
  *out = A;
  return LB_OK;
}

lb_status_t lb_csr_destroy(lb_csr_t A) {
  if (!A) return LB_OK;
  destroy_multi_state(A);
  destroy_host_state(A);
  drop_plan(A);
  lb_csr_trace_phases(A, 0);
  if (A->owns_scratch && A->coords) cudaFree(A->coords);
  if (A->sssp.mem) cudaFree(A->sssp.mem);
  if (A->bins.mem) cudaFree(A->bins.mem);
  delete A;
  return LB_OK;
}

lb_status_t lb_csr_set_items_per_tile(lb_csr_t A, int32_t items_per_tile) {
  g_err.clear();
  if (!A) return fail(LB_ERR_INVALID_ARG, "null handle");
  int L = items_per_tile == 0 ? auto_tile_length(A->rows, A->nnz) : items_per_tile;
  if (l_index(L) < 0) return fail(LB_ERR_INVALID_ARG, "items_per_tile %d unsupported (504, 1016, 2040, 3064, 4088)", L);
  A->L = L;
  A->coords_valid = false;
  A->chunks.L = 0;  // chunk cuts belong to a tile length
  return LB_OK;
}

lb_status_t lb_partition_size(lb_csr_t A, int32_t items_per_tile, int64_t* n) {
  g_err.clear();
  if (!A || !n) return fail(LB_ERR_INVALID_ARG, "null argument");
  int64_t L = items_per_tile == 0 ? A->L : items_per_tile;
  if (L <= 0) return fail(LB_ERR_INVALID_ARG, "items_per_tile must be >= 1");
  *n = num_tiles(A->rows, A->nnz, L);
  return LB_OK;
}

lb_status_t lb_partition(lb_csr_t A, int32_t items_per_tile, int32_t* d_coords, void* stream) {
  LB_NVTX("lb_partition");
  g_err.clear();
  if (!A || !d_coords) return fail(LB_ERR_INVALID_ARG, "null argument");
  int64_t L = items_per_tile == 0 ? A->L : items_per_tile;
  if (L <= 0) return fail(LB_ERR_INVALID_ARG, "items_per_tile must be >= 1");
  return launch_partition(A, L, reinterpret_cast<int2*>(d_coords), S(stream));
}

lb_status_t lb_partition_nz(lb_csr_t A, int32_t items_per_tile, int32_t* d_coords, void* stream) {
  g_err.clear();
  if (!A || !d_coords) return fail(LB_ERR_INVALID_ARG, "null argument");
  const int64_t L = items_per_tile == 0 ? kNzL : items_per_tile;
  if (L <= 0) return fail(LB_ERR_INVALID_ARG, "items_per_tile must be >= 1");
  return launch_partition_nz(A, L, reinterpret_cast<int2*>(d_coords), S(stream));
}

}  // extern "C"
