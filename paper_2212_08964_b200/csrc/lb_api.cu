// lb_api.cu -- C ABI of liblb.so (declared and documented in include/lb.h).
// Handle management, argument checking, launch configuration and the multi-GPU layer.
// All compute runs in the kernels of lb_kernels.cuh; there is no CPU fallback.
#include "lb.h"
#include "lb_kernels.cuh"

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

namespace {

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

#define LB_CUDA(call)                                                                         \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) return fail(LB_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

#define LB_LAUNCHED()                                                                                      \
  do {                                                                                                     \
    g_launches.fetch_add(1, std::memory_order_relaxed);                                                    \
    cudaError_t e_ = cudaGetLastError();                                                                   \
    if (e_ != cudaSuccess) return fail(LB_ERR_CUDA, "kernel launch (%s:%d): %s", __FILE__, __LINE__,        \
                                       cudaGetErrorString(e_));                                            \
  } while (0)

constexpr int kNT = 256;
// rows + nnz limit: int32 indices with 2^16 of headroom for the rounds / tiles that overshoot the last
// nonzero inside the kernels' int32 position arithmetic
constexpr int64_t kMaxMergeItems = (1ll << 31) - (1ll << 16) - 1;
constexpr int kMaxCtas = 8192;      // carry slots per handle (>= SMs x resident CTAs)
constexpr int kCarryVals = 32 * kMaxCtas;  // carry values per handle (SpMM: up to 32 per carry slot)
constexpr int kMinTile = 504;       // smallest supported L: sizes the partition cache

// Merge-path tile lengths.  The pipelined kernel runs NT threads x E nonzeros per tile, so a
// tile holds L = NT*E - 8 merge items (its 16-byte-aligned nonzero range spans <= L + 6).
constexpr int kNumL = 5;
constexpr int kTileL[kNumL] = {504, 1016, 2040, 3064, 4088};
constexpr int kPipeStages = 2;
inline int l_index(int L) {
  for (int i = 0; i < kNumL; ++i)
    if (kTileL[i] == L) return i;
  return -1;
}

using stream_t = cudaStream_t;
inline stream_t S(void* s) { return reinterpret_cast<stream_t>(s); }

typedef lb_status_t (*pipe_launch_fn)(lb_csr_s* A, const float* x, float* y, int grid_max, stream_t s);
typedef lb_status_t (*pipe_prepare_fn)(int* blocks_per_sm);

// One configuration of a merge-path tile kernel (kind 0: direct, kind 1: TMA-staged).
struct PipeVariant {
  int L, nt, e, minb, kind;  // kind 0: merge_direct_kernel, 1: merge_pipe_kernel, 2: merge_wide_kernel
  pipe_prepare_fn prepare;
  pipe_launch_fn launch;
};

template <int NT, int E, int MINB>
size_t pipe_smem() { return sizeof(typename lbk::PipeCfg<NT, E, kPipeStages>::Smem); }

template <int NT, int E, int MINB>
lb_status_t pipe_prepare(int* blocks) {
  auto k = lbk::merge_pipe_kernel<NT, E, kPipeStages, MINB>;
  LB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pipe_smem<NT, E, MINB>()));
  LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, k, NT, pipe_smem<NT, E, MINB>()));
  return LB_OK;
}

template <int NT, int E, int MINB>
lb_status_t pipe_launch(lb_csr_s* A, const float* x, float* y, int grid_max, stream_t s);

// Direct kernel: static smem only; after the occupancy query, ask for the smallest shared-memory
// carve-out that still fits that occupancy, leaving the rest of the 256 KB to L1 (gather MLP).
template <int NT, int MINB, bool XK>
lb_status_t direct_prepare(int* blocks) {
  auto k = lbk::merge_direct_kernel<NT, MINB, XK>;
  cudaFuncAttributes fa;
  LB_CUDA(cudaFuncGetAttributes(&fa, k));
  LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, k, NT, 0));
  const double need = (double)(*blocks) * (fa.sharedSizeBytes + 1024);
  int pct = (int)(100.0 * need / (228.0 * 1024.0)) + 1;
  pct = std::min(100, std::max(1, pct));
  LB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
  LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, k, NT, 0));
  return LB_OK;
}

template <int NT, int MINB, bool XK>
lb_status_t direct_launch(lb_csr_s* A, const float* x, float* y, int grid_max, stream_t s);

template <int NT, int E, int MINB>
lb_status_t wide_prepare(int* blocks) {
  auto k = lbk::merge_wide_kernel<NT, E, MINB>;
  cudaFuncAttributes fa;
  LB_CUDA(cudaFuncGetAttributes(&fa, k));
  LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, k, NT, 0));
  const double need = (double)(*blocks) * (fa.sharedSizeBytes + 1024);
  int pct = (int)(100.0 * need / (228.0 * 1024.0)) + 1;
  pct = std::min(100, std::max(1, pct));
  LB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
  LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, k, NT, 0));
  return LB_OK;
}
template <int NT, int E, int MINB>
lb_status_t wide_launch(lb_csr_s* A, const float* x, float* y, int grid_max, stream_t s);
#define LB_WIDE_VARIANT(NT, E, MINB) {NT * E - 8, NT, E, MINB, 2, wide_prepare<NT, E, MINB>, wide_launch<NT, E, MINB>}

template <int W, int R, int MINB, bool XK>
lb_status_t stream_prepare(int* blocks) {
  auto k = lbk::merge_stream_kernel<W, R, MINB, XK>;
  cudaFuncAttributes fa;
  LB_CUDA(cudaFuncGetAttributes(&fa, k));
  LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, k, W * 32, 0));
  const double need = (double)(*blocks) * (fa.sharedSizeBytes + 1024);
  int pct = (int)(100.0 * need / (228.0 * 1024.0)) + 1;
  pct = std::min(100, std::max(1, pct));
  LB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
  LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, k, W * 32, 0));
  return LB_OK;
}
template <int W, int R, int MINB, bool XK>
lb_status_t stream_launch(lb_csr_s* A, const float* x, float* y, int grid_max, stream_t s);
// warp-streamed tiles: L = 256*R - 8, W warps per CTA (nt = W*32, e = 8 nonzeros per lane per round)
#define LB_STREAM_VARIANT(W, R, MINB) \
  {256 * R - 8, W * 32, 8, MINB, 3, stream_prepare<W, R, MINB, false>, stream_launch<W, R, MINB, false>}
#define LB_STREAM_VARIANT_XK(W, R, MINB) \
  {256 * R - 8, W * 32, 8, MINB, 3, stream_prepare<W, R, MINB, true>, stream_launch<W, R, MINB, true>}

#define LB_DIRECT_VARIANT(NT, MINB, XK) \
  {NT * 4 - 8, NT, 4, MINB, 0, direct_prepare<NT, MINB, XK>, direct_launch<NT, MINB, XK>}
#define LB_PIPE_VARIANT(NT, E, MINB) {NT * E - 8, NT, E, MINB, 1, pipe_prepare<NT, E, MINB>, pipe_launch<NT, E, MINB>}
const PipeVariant kVariants[] = {
    LB_STREAM_VARIANT(8, 4, 2),        // 0  L=1016 default: warp-streamed (C3 R-MAT, C4 skewed: best measured)
    LB_WIDE_VARIANT(256, 8, 4),        // 1  L=2040 default: CTA tiles, 8 nonzeros/thread (C2 stencil: best)
    LB_WIDE_VARIANT(256, 16, 2),       // 2  L=4088 default
    LB_STREAM_VARIANT(4, 2, 4),        // 3  L=504  default
    LB_PIPE_VARIANT(256, 12, 2),       // 4  L=3064 default (TMA-staged)
    LB_PIPE_VARIANT(256, 4, 2),        // 5  L=1016 alternative: TMA bulk-copy staging of col/val/off
    LB_DIRECT_VARIANT(256, 2, false),  // 6  L=1016 alternative: 128-bit loads, 4 nonzeros per thread
    LB_DIRECT_VARIANT(128, 8, false),  // 7  L=504  alternative
    LB_DIRECT_VARIANT(128, 4, true),   // 8  L=504  alternative: x gathers with L2 evict_last
    LB_WIDE_VARIANT(128, 8, 8),        // 9  L=1016 alternative: CTA tiles, 8 nonzeros/thread
    LB_STREAM_VARIANT(4, 4, 4),        // 10 L=1016 alternative: warp-streamed, 4 warps/CTA
    LB_STREAM_VARIANT(4, 8, 4),        // 11 L=2040 alternative: warp-streamed
    LB_WIDE_VARIANT(64, 8, 16),        // 12 L=504  alternative
    LB_STREAM_VARIANT_XK(8, 4, 2),     // 13 L=1016 warp-streamed, x gathers with L2 evict_last
};
constexpr int kNumVariants = sizeof(kVariants) / sizeof(kVariants[0]);
// default variant per tile length (index into kVariants), chosen by measurement
constexpr int kDefaultVariant[kNumL] = {3, 0, 1, 4, 2};  // per kTileL entry (504, 1016, 2040, 3064, 4088)

struct DeviceInfo {
  int sm_count = 0;
  int fb_grid[kNumL] = {0};              // persistent grid of the fallback (unaligned) merge kernel per L
  int pipe_grid[kNumVariants] = {0};     // persistent grid of each pipelined variant
};

DeviceInfo g_dev[64];
std::mutex g_dev_mu;

template <int L>
size_t fb_smem() { return sizeof(typename lbk::MergeCfg<kNT, L, true>::Smem); }

template <int L>
lb_status_t fb_prepare(int* blocks) {
  auto k1 = lbk::merge_tile_kernel<kNT, L, true>;
  auto k2 = lbk::merge_tile_kernel<kNT, L, false>;
  int b1 = 0, b2 = 0;
  LB_CUDA(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fb_smem<L>()));
  LB_CUDA(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fb_smem<L>()));
  LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b1, k1, kNT, fb_smem<L>()));
  LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b2, k2, kNT, fb_smem<L>()));
  *blocks = std::min(b1, b2);
  return LB_OK;
}

lb_status_t device_info(int dev, const DeviceInfo** out) {
  if (dev < 0 || dev >= 64) return fail(LB_ERR_INVALID_ARG, "device ordinal %d out of range", dev);
  std::lock_guard<std::mutex> g(g_dev_mu);
  DeviceInfo& d = g_dev[dev];
  if (d.sm_count == 0) {
    int sms = 0;
    LB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    int fb[kNumL];
    lb_status_t st;
    if ((st = fb_prepare<504>(&fb[0])) != LB_OK) return st;
    if ((st = fb_prepare<1016>(&fb[1])) != LB_OK) return st;
    if ((st = fb_prepare<2040>(&fb[2])) != LB_OK) return st;
    if ((st = fb_prepare<3064>(&fb[3])) != LB_OK) return st;
    if ((st = fb_prepare<4088>(&fb[4])) != LB_OK) return st;
    for (int i = 0; i < kNumL; ++i) d.fb_grid[i] = sms * std::max(1, fb[i]);
    for (int v = 0; v < kNumVariants; ++v) {
      int b = 0;
      if ((st = kVariants[v].prepare(&b)) != LB_OK) return st;
      d.pipe_grid[v] = sms * std::max(1, b);
    }
    d.sm_count = sms;
  }
  *out = &d;
  return LB_OK;
}

// Development override: LB_PIPE_VARIANT=<index> forces a pipelined variant (its L must match).
int pipe_variant_for(int L) {
  const int li = l_index(L);
  const char* env = getenv("LB_PIPE_VARIANT");
  if (env) {
    const int v = atoi(env);
    if (v >= 0 && v < kNumVariants && kVariants[v].L == L) return v;
  }
  return kDefaultVariant[li];
}

}  // namespace

constexpr int kChunksMax = 8;  // LB_SPMV_CHUNKED: row chunks whose y copies overlap the next chunk

struct lb_csr_s {
  int64_t rows = 0, cols = 0, nnz = 0;
  const int32_t* off = nullptr;
  const int32_t* col = nullptr;
  const float* val = nullptr;
  int device = 0;
  const DeviceInfo* dev = nullptr;
  bool vec = true;            // col/val 16-byte aligned -> 128-bit loads
  bool pipe = true;           // off/col/val 16-byte aligned -> TMA-pipelined tile kernel
  bool vec32 = true;          // col/val 32-byte aligned -> 256-bit loads (wide tile kernel)
  int L = LB_DEFAULT_ITEMS_PER_TILE;
  bool coords_valid = false;
  int coords_L = 0;           // tile length the cached partition was computed for
  int coords_kind = 0;        // 0: merge-path, 1: nonzero-split
  bool owns_scratch = true;
  int2* coords = nullptr;     // partition cache [(T_max+1)]
  int* carry_row = nullptr;   // [kMaxCtas]
  float* carry_val = nullptr; // [kMaxCtas]
  int* flags = nullptr;       // [4] validation flags
  unsigned* ticket = nullptr; // [1] last-CTA ticket of the pipelined kernel (kept at 0 between launches)
  int max_row = -1;           // longest row (LB_SCHED_AUTO), -1 until computed
  // hot-column plan (lb_csr_plan_hot_x; one allocation at plan_mem)
  void* plan_mem = nullptr;
  int32_t* hcol = nullptr;     // [nnz] col_idx with hot entries replaced by ~slot
  int32_t* hot_cols = nullptr; // [hot_n] slot -> column
  float* x_hot = nullptr;      // [hot_n4 * 4] x of the hot columns, gathered every call
  int hot_n = 0;               // planned hot columns (0: no plan)
  int hot_n4 = 0;              // ceil(hot_n / 4)
  int64_t hot_nnz = 0;         // stored entries in hot columns
  int32_t* warm_cols = nullptr; // [warm_n] warm index -> column (ascending)
  float* x_warm = nullptr;      // [warm_n] x of the warm columns, gathered every call
  int warm_n = 0;
  int64_t warm_nnz = 0;
  bool compact = false;
  unsigned* wmask = nullptr;    // compact: [ceil(cols/32)] bit c = column c is warm
  int* wbase = nullptr;         // compact: [ceil(cols/32)] warm index of the word's first warm column         // warm_cols = -2: every referenced non-hot column is warm and the tile
                                // kernel gathers from the dense x_warm as its x (TIER 1 path)
  // SSSP workspace (lb_sssp; allocated on first use)
  void* sssp_mem = nullptr;
  float* hx_stage = nullptr;   // [cols + rows] device staging of lb_spmv_host_x (x, then y)
  // lb_spmv_host_x_async: two staging slots [x | y], an H2D and a D2H stream, per-slot events
  void* hp_mem = nullptr;
  float* hp_x[2] = {nullptr, nullptr};
  float* hp_y[2] = {nullptr, nullptr};
  cudaStream_t hp_h2d = nullptr, hp_d2h = nullptr;
  cudaEvent_t hp_xready[2] = {nullptr, nullptr};  // x of the slot is on the device
  cudaEvent_t hp_done[2] = {nullptr, nullptr};    // the slot's SpMV finished (x slot reusable)
  cudaEvent_t hp_out[2] = {nullptr, nullptr};     // the slot's y reached the host (y slot reusable)
  int hp_next = 0;
  // tile range of the next merge-path tile-kernel launch (LB_SPMV_CHUNKED; tr_t1 < 0: all tiles)
  int64_t tr_t0 = 0, tr_t1 = -1;
  // cached clean chunk boundaries for LB_SPMV_CHUNKED: tiles ch_t[0..ch_n], first rows ch_i[0..ch_n]
  int ch_L = 0, ch_n = 0;
  int64_t ch_t[kChunksMax + 1] = {}, ch_i[kChunksMax + 1] = {};
  cudaStream_t ch_d2h = nullptr;
  cudaEvent_t ch_ev[kChunksMax] = {};
  // lb_spmv_multi_ex(LB_SPMV_CHUNKED): every rank's local chunk cut rows [nranks][kChunksMax + 1]
  // (exchanged once per communicator and tile length), the exchange stream and its done event
  std::vector<int64_t> mc_rows;
  const void* mc_comm = nullptr;
  int mc_L = 0, mc_gen = -1;
  int plan_gen = 0;             // bumped by every plan build / drop (keys the exchanged cut table)
  cudaStream_t mc_stream = nullptr;
  cudaEvent_t mc_done = nullptr;
  int* q_a = nullptr;          // [rows] frontier lists (ping-pong)
  int* q_b = nullptr;
  int* stamp = nullptr;        // [rows] round of the last push
  int* fo = nullptr;           // [rows + 1] frontier degree prefix (merge-path)
  int* bsum = nullptr;         // [rows / kScanChunk + 2] scan block sums
  int* counts = nullptr;       // [4] frontier size, next size, negative-weight flag
  int* tc = nullptr;           // [(rows + nnz) / kSsspTile + 2] tile boundaries of a merge-path round
  // BINNING workspace (allocated on first use): [CTA | warp | thread] bin row ids, per-block counts
  void* bin_mem = nullptr;
  int* bin_ids = nullptr;      // [rows]
  int* bin_counts = nullptr;   // [3 * nb] counts, then write offsets
  int* bin_sizes = nullptr;    // [3]
};

namespace {

int64_t num_tiles(int64_t rows, int64_t nnz, int64_t L) { return (rows + nnz + L - 1) / L; }

size_t align256(size_t n) { return (n + 255) & ~size_t(255); }

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
// short rows (< 8 nonzeros per row on average, e.g. stencils) run best on the CTA-tile kernel
// with L = 2040; longer / irregular rows on the warp-streamed kernel with L = 1016.
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
  A->pipe = A->vec && (reinterpret_cast<uintptr_t>(off) % 16 == 0);
  A->vec32 = (reinterpret_cast<uintptr_t>(col) % 32 == 0) && (reinterpret_cast<uintptr_t>(val) % 32 == 0);
  A->L = auto_tile_length(rows, nnz);
  return LB_OK;
}

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

lb_status_t launch_partition(const lb_csr_s* A, int64_t L, int2* coords, stream_t s) {
  const int64_t T = num_tiles(A->rows, A->nnz, L);
  const int64_t n = T + 1;
  const int grid = (int)((n + kNT - 1) / kNT);
  lbk::partition_kernel<<<grid, kNT, 0, s>>>((int)A->rows, (int)A->nnz, A->off, L, T, coords);
  LB_LAUNCHED();
  return LB_OK;
}

// Phase hooks for lb_spmv_phase_times (events recorded between phases when non-null).
struct PhaseEvents {
  cudaEvent_t ev[4];
};

int64_t num_tiles_nz(int64_t nnz, int64_t L) { return std::max<int64_t>(1, (nnz + L - 1) / L); }

lb_status_t launch_partition_nz(const lb_csr_s* A, int64_t L, int2* coords, stream_t s) {
  const int64_t T = num_tiles_nz(A->nnz, L);
  const int grid = (int)((T + 1 + kNT - 1) / kNT);
  lbk::partition_nz_kernel<<<grid, kNT, 0, s>>>((int)A->rows, (int)A->nnz, A->off, L, T, coords);
  LB_LAUNCHED();
  return LB_OK;
}

template <int L, bool VEC>
lb_status_t launch_merge_tiles(lb_csr_s* A, const float* x, float* y, int grid_max, int* grid_used, stream_t s) {
  const int T = (int)num_tiles(A->rows, A->nnz, L);
  int grid = std::min(T, std::min(grid_max, kMaxCtas));
  const int tpc = (T + grid - 1) / grid;
  grid = (T + tpc - 1) / tpc;  // every CTA owns >= 1 tile
  lbk::MergeArgs a;
  a.off = A->off; a.col = A->col; a.val = A->val; a.x = x; a.y = y;
  a.coords = A->coords; a.rows = (int)A->rows; a.nnz = (int)A->nnz;
  a.num_tiles = T; a.tiles_per_cta = tpc;
  a.carry_row = A->carry_row; a.carry_val = A->carry_val;
  lbk::merge_tile_kernel<kNT, L, VEC><<<grid, kNT, fb_smem<L>(), s>>>(a);
  LB_LAUNCHED();
  *grid_used = grid;
  return LB_OK;
}

template <int NT, int E, int MINB>
lb_status_t pipe_launch(lb_csr_s* A, const float* x, float* y, int grid_max, stream_t s) {
  constexpr int L = NT * E - 8;
  const int T = (int)num_tiles(A->rows, A->nnz, L);
  int grid = std::min(T, std::min(grid_max, kMaxCtas));
  const int tpc = (T + grid - 1) / grid;
  grid = (T + tpc - 1) / tpc;
  lbk::PipeArgs a;
  a.off = A->off; a.col = A->col; a.val = A->val; a.x = x; a.y = y;
  a.coords = A->coords; a.rows = (int)A->rows; a.nnz = (int)A->nnz;
  a.num_tiles = T; a.tiles_per_cta = tpc;
  a.carry_row = A->carry_row; a.carry_val = A->carry_val; a.ticket = A->ticket;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = pipe_smem<NT, E, MINB>();
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL after lb_partition
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  LB_CUDA(cudaLaunchKernelEx(&cfg, lbk::merge_pipe_kernel<NT, E, kPipeStages, MINB>, a));
  LB_LAUNCHED();
  return LB_OK;
}

template <int NT, int MINB, bool XK>
lb_status_t direct_launch(lb_csr_s* A, const float* x, float* y, int grid_max, stream_t s) {
  constexpr int L = NT * 4 - 8;
  const int T = (int)num_tiles(A->rows, A->nnz, L);
  int grid = std::min(T, std::min(grid_max, kMaxCtas));
  const int tpc = (T + grid - 1) / grid;
  grid = (T + tpc - 1) / tpc;
  lbk::PipeArgs a;
  a.off = A->off; a.col = A->col; a.val = A->val; a.x = x; a.y = y;
  a.coords = A->coords; a.rows = (int)A->rows; a.nnz = (int)A->nnz;
  a.num_tiles = T; a.tiles_per_cta = tpc;
  a.carry_row = A->carry_row; a.carry_val = A->carry_val; a.ticket = A->ticket;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL after lb_partition
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  LB_CUDA(cudaLaunchKernelEx(&cfg, lbk::merge_direct_kernel<NT, MINB, XK>, a));
  LB_LAUNCHED();
  return LB_OK;
}

template <int NT, int E, int MINB>
lb_status_t wide_launch(lb_csr_s* A, const float* x, float* y, int grid_max, stream_t s) {
  constexpr int L = NT * E - 8;
  const int T = (int)num_tiles(A->rows, A->nnz, L);
  int grid = std::min(T, std::min(grid_max, kMaxCtas));
  const int tpc = (T + grid - 1) / grid;
  grid = (T + tpc - 1) / tpc;
  lbk::PipeArgs a;
  a.off = A->off; a.col = A->col; a.val = A->val; a.x = x; a.y = y;
  a.coords = A->coords; a.rows = (int)A->rows; a.nnz = (int)A->nnz;
  a.num_tiles = T; a.tiles_per_cta = tpc;
  a.carry_row = A->carry_row; a.carry_val = A->carry_val; a.ticket = A->ticket;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL after lb_partition
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  LB_CUDA(cudaLaunchKernelEx(&cfg, lbk::merge_wide_kernel<NT, E, MINB>, a));
  LB_LAUNCHED();
  return LB_OK;
}

template <int W, int R, int MINB, bool XK>
lb_status_t stream_launch(lb_csr_s* A, const float* x, float* y, int grid_max, stream_t s) {
  constexpr int L = 256 * R - 8;
  const int T = (int)num_tiles(A->rows, A->nnz, L);
  const int warps_max = std::min(grid_max * W, kMaxCtas);
  const int tpw = (T + warps_max - 1) / warps_max;   // tiles per warp
  const int warps = (T + tpw - 1) / tpw;
  const int grid = (warps + W - 1) / W;
  lbk::PipeArgs a;
  a.off = A->off; a.col = A->col; a.val = A->val; a.x = x; a.y = y;
  a.coords = A->coords; a.rows = (int)A->rows; a.nnz = (int)A->nnz;
  a.num_tiles = T; a.tiles_per_cta = tpw;
  a.carry_row = A->carry_row; a.carry_val = A->carry_val; a.ticket = A->ticket;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(W * 32);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL after lb_partition
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  LB_CUDA(cudaLaunchKernelEx(&cfg, lbk::merge_stream_kernel<W, R, MINB, XK>, a));
  LB_LAUNCHED();
  return LB_OK;
}

// nonzero-split: tiles of kNzL nonzeros on the warp-streamed processor with 32-bit row ids
constexpr int kNzL = 1016;
lb_status_t launch_nz_tiles(lb_csr_s* A, const float* x, float* y, stream_t s) {
  constexpr int W = 8, R = 4, MINB = 2;
  auto k = lbk::merge_stream_kernel<W, R, MINB, false, unsigned>;
  static int blocks_cache[64] = {0};
  int& blocks = blocks_cache[A->device];
  if (blocks == 0) {
    cudaFuncAttributes fa;
    LB_CUDA(cudaFuncGetAttributes(&fa, k));
    LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k, W * 32, 0));
    const double need = (double)blocks * (fa.sharedSizeBytes + 1024);
    int pct = std::min(100, std::max(1, (int)(100.0 * need / (228.0 * 1024.0)) + 1));
    LB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
    LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k, W * 32, 0));
    blocks = std::max(1, blocks);
  }
  const int T = (int)num_tiles_nz(A->nnz, kNzL);
  const int warps_max = std::min(A->dev->sm_count * blocks * W, kMaxCtas);
  const int tpw = (T + warps_max - 1) / warps_max;
  const int warps = (T + tpw - 1) / tpw;
  const int grid = (warps + W - 1) / W;
  lbk::PipeArgs a;
  a.off = A->off; a.col = A->col; a.val = A->val; a.x = x; a.y = y;
  a.coords = A->coords; a.rows = (int)A->rows; a.nnz = (int)A->nnz;
  a.num_tiles = T; a.tiles_per_cta = tpw;
  a.carry_row = A->carry_row; a.carry_val = A->carry_val; a.ticket = A->ticket;
  k<<<grid, W * 32, 0, s>>>(a);
  LB_LAUNCHED();
  return LB_OK;
}

// ----------------------------------------------------------------------------- hot-column plan
// Tile kernel with the plan: warp-streamed, one CTA of W warps per SM, x of the hot columns staged
// in dynamic shared memory.  W and the slot budget were chosen by measurement;
// LB_HOT_W overrides W (8, 16) for sweeps.
constexpr int kHotSlotsDefault = 16384;  // 64 KB of shared memory per SM (best measured on C3)
constexpr int kHotSlotsMax = 45056;      // 176 KB
constexpr int kHotDynMax = kHotSlotsMax * 4;
constexpr int64_t kWarmCompact = -2;  // lb_csr_plan_hot_x warm_cols: compact x (all referenced columns)
constexpr int64_t kWarmDefaultBytes = 48ll << 20;  // warm tier budget when x exceeds the L2

// Peer targets of the fused multi-GPU epilogue (lb_spmv_peers / lb_spmv_multi_fused): the other ranks'
// y, already offset to this rank's first row.
struct PeerArgs {
  float* y[lbk::kMaxPeers];
  int n = 0;
};

void set_peers(lbk::PipeArgs& a, const PeerArgs* pa) {
  a.npeers = pa ? pa->n : 0;
  for (int p = 0; p < lbk::kMaxPeers; ++p) a.peer_y[p] = pa && p < pa->n ? pa->y[p] : nullptr;
}

template <int W, int R, int TIER, bool PEERS = false>
lb_status_t hot_launch_wr(lb_csr_s* A, const float* x, float* y, stream_t s, const PeerArgs* pa = nullptr) {
  auto k = lbk::merge_stream_kernel<W, R, 1, false, unsigned short, TIER, PEERS>;
  static int conf_dyn[64] = {0};  // dynamic smem size the carve-out was set for, per device
  const int dyn = A->hot_n4 * 16;
  if (conf_dyn[A->device] != dyn) {
    cudaFuncAttributes fa;
    LB_CUDA(cudaFuncGetAttributes(&fa, k));
    LB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kHotDynMax));
    const double need = (double)fa.sharedSizeBytes + dyn + 1024.0;
    const int pct = std::min(100, std::max(1, (int)(100.0 * need / (228.0 * 1024.0)) + 1));
    LB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
    int blocks = 0;
    LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k, W * 32, dyn));
    if (blocks < 1) return fail(LB_ERR_UNSUPPORTED, "hot tile kernel does not fit with %d bytes of x_hot", dyn);
    conf_dyn[A->device] = dyn;
  }
  constexpr int L = 256 * R - 8;
  const bool ranged = A->tr_t1 >= 0;  // LB_SPMV_CHUNKED: tiles [tr_t0, tr_t1) only
  const int T = ranged ? (int)(A->tr_t1 - A->tr_t0) : (int)num_tiles(A->rows, A->nnz, L);
  if (T <= 0) return LB_OK;
  const int warps_max = std::min(A->dev->sm_count * W, kMaxCtas);
  const int tpw = (T + warps_max - 1) / warps_max;
  const int warps = (T + tpw - 1) / tpw;
  const int grid = (warps + W - 1) / W;
  lbk::PipeArgs a;
  a.off = A->off; a.col = A->hcol; a.val = A->val; a.x = x; a.y = y;
  a.coords = A->coords + (ranged ? A->tr_t0 : 0); a.rows = (int)A->rows; a.nnz = (int)A->nnz;
  a.num_tiles = T; a.tiles_per_cta = tpw;
  a.carry_row = A->carry_row; a.carry_val = A->carry_val; a.ticket = A->ticket;
  a.x_hot = A->x_hot; a.hot_n4 = A->hot_n4;
  a.x_warm = A->x_warm; a.cols = (int)A->cols;
  set_peers(a, pa);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(W * 32);
  cfg.dynamicSmemBytes = (size_t)dyn;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL after partition_xhot_kernel
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  LB_CUDA(cudaLaunchKernelEx(&cfg, k, a));
  LB_LAUNCHED();
  return LB_OK;
}

int hot_warps() {
  const char* env = getenv("LB_HOT_W");
  const int w = env ? atoi(env) : 16;
  return w == 8 ? 8 : 16;
}

bool hot_usable(const lb_csr_s* A) { return A->hot_n > 0 && A->vec32 && (A->L == 1016 || A->L == 504); }

template <int TIER>
lb_status_t hot_launch_t(lb_csr_s* A, const float* x, float* y, stream_t s, const PeerArgs* pa) {
  if (pa) {  // fused multi-GPU epilogue: 16 warps per CTA only
    if (A->L == 1016) return hot_launch_wr<16, 4, TIER, true>(A, x, y, s, pa);
    return hot_launch_wr<16, 2, TIER, true>(A, x, y, s, pa);
  }
  const bool w8 = hot_warps() == 8;
  if (A->L == 1016) return w8 ? hot_launch_wr<8, 4, TIER>(A, x, y, s) : hot_launch_wr<16, 4, TIER>(A, x, y, s);
  return w8 ? hot_launch_wr<8, 2, TIER>(A, x, y, s) : hot_launch_wr<16, 2, TIER>(A, x, y, s);
}

lb_status_t hot_launch(lb_csr_s* A, const float* x, float* y, stream_t s, const PeerArgs* pa = nullptr) {
  if (A->compact) return hot_launch_t<1>(A, A->x_warm, y, s, pa);
  return A->warm_n > 0 ? hot_launch_t<2>(A, x, y, s, pa) : hot_launch_t<1>(A, x, y, s, pa);
}

// Fused epilogue without a plan: the warp-streamed kernel at L = 1016 (8 warps, 2 CTAs per SM, the
// plain default) or L = 504, with peer stores.
template <int R>
lb_status_t peers_stream_launch(lb_csr_s* A, const float* x, float* y, stream_t s, const PeerArgs* pa) {
  constexpr int W = 8, MINB = 2;
  auto k = lbk::merge_stream_kernel<W, R, MINB, false, unsigned short, 0, true>;
  static int blocks_cache[64] = {0};
  int& blocks = blocks_cache[A->device];
  if (blocks == 0) {
    cudaFuncAttributes fa;
    LB_CUDA(cudaFuncGetAttributes(&fa, k));
    LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k, W * 32, 0));
    const double need = (double)blocks * (fa.sharedSizeBytes + 1024);
    const int pct = std::min(100, std::max(1, (int)(100.0 * need / (228.0 * 1024.0)) + 1));
    LB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
    LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k, W * 32, 0));
    blocks = std::max(1, blocks);
  }
  constexpr int L = 256 * R - 8;
  const int T = (int)num_tiles(A->rows, A->nnz, L);
  const int warps_max = std::min(A->dev->sm_count * blocks * W, kMaxCtas);
  const int tpw = (T + warps_max - 1) / warps_max;
  const int warps = (T + tpw - 1) / tpw;
  const int grid = (warps + W - 1) / W;
  lbk::PipeArgs a;
  a.off = A->off; a.col = A->col; a.val = A->val; a.x = x; a.y = y;
  a.coords = A->coords; a.rows = (int)A->rows; a.nnz = (int)A->nnz;
  a.num_tiles = T; a.tiles_per_cta = tpw;
  a.carry_row = A->carry_row; a.carry_val = A->carry_val; a.ticket = A->ticket;
  a.x_hot = nullptr; a.hot_n4 = 0; a.x_warm = nullptr; a.cols = (int)A->cols;
  set_peers(a, pa);
  k<<<grid, W * 32, 0, s>>>(a);
  LB_LAUNCHED();
  return LB_OK;
}

// stream+gather ceiling probe (lb_probe_stream_gather); TIER as in the tile kernel
template <int TIER>
lb_status_t probe_launch(lb_csr_s* A, const float* x, stream_t s) {
  auto k = lbk::probe_stream_gather_kernel<TIER>;
  const int dyn = TIER >= 1 ? A->hot_n4 * 16 : 0;
  static int conf_dyn[64] = {0};
  static int blocks_cache[64] = {0};  // 0: not configured yet on this device
  if (blocks_cache[A->device] == 0 || conf_dyn[A->device] != dyn) {
    LB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kHotDynMax));
    const int pct = TIER >= 1 ? std::min(100, (int)(100.0 * (dyn + 1024.0) / (228.0 * 1024.0)) + 1) : 0;
    LB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
    int blocks = 0;
    LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k, 512, dyn));
    // with a plan: one CTA (16 warps) per SM so x_hot is staged once per SM, as in the tile kernel
    blocks_cache[A->device] = TIER >= 1 ? 1 : std::max(1, blocks);
    conf_dyn[A->device] = dyn;
  }
  const int grid = A->dev->sm_count * blocks_cache[A->device];
  k<<<grid, 512, dyn, s>>>((int)A->nnz, TIER >= 1 ? A->hcol : A->col, A->val, x, A->x_hot, A->hot_n4, A->x_warm,
                           (int)A->cols, 0, nullptr);
  LB_LAUNCHED();
  return LB_OK;
}

// partition (T >= 0) and/or the x_hot gather in one launch
lb_status_t launch_partition_xhot(const lb_csr_s* A, int64_t L, bool partition, const float* x, stream_t s) {
  const int64_t T = partition ? num_tiles(A->rows, A->nnz, L) : -1;
  const int warm_idx = A->compact ? 0 : A->warm_n;               // warm gather by index
  const int64_t nquad = A->compact ? (A->cols + 3) / 4 : 0;      // or by mask (compact plan)
  const int64_t n = T + 1 + A->hot_n + warm_idx + nquad;
  const int grid = (int)std::max<int64_t>(1, (n + kNT - 1) / kNT);
  lbk::partition_xhot_kernel<<<grid, kNT, 0, s>>>((int)A->rows, (int)A->nnz, A->off, L, T, A->coords, A->hot_cols,
                                                   A->hot_n, A->warm_cols, warm_idx, x, A->x_hot, A->x_warm,
                                                   A->wmask, A->wbase, nquad);
  LB_LAUNCHED();
  return LB_OK;
}

void drop_plan(lb_csr_s* A) {
  ++A->plan_gen;
  if (A->plan_mem) cudaFree(A->plan_mem);
  A->plan_mem = nullptr;
  A->hcol = A->hot_cols = A->warm_cols = nullptr;
  A->x_hot = A->x_warm = nullptr;
  A->hot_n = A->hot_n4 = A->warm_n = 0;
  A->hot_nnz = A->warm_nnz = 0;
  A->compact = false;
  A->wmask = nullptr;
  A->wbase = nullptr;
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
  A->plan_mem = pm;
  A->hcol = hcol;
  A->hot_cols = hot_cols;
  A->x_hot = x_hot;
  A->hot_n = hot_n;
  A->hot_n4 = hot_n4;
  A->hot_nnz = (int64_t)sums[0];
  A->warm_cols = warm_cols;
  A->x_warm = x_warm;
  A->warm_n = warm_n;
  A->compact = cmp;
  A->wmask = wmask;
  A->wbase = wbase;
  A->warm_nnz = (int64_t)sums[1];
  return LB_OK;
}

template <int L>
lb_status_t launch_merge(lb_csr_s* A, const float* x, float* y, stream_t s, PhaseEvents* pe) {
  const int li = l_index(L);
  const int v = pipe_variant_for(L);
  const bool ok = kVariants[v].kind == 0 ? A->vec : kVariants[v].kind == 1 ? A->pipe : A->vec32;  // 2, 3: 256-bit
  if (ok) {
    lb_status_t st = kVariants[v].launch(A, x, y, A->dev->pipe_grid[v], s);
    if (st != LB_OK) return st;
    if (pe) { LB_CUDA(cudaEventRecord(pe->ev[2], s)); LB_CUDA(cudaEventRecord(pe->ev[3], s)); }
    return LB_OK;
  }
  int grid = 0;
  lb_status_t st = A->vec ? launch_merge_tiles<L, true>(A, x, y, A->dev->fb_grid[li], &grid, s)
                          : launch_merge_tiles<L, false>(A, x, y, A->dev->fb_grid[li], &grid, s);
  if (st != LB_OK) return st;
  if (pe) LB_CUDA(cudaEventRecord(pe->ev[2], s));
  lbk::fixup_kernel<<<(grid + kNT - 1) / kNT, kNT, 0, s>>>((int)A->rows, grid, A->carry_row, A->carry_val, y);
  LB_LAUNCHED();
  if (pe) LB_CUDA(cudaEventRecord(pe->ev[3], s));
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

constexpr int kWarpRows = 4;  // WARP_MAPPED: rows per warp

// BINNING (Alg.4): build the three bins on the device (stable compaction; no host sync)
lb_status_t launch_bins(lb_csr_s* A, stream_t s) {
  const int nb = (int)((A->rows + lbk::kBinRows - 1) / lbk::kBinRows);
  if (!A->bin_mem) {
    const size_t bytes = align256((size_t)A->rows * 4) + align256((size_t)3 * nb * 4) + align256(16);
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) { cudaGetLastError(); return fail(LB_ERR_OOM, "binning workspace"); }
    char* q = static_cast<char*>(p);
    A->bin_mem = p;
    A->bin_ids = reinterpret_cast<int*>(q); q += align256((size_t)A->rows * 4);
    A->bin_counts = reinterpret_cast<int*>(q); q += align256((size_t)3 * nb * 4);
    A->bin_sizes = reinterpret_cast<int*>(q);
  }
  lbk::bin_count_kernel<<<nb, 256, 0, s>>>((int)A->rows, A->off, nb, A->bin_counts);
  LB_LAUNCHED();
  lbk::bin_scan_kernel<<<1, 1024, 0, s>>>(nb, A->bin_counts, A->bin_sizes);
  LB_LAUNCHED();
  lbk::bin_scatter_kernel<<<nb, 256, 0, s>>>((int)A->rows, A->off, nb, A->bin_counts, A->bin_ids);
  LB_LAUNCHED();
  return LB_OK;
}

// the three bin kernels (one specialised kernel per bin), persistent grids
lb_status_t launch_bin_kernels(lb_csr_s* A, const float* x, float* y, stream_t s) {
  const int sms = A->dev->sm_count;
  lbk::bin_cta_kernel<<<sms * 8, 256, 0, s>>>(A->bin_ids, A->bin_sizes, A->off, A->col, A->val, x, y);
  LB_LAUNCHED();
  lbk::bin_warp_kernel<<<sms * 8, 256, 0, s>>>(A->bin_ids, A->bin_sizes, A->off, A->col, A->val, x, y);
  LB_LAUNCHED();
  lbk::bin_thread_kernel<<<sms * 16, 256, 0, s>>>(A->bin_ids, A->bin_sizes, A->off, A->col, A->val, x, y);
  LB_LAUNCHED();
  return LB_OK;
}

lb_status_t spmv_impl(lb_csr_s* A, lb_schedule_t sched, const float* x, float* y, uint32_t flags, stream_t s,
                      PhaseEvents* pe, const PeerArgs* pa = nullptr, bool* fused = nullptr) {
  if (fused) *fused = false;
  if (!A) return fail(LB_ERR_INVALID_ARG, "null handle");
  if (A->rows == 0) return LB_OK;
  if (!y || (!x && A->nnz > 0)) return fail(LB_ERR_INVALID_ARG, "null x or y");
  if ((const void*)x == (const void*)y) return fail(LB_ERR_INVALID_ARG, "x and y must not alias");
  if (sched == LB_SCHED_AUTO) {
    lb_status_t st = select_schedule(A, s, &sched);
    if (st != LB_OK) return st;
  }
  if (pe) LB_CUDA(cudaEventRecord(pe->ev[0], s));
  switch (sched) {
    case LB_SCHED_THREAD_MAPPED: {
      if (pe) LB_CUDA(cudaEventRecord(pe->ev[1], s));
      // Listing 3: blocks of 256 threads, grid = ceil(rows / 256)
      const int64_t grid = (A->rows + kNT - 1) / kNT;
      lbk::thread_mapped_kernel<<<(unsigned)grid, kNT, 0, s>>>((int)A->rows, A->off, A->col, A->val, x, y);
      LB_LAUNCHED();
      if (pe) { LB_CUDA(cudaEventRecord(pe->ev[2], s)); LB_CUDA(cudaEventRecord(pe->ev[3], s)); }
      return LB_OK;
    }
    case LB_SCHED_GROUP_MAPPED:
    case LB_SCHED_BLOCK_MAPPED: {
      if (pe) LB_CUDA(cudaEventRecord(pe->ev[1], s));
      const int G = sched == LB_SCHED_GROUP_MAPPED ? 32 : 256;
      const int64_t groups = (A->rows + G - 1) / G;
      const int64_t groups_per_cta = kNT / G;
      const int64_t grid = std::max<int64_t>(1, (groups + groups_per_cta - 1) / groups_per_cta);
      if (G == 32)
        lbk::group_mapped_kernel<32><<<(unsigned)grid, kNT, 0, s>>>((int)A->rows, A->off, A->col, A->val, x, y);
      else
        lbk::group_mapped_kernel<256><<<(unsigned)grid, kNT, 0, s>>>((int)A->rows, A->off, A->col, A->val, x, y);
      LB_LAUNCHED();
      if (pe) { LB_CUDA(cudaEventRecord(pe->ev[2], s)); LB_CUDA(cudaEventRecord(pe->ev[3], s)); }
      return LB_OK;
    }
    case LB_SCHED_MERGE_PATH: {
      lb_status_t st;
      const bool repart = !A->coords_valid || A->coords_kind != 0 || A->coords_L != A->L || (flags & LB_SPMV_REPARTITION);
      if (hot_usable(A)) {  // hot-column plan: partition + x_hot gather in one launch, then the hot tile kernel
        if ((st = launch_partition_xhot(A, A->L, repart, x, s)) != LB_OK) return st;
        if (repart) { A->coords_valid = true; A->coords_L = A->L; A->coords_kind = 0; }
        if (pe) LB_CUDA(cudaEventRecord(pe->ev[1], s));
        if ((st = hot_launch(A, x, y, s, pa)) != LB_OK) return st;
        if (fused) *fused = pa != nullptr;
        if (pe) { LB_CUDA(cudaEventRecord(pe->ev[2], s)); LB_CUDA(cudaEventRecord(pe->ev[3], s)); }
        return LB_OK;
      }
      if (pa && A->vec32 && (A->L == 1016 || A->L == 504)) {  // fused epilogue, plain CSR
        if (repart) {
          if ((st = launch_partition(A, A->L, A->coords, s)) != LB_OK) return st;
          A->coords_valid = true; A->coords_L = A->L; A->coords_kind = 0;
        }
        if (pe) LB_CUDA(cudaEventRecord(pe->ev[1], s));
        st = A->L == 1016 ? peers_stream_launch<4>(A, x, y, s, pa) : peers_stream_launch<2>(A, x, y, s, pa);
        if (st != LB_OK) return st;
        if (fused) *fused = true;
        if (pe) { LB_CUDA(cudaEventRecord(pe->ev[2], s)); LB_CUDA(cudaEventRecord(pe->ev[3], s)); }
        return LB_OK;
      }
      if (repart) {
        if ((st = launch_partition(A, A->L, A->coords, s)) != LB_OK) return st;
        A->coords_valid = true;
        A->coords_L = A->L;
        A->coords_kind = 0;
      }
      if (pe) LB_CUDA(cudaEventRecord(pe->ev[1], s));
      switch (A->L) {
        case 504: return launch_merge<504>(A, x, y, s, pe);
        case 1016: return launch_merge<1016>(A, x, y, s, pe);
        case 2040: return launch_merge<2040>(A, x, y, s, pe);
        case 3064: return launch_merge<3064>(A, x, y, s, pe);
        case 4088: return launch_merge<4088>(A, x, y, s, pe);
        default: return fail(LB_ERR_INVALID_ARG, "unsupported tile length %d", A->L);
      }
    }
    case LB_SCHED_WARP_MAPPED: {
      if (pe) LB_CUDA(cudaEventRecord(pe->ev[1], s));
      // an equal share of rows per warp, kWarpRows rows each, with the warps
      // oversubscribed so that the hardware scheduler absorbs the imbalance
      const int64_t rpw = kWarpRows;
      const int64_t grid = ((A->rows + rpw - 1) / rpw * 32 + kNT - 1) / kNT;
      lbk::warp_mapped_kernel<<<(unsigned)grid, kNT, 0, s>>>((int)A->rows, (int)rpw, A->off, A->col, A->val, x, y);
      LB_LAUNCHED();
      if (pe) { LB_CUDA(cudaEventRecord(pe->ev[2], s)); LB_CUDA(cudaEventRecord(pe->ev[3], s)); }
      return LB_OK;
    }
    case LB_SCHED_BINNING: {
      lb_status_t st;
      if ((st = launch_bins(A, s)) != LB_OK) return st;  // bins depend only on A, rebuilt every call (Alg.4 runtime phase)
      if (pe) LB_CUDA(cudaEventRecord(pe->ev[1], s));
      if ((st = launch_bin_kernels(A, x, y, s)) != LB_OK) return st;
      if (pe) { LB_CUDA(cudaEventRecord(pe->ev[2], s)); LB_CUDA(cudaEventRecord(pe->ev[3], s)); }
      return LB_OK;
    }
    case LB_SCHED_NONZERO_SPLIT: {
      if (!A->vec32) return fail(LB_ERR_UNSUPPORTED, "nonzero-split needs 32-byte aligned col_idx/values");
      lb_status_t st;
      if (!A->coords_valid || A->coords_kind != 1 || A->coords_L != kNzL || (flags & LB_SPMV_REPARTITION)) {
        if ((st = launch_partition_nz(A, kNzL, A->coords, s)) != LB_OK) return st;
        A->coords_valid = true;
        A->coords_L = kNzL;
        A->coords_kind = 1;
      }
      if (pe) LB_CUDA(cudaEventRecord(pe->ev[1], s));
      if ((st = launch_nz_tiles(A, x, y, s)) != LB_OK) return st;
      if (pe) { LB_CUDA(cudaEventRecord(pe->ev[2], s)); LB_CUDA(cudaEventRecord(pe->ev[3], s)); }
      return LB_OK;
    }
    default:
      return fail(LB_ERR_INVALID_ARG, "unknown schedule id %d", (int)sched);
  }
}

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
  if (!A->sssp_mem) {
    const size_t ntc = (size_t)((n + A->nnz) / lbk::kSsspTile + 2);  // tile boundaries of the largest round
    const size_t bytes = 3 * align256((size_t)n * 4) + align256(((size_t)n + 1) * 4) + align256((size_t)nb_max * 4 + 4) +
                         align256(16) + align256(ntc * 4);
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) { cudaGetLastError(); return fail(LB_ERR_OOM, "SSSP workspace"); }
    char* q = static_cast<char*>(p);
    A->sssp_mem = p;
    A->q_a = reinterpret_cast<int*>(q); q += align256((size_t)n * 4);
    A->q_b = reinterpret_cast<int*>(q); q += align256((size_t)n * 4);
    A->stamp = reinterpret_cast<int*>(q); q += align256((size_t)n * 4);
    A->fo = reinterpret_cast<int*>(q); q += align256(((size_t)n + 1) * 4);
    A->bsum = reinterpret_cast<int*>(q); q += align256((size_t)nb_max * 4 + 4);
    A->counts = reinterpret_cast<int*>(q); q += align256(16);
    A->tc = reinterpret_cast<int*>(q);
  }
  const int sms = A->dev->sm_count;
  lbk::sssp_init_kernel<<<sms * 8, kNT, 0, s>>>(n, (int)source, dist, A->stamp, A->q_a, A->counts);
  LB_LAUNCHED();
  if (A->nnz > 0) {
    lbk::sssp_check_weights_kernel<<<sms * 8, kNT, 0, s>>>(A->nnz, A->val, A->counts + 2);
    LB_LAUNCHED();
  }
  int h[3];
  LB_CUDA(cudaMemcpyAsync(h, A->counts, sizeof h, cudaMemcpyDeviceToHost, s));
  LB_CUDA(cudaStreamSynchronize(s));
  if (h[2]) return fail(LB_ERR_INVALID_ARG, "negative (or NaN) edge weight");
  int F = 1, round = 0;
  int* qi = A->q_a;
  int* qo = A->q_b;
  while (F > 0) {
    LB_CUDA(cudaMemsetAsync(A->counts + 1, 0, sizeof(int), s));
    if (sched == LB_SCHED_THREAD_MAPPED) {
      lbk::sssp_thread_kernel<<<(F + kNT - 1) / kNT, kNT, 0, s>>>(F, qi, A->off, A->col, A->val, dist, A->stamp, round,
                                                                   qo, A->counts + 1);
      LB_LAUNCHED();
    } else if (sched == LB_SCHED_GROUP_MAPPED) {
      const int64_t warps = (F + 31) / 32;
      const int grid = (int)std::min<int64_t>((warps * 32 + kNT - 1) / kNT, (int64_t)sms * 16);
      lbk::sssp_warp_kernel<<<grid, kNT, 0, s>>>(F, qi, A->off, A->col, A->val, dist, A->stamp, round, qo,
                                                 A->counts + 1);
      LB_LAUNCHED();
    } else {
      const int nb = (F + lbk::kScanChunk - 1) / lbk::kScanChunk;
      lbk::frontier_deg_sum_kernel<<<nb, 256, 0, s>>>(F, qi, A->off, A->bsum);
      LB_LAUNCHED();
      lbk::frontier_bsum_scan_kernel<<<1, 1024, 0, s>>>(nb, A->bsum);
      LB_LAUNCHED();
      lbk::frontier_deg_scan_kernel<<<nb, 256, 0, s>>>(F, qi, A->off, A->bsum, nb, A->fo);
      LB_LAUNCHED();
      // the round's CTA tiles: boundaries in parallel (host-side tile count from F + E_f is not known
      // without a sync, so the boundary kernel covers the largest possible count and each tile kernel
      // CTA stops at F + E_f)
      const int T = (int)((F + A->nnz + lbk::kSsspTile - 1) / lbk::kSsspTile);
      lbk::sssp_tile_coords_kernel<<<(T + 1 + 255) / 256, 256, 0, s>>>(F, A->fo, T, A->tc);
      LB_LAUNCHED();
      const int grid = sms * 8;  // persistent over the round's CTA tiles
      lbk::sssp_merge_kernel<<<grid, kNT, 0, s>>>(F, qi, A->fo, A->off, A->col, A->val, dist, A->stamp, round, qo,
                                                  A->counts + 1, A->tc);
      LB_LAUNCHED();
    }
    LB_CUDA(cudaMemcpyAsync(&F, A->counts + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
    LB_CUDA(cudaStreamSynchronize(s));
    std::swap(qi, qo);
    ++round;
  }
  if (rounds_out) *rounds_out = round;
  return LB_OK;
}

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

// ============================================================================ C ABI
extern "C" {

const char* lb_last_error(void) { return g_err.c_str(); }

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
    case LB_SCHED_MERGE_PATH: {
      if (!A || l_index(A->L) < 0) return "";
      if (hot_usable(A)) {
        snprintf(buf, sizeof buf, "merge_stream_kernel<%d,%d,1,%s>", hot_warps(), (A->L + 8) / 256,
                 A->warm_n > 0 ? "hot+warm" : "hot");
        return buf;
      }
      const PipeVariant& v = kVariants[pipe_variant_for(A->L)];
      const bool ok = v.kind == 0 ? A->vec : v.kind == 1 ? A->pipe : A->vec32;
      if (!ok) { snprintf(buf, sizeof buf, "merge_tile_kernel<256,%d> + fixup_kernel", A->L); return buf; }
      static const char* kinds[4] = {"merge_direct_kernel", "merge_pipe_kernel", "merge_wide_kernel",
                                     "merge_stream_kernel"};
      if (v.kind == 0) snprintf(buf, sizeof buf, "%s<%d,%d>", kinds[0], v.nt, v.minb);
      else if (v.kind == 3) snprintf(buf, sizeof buf, "%s<%d,%d,%d>", kinds[3], v.nt / 32, (v.L + 8) / 256, v.minb);
      else snprintf(buf, sizeof buf, "%s<%d,%d,%d>", kinds[v.kind], v.nt, v.e, v.minb);
      return buf;
    }
    default: return "";
  }
}
uint64_t lb_launch_count(void) { return g_launches.load(); }
const char* lb_version(void) { return "liblb 0.1 (sm_100a)"; }

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

lb_status_t lb_bins(lb_csr_t A, int32_t* d_ids, int64_t h_sizes[3], void* stream) {
  g_err.clear();
  if (!A || !h_sizes || (!d_ids && A->rows > 0)) return fail(LB_ERR_INVALID_ARG, "bad lb_bins arguments");
  h_sizes[0] = h_sizes[1] = h_sizes[2] = 0;
  if (A->rows == 0) return LB_OK;
  stream_t s = S(stream);
  lb_status_t st;
  if ((st = launch_bins(A, s)) != LB_OK) return st;
  LB_CUDA(cudaMemcpyAsync(d_ids, A->bin_ids, (size_t)A->rows * 4, cudaMemcpyDeviceToDevice, s));
  int h[3];
  LB_CUDA(cudaMemcpyAsync(h, A->bin_sizes, sizeof h, cudaMemcpyDeviceToHost, s));
  LB_CUDA(cudaStreamSynchronize(s));
  for (int q = 0; q < 3; ++q) h_sizes[q] = h[q];
  return LB_OK;
}

lb_status_t lb_csr_destroy(lb_csr_t A) {
  if (!A) return LB_OK;
  if (A->owns_scratch && A->coords) cudaFree(A->coords);
  if (A->plan_mem) cudaFree(A->plan_mem);
  if (A->sssp_mem) cudaFree(A->sssp_mem);
  if (A->bin_mem) cudaFree(A->bin_mem);
  if (A->hx_stage) cudaFree(A->hx_stage);
  if (A->mc_stream) {
    cudaStreamSynchronize(A->mc_stream);
    cudaStreamDestroy(A->mc_stream);
    if (A->mc_done) cudaEventDestroy(A->mc_done);
  }
  if (A->ch_d2h) {
    cudaStreamSynchronize(A->ch_d2h);
    for (auto& e : A->ch_ev)
      if (e) cudaEventDestroy(e);
    cudaStreamDestroy(A->ch_d2h);
  }
  if (A->hp_mem) {
    if (A->hp_h2d) cudaStreamSynchronize(A->hp_h2d);
    if (A->hp_d2h) cudaStreamSynchronize(A->hp_d2h);
    for (int i = 0; i < 2; ++i) {
      if (A->hp_xready[i]) cudaEventDestroy(A->hp_xready[i]);
      if (A->hp_done[i]) cudaEventDestroy(A->hp_done[i]);
      if (A->hp_out[i]) cudaEventDestroy(A->hp_out[i]);
    }
    if (A->hp_h2d) cudaStreamDestroy(A->hp_h2d);
    if (A->hp_d2h) cudaStreamDestroy(A->hp_d2h);
    cudaFree(A->hp_mem);
  }
  delete A;
  return LB_OK;
}

lb_status_t lb_csr_set_items_per_tile(lb_csr_t A, int32_t items_per_tile) {
  if (!A) return fail(LB_ERR_INVALID_ARG, "null handle");
  int L = items_per_tile == 0 ? auto_tile_length(A->rows, A->nnz) : items_per_tile;
  if (l_index(L) < 0) return fail(LB_ERR_INVALID_ARG, "items_per_tile %d unsupported (504, 1016, 2040, 3064, 4088)", L);
  A->L = L;
  A->coords_valid = false;
  return LB_OK;
}

lb_status_t lb_partition_size(lb_csr_t A, int32_t items_per_tile, int64_t* n) {
  if (!A || !n) return fail(LB_ERR_INVALID_ARG, "null argument");
  int64_t L = items_per_tile == 0 ? A->L : items_per_tile;
  if (L <= 0) return fail(LB_ERR_INVALID_ARG, "items_per_tile must be >= 1");
  *n = num_tiles(A->rows, A->nnz, L);
  return LB_OK;
}

lb_status_t lb_partition(lb_csr_t A, int32_t items_per_tile, int32_t* d_coords, void* stream) {
  g_err.clear();
  if (!A || !d_coords) return fail(LB_ERR_INVALID_ARG, "null argument");
  int64_t L = items_per_tile == 0 ? A->L : items_per_tile;
  if (L <= 0) return fail(LB_ERR_INVALID_ARG, "items_per_tile must be >= 1");
  return launch_partition(A, L, reinterpret_cast<int2*>(d_coords), S(stream));
}

lb_status_t lb_probe_stream_gather(lb_csr_t A, const float* d_x, int32_t reps, void* stream, float* ms_out) {
  g_err.clear();
  if (!A || !ms_out || reps < 1 || (!d_x && A->nnz > 0)) return fail(LB_ERR_INVALID_ARG, "bad probe arguments");
  if (!A->vec32) return fail(LB_ERR_UNSUPPORTED, "probe needs 32-byte aligned col_idx/values");
  stream_t s = S(stream);
  const int tier = A->hot_n > 0 ? (A->warm_n > 0 && !A->compact ? 2 : 1) : 0;
  lb_status_t st;
  if (tier > 0 && (st = launch_partition_xhot(A, 0, false, d_x, s)) != LB_OK) return st;  // x_hot / x_warm of this x
  const float* xg = A->compact ? A->x_warm : d_x;
  auto launch = [&]() { return tier == 2 ? probe_launch<2>(A, d_x, s) : tier == 1 ? probe_launch<1>(A, xg, s)
                                                                                   : probe_launch<0>(A, d_x, s); };
  if ((st = launch()) != LB_OK) return st;  // warm-up
  cudaEvent_t e0, e1;
  LB_CUDA(cudaEventCreate(&e0));
  LB_CUDA(cudaEventCreate(&e1));
  LB_CUDA(cudaEventRecord(e0, s));
  for (int r = 0; r < reps; ++r)
    if ((st = launch()) != LB_OK) return st;
  LB_CUDA(cudaEventRecord(e1, s));
  LB_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  LB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  *ms_out = ms / reps;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return LB_OK;
}

lb_status_t lb_probe_stream(lb_csr_t A, int32_t reps, void* stream, float* ms_out) {
  g_err.clear();
  if (!A || !ms_out || reps < 1) return fail(LB_ERR_INVALID_ARG, "bad probe arguments");
  if (!A->vec32) return fail(LB_ERR_UNSUPPORTED, "probe needs 32-byte aligned col_idx/values");
  stream_t s = S(stream);
  int blocks = 0;
  LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, lbk::probe_stream_kernel, 512, 0));
  const int grid = A->dev->sm_count * std::max(1, blocks);
  auto launch = [&]() -> lb_status_t {
    lbk::probe_stream_kernel<<<grid, 512, 0, s>>>((int)A->nnz, A->col, A->val, 0, nullptr);
    LB_LAUNCHED();
    return LB_OK;
  };
  lb_status_t st;
  if ((st = launch()) != LB_OK) return st;  // warm-up
  cudaEvent_t e0, e1;
  LB_CUDA(cudaEventCreate(&e0));
  LB_CUDA(cudaEventCreate(&e1));
  LB_CUDA(cudaEventRecord(e0, s));
  for (int r = 0; r < reps; ++r)
    if ((st = launch()) != LB_OK) return st;
  LB_CUDA(cudaEventRecord(e1, s));
  LB_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  LB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  *ms_out = ms / reps;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return LB_OK;
}

lb_status_t lb_csr_plan_hot_x(lb_csr_t A, int32_t slots, int64_t warm_cols, void* stream, int32_t* hot_cols_out,
                              int64_t* hot_nnz_out) {
  g_err.clear();
  if (!A) return fail(LB_ERR_INVALID_ARG, "null handle");
  if (slots < 0) {
    drop_plan(A);
  } else {
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
    }
  }
  if (hot_cols_out) *hot_cols_out = A->hot_n;
  if (hot_nnz_out) *hot_nnz_out = A->hot_nnz;
  return LB_OK;
}

lb_status_t lb_csr_hot_plan(lb_csr_t A, int32_t* hot_n, int64_t* hot_nnz, int64_t* warm_n, int64_t* warm_nnz,
                            int32_t* d_hot_cols_out, int32_t* d_warm_cols_out, int32_t* d_col_out, void* stream) {
  g_err.clear();
  if (!A) return fail(LB_ERR_INVALID_ARG, "null handle");
  if (hot_n) *hot_n = A->hot_n;
  if (hot_nnz) *hot_nnz = A->hot_nnz;
  if (warm_n) *warm_n = A->warm_n;
  if (warm_nnz) *warm_nnz = A->warm_nnz;
  if (A->hot_n > 0) {
    if (d_hot_cols_out)
      LB_CUDA(cudaMemcpyAsync(d_hot_cols_out, A->hot_cols, (size_t)A->hot_n * 4, cudaMemcpyDeviceToDevice, S(stream)));
    if (d_warm_cols_out && A->warm_n > 0)
      LB_CUDA(cudaMemcpyAsync(d_warm_cols_out, A->warm_cols, (size_t)A->warm_n * 4, cudaMemcpyDeviceToDevice, S(stream)));
    if (d_col_out)
      LB_CUDA(cudaMemcpyAsync(d_col_out, A->hcol, (size_t)A->nnz * 4, cudaMemcpyDeviceToDevice, S(stream)));
  }
  return LB_OK;
}

lb_status_t lb_partition_nz(lb_csr_t A, int32_t items_per_tile, int32_t* d_coords, void* stream) {
  g_err.clear();
  if (!A || !d_coords) return fail(LB_ERR_INVALID_ARG, "null argument");
  const int64_t L = items_per_tile == 0 ? kNzL : items_per_tile;
  if (L <= 0) return fail(LB_ERR_INVALID_ARG, "items_per_tile must be >= 1");
  return launch_partition_nz(A, L, reinterpret_cast<int2*>(d_coords), S(stream));
}

lb_status_t lb_spmv(lb_csr_t A, lb_schedule_t sched, const float* d_x, float* d_y, void* stream) {
  g_err.clear();
  return spmv_impl(A, sched, d_x, d_y, 0u, S(stream), nullptr);
}

lb_status_t lb_sssp(lb_csr_t A, int64_t source, lb_schedule_t sched, float* d_dist, void* stream, int32_t* rounds_out) {
  g_err.clear();
  return sssp_impl(A, source, sched, d_dist, S(stream), rounds_out);
}

lb_status_t lb_spmm(lb_csr_t A, int64_t n, const float* d_X, int64_t ldx, float* d_Y, int64_t ldy, void* stream) {
  g_err.clear();
  return spmm_impl(A, n, d_X, ldx, d_Y, ldy, S(stream));
}

lb_status_t lb_spmv_ex(lb_csr_t A, lb_schedule_t sched, const float* d_x, float* d_y, uint32_t flags, void* stream) {
  g_err.clear();
  return spmv_impl(A, sched, d_x, d_y, flags, S(stream), nullptr);
}

lb_status_t lb_spmv_peers(lb_csr_t A, const float* d_x, float* d_y, float* const* h_peer_y, int32_t npeers,
                          uint32_t flags, void* stream) {
  g_err.clear();
  if (!A) return fail(LB_ERR_INVALID_ARG, "null handle");
  if (npeers < 0 || npeers > lbk::kMaxPeers) return fail(LB_ERR_INVALID_ARG, "npeers %d not in [0, %d]", npeers, lbk::kMaxPeers);
  if (npeers > 0 && !h_peer_y) return fail(LB_ERR_INVALID_ARG, "null peer array");
  PeerArgs pa;
  pa.n = npeers;
  for (int p = 0; p < npeers; ++p) {
    if (!h_peer_y[p]) return fail(LB_ERR_INVALID_ARG, "null peer %d", p);
    pa.y[p] = h_peer_y[p];
  }
  bool fused = false;
  lb_status_t st = spmv_impl(A, LB_SCHED_MERGE_PATH, d_x, d_y, flags, S(stream), nullptr, &pa, &fused);
  if (st != LB_OK) return st;
  if (!fused) return fail(LB_ERR_UNSUPPORTED, "no fused kernel for this handle (needs L = 504 or 1016 and 32-byte aligned arrays)");
  return LB_OK;
}

lb_status_t lb_spmv_phase_times(lb_csr_t A, lb_schedule_t sched, const float* d_x, float* d_y, void* stream,
                                float* ms_out) {
  g_err.clear();
  if (!ms_out) return fail(LB_ERR_INVALID_ARG, "null ms_out");
  PhaseEvents pe;
  for (auto& e : pe.ev) LB_CUDA(cudaEventCreate(&e));
  lb_status_t st = spmv_impl(A, sched, d_x, d_y, LB_SPMV_REPARTITION, S(stream), &pe);
  if (st == LB_OK && A->rows > 0) {
    LB_CUDA(cudaEventSynchronize(pe.ev[3]));
    for (int i = 0; i < 3; ++i) LB_CUDA(cudaEventElapsedTime(&ms_out[i], pe.ev[i], pe.ev[i + 1]));
  } else if (st == LB_OK) {
    ms_out[0] = ms_out[1] = ms_out[2] = 0.f;
  }
  for (auto& e : pe.ev) cudaEventDestroy(e);
  return st;
}

constexpr int kChunks = 8;

// Clean chunk cuts of A's merge-path tiles at its tile length (computed once per tile length; the
// partition must be current).  Synchronises `s` on first use.
lb_status_t ensure_chunks(lb_csr_s* A, stream_t s) {
  const int64_t T = num_tiles(A->rows, A->nnz, A->L);
  if (A->ch_L != A->L) {  // chunk boundaries of this tile length (deterministic: computed once)
    int* d_out = nullptr;
    if (cudaMalloc(&d_out, 2 * kChunks * sizeof(int)) != cudaSuccess) { cudaGetLastError(); return fail(LB_ERR_OOM, "chunks"); }
    // a hot tile-kernel launch has `wave` warps and takes ceil(tiles / wave) tiles per warp: cut after
    // q whole waves minus a slack of 32 tiles, so a clean cut found within the slack (a clean start
    // every ~1 + nnz/rows merge items) keeps the chunk at q waves
    const int64_t wave = std::min(A->dev->sm_count * hot_warps(), kMaxCtas), slack = 32;
    const int64_t q = T / ((int64_t)kChunks * wave);
    const int64_t step = q >= 1 && q * wave > 4 * slack ? q * wave - slack : T / kChunks;
    lbk::clean_tiles_kernel<<<1, 32, 0, s>>>(A->coords, A->off, T, kChunks, 4096, step, d_out);
    LB_LAUNCHED();
    int h[2 * kChunks] = {};
    cudaError_t e1 = cudaMemcpyAsync(h, d_out, sizeof h, cudaMemcpyDeviceToHost, s);
    cudaError_t e2 = e1 == cudaSuccess ? cudaStreamSynchronize(s) : e1;
    cudaFree(d_out);
    if (e2 != cudaSuccess) return fail(LB_ERR_CUDA, "chunk boundaries: %s", cudaGetErrorString(e2));
    int n = 0;
    A->ch_t[0] = 0; A->ch_i[0] = 0;
    for (int k = 1; k < kChunks; ++k)
      if (h[k] > A->ch_t[n] && h[k] < T) { ++n; A->ch_t[n] = h[k]; A->ch_i[n] = h[kChunks + k]; }
    ++n;
    A->ch_t[n] = T; A->ch_i[n] = A->rows;
    A->ch_n = n;
    A->ch_L = A->L;
  }
  return LB_OK;
}

// LB_SPMV_CHUNKED: the merge-path step with the hot plan as kChunks tile-kernel launches over tile
// ranges that start and end on clean merge-path coordinates (no row split across a boundary, so each
// launch's rows are final when it ends); the D2H copy of chunk k's rows overlaps chunk k+1.
lb_status_t host_x_chunked(lb_csr_s* A, const float* d_x, float* d_y, float* h_y, uint32_t flags, stream_t s) {
  lb_status_t st;
  const bool repart = !A->coords_valid || A->coords_kind != 0 || A->coords_L != A->L || (flags & LB_SPMV_REPARTITION);
  if ((st = launch_partition_xhot(A, A->L, repart, d_x, s)) != LB_OK) return st;
  if (repart) { A->coords_valid = true; A->coords_L = A->L; A->coords_kind = 0; }
  if (!A->ch_d2h) {
    LB_CUDA(cudaStreamCreateWithFlags(&A->ch_d2h, cudaStreamNonBlocking));
    for (auto& e : A->ch_ev) LB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  if ((st = ensure_chunks(A, s)) != LB_OK) return st;
  for (int k = 0; k < A->ch_n; ++k) {
    A->tr_t0 = A->ch_t[k];
    A->tr_t1 = A->ch_t[k + 1];
    st = hot_launch(A, d_x, d_y, s);
    A->tr_t0 = 0;
    A->tr_t1 = -1;
    if (st != LB_OK) return st;
    LB_CUDA(cudaEventRecord(A->ch_ev[k], s));
    LB_CUDA(cudaStreamWaitEvent(A->ch_d2h, A->ch_ev[k], 0));
    const int64_t r0 = A->ch_i[k], r1 = A->ch_i[k + 1];
    if (r1 > r0)
      LB_CUDA(cudaMemcpyAsync(h_y + r0, d_y + r0, (size_t)(r1 - r0) * 4, cudaMemcpyDeviceToHost, A->ch_d2h));
  }
  LB_CUDA(cudaStreamSynchronize(A->ch_d2h));
  LB_CUDA(cudaStreamSynchronize(s));
  return LB_OK;
}

lb_status_t lb_spmv_host_x(lb_csr_t A, lb_schedule_t sched, const float* h_x, float* h_y, uint32_t flags,
                           void* stream) {
  g_err.clear();
  if (!A) return fail(LB_ERR_INVALID_ARG, "null handle");
  if (A->rows == 0) return LB_OK;
  if (!h_y || (!h_x && A->cols > 0)) return fail(LB_ERR_INVALID_ARG, "null host x or y");
  if (!A->hx_stage) {
    void* p = nullptr;
    // x and y separately aligned (256 B) inside one allocation
    if (cudaMalloc(&p, align256((size_t)A->cols * 4) + (size_t)A->rows * 4) != cudaSuccess) {
      cudaGetLastError();
      return fail(LB_ERR_OOM, "lb_spmv_host_x staging");
    }
    A->hx_stage = static_cast<float*>(p);
  }
  stream_t s = S(stream);
  float* d_x = A->hx_stage;
  float* d_y = reinterpret_cast<float*>(reinterpret_cast<char*>(A->hx_stage) + align256((size_t)A->cols * 4));
  if (A->cols > 0) LB_CUDA(cudaMemcpyAsync(d_x, h_x, (size_t)A->cols * 4, cudaMemcpyHostToDevice, s));
  if ((flags & LB_SPMV_CHUNKED) && sched == LB_SCHED_MERGE_PATH && hot_usable(A))
    return host_x_chunked(A, d_x, d_y, h_y, flags, s);
  lb_status_t st = spmv_impl(A, sched, d_x, d_y, flags, s, nullptr);
  if (st != LB_OK) return st;
  LB_CUDA(cudaMemcpyAsync(h_y, d_y, (size_t)A->rows * 4, cudaMemcpyDeviceToHost, s));
  LB_CUDA(cudaStreamSynchronize(s));
  return LB_OK;
}

lb_status_t lb_spmv_host_x_async(lb_csr_t A, lb_schedule_t sched, const float* h_x, float* h_y, uint32_t flags,
                                 void* stream) {
  g_err.clear();
  if (!A) return fail(LB_ERR_INVALID_ARG, "null handle");
  if (A->rows == 0) return LB_OK;
  if (!h_y || (!h_x && A->cols > 0)) return fail(LB_ERR_INVALID_ARG, "null host x or y");
  if (!A->hp_mem) {
    const size_t xb = align256((size_t)A->cols * 4), yb = align256((size_t)A->rows * 4);
    void* p = nullptr;
    if (cudaMalloc(&p, 2 * (xb + yb)) != cudaSuccess) {
      cudaGetLastError();
      return fail(LB_ERR_OOM, "lb_spmv_host_x_async staging");
    }
    A->hp_mem = p;
    char* b = static_cast<char*>(p);
    for (int i = 0; i < 2; ++i) {
      A->hp_x[i] = reinterpret_cast<float*>(b + i * (xb + yb));
      A->hp_y[i] = reinterpret_cast<float*>(b + i * (xb + yb) + xb);
      LB_CUDA(cudaEventCreateWithFlags(&A->hp_xready[i], cudaEventDisableTiming));
      LB_CUDA(cudaEventCreateWithFlags(&A->hp_done[i], cudaEventDisableTiming));
      LB_CUDA(cudaEventCreateWithFlags(&A->hp_out[i], cudaEventDisableTiming));
    }
    LB_CUDA(cudaStreamCreateWithFlags(&A->hp_h2d, cudaStreamNonBlocking));
    LB_CUDA(cudaStreamCreateWithFlags(&A->hp_d2h, cudaStreamNonBlocking));
  }
  const int k = A->hp_next;
  stream_t s = S(stream);
  // x slot k is free once the SpMV of the call two back (same slot) has read it
  LB_CUDA(cudaStreamWaitEvent(A->hp_h2d, A->hp_done[k], 0));
  if (A->cols > 0)
    LB_CUDA(cudaMemcpyAsync(A->hp_x[k], h_x, (size_t)A->cols * 4, cudaMemcpyHostToDevice, A->hp_h2d));
  LB_CUDA(cudaEventRecord(A->hp_xready[k], A->hp_h2d));
  // the SpMV waits for its x and for y slot k to have been copied out by the call two back
  LB_CUDA(cudaStreamWaitEvent(s, A->hp_xready[k], 0));
  LB_CUDA(cudaStreamWaitEvent(s, A->hp_out[k], 0));
  lb_status_t st = spmv_impl(A, sched, A->hp_x[k], A->hp_y[k], flags, s, nullptr);
  if (st != LB_OK) return st;
  LB_CUDA(cudaEventRecord(A->hp_done[k], s));
  LB_CUDA(cudaStreamWaitEvent(A->hp_d2h, A->hp_done[k], 0));
  LB_CUDA(cudaMemcpyAsync(h_y, A->hp_y[k], (size_t)A->rows * 4, cudaMemcpyDeviceToHost, A->hp_d2h));
  LB_CUDA(cudaEventRecord(A->hp_out[k], A->hp_d2h));
  A->hp_next = k ^ 1;
  return LB_OK;
}

lb_status_t lb_spmv_host_x_wait(lb_csr_t A) {
  g_err.clear();
  if (!A) return fail(LB_ERR_INVALID_ARG, "null handle");
  if (!A->hp_mem) return LB_OK;
  LB_CUDA(cudaStreamSynchronize(A->hp_h2d));
  LB_CUDA(cudaStreamSynchronize(A->hp_d2h));
  return LB_OK;
}

size_t lb_spmv_host_workspace_size(int64_t rows, int64_t cols, int64_t nnz) {
  if (rows < 0 || cols < 0 || nnz < 0) return 0;
  return align256((rows + 1) * 4) + 2 * align256(nnz * 4) + align256(cols * 4) + align256(rows * 4) +
         scratch_bytes(rows, nnz);
}

lb_status_t lb_spmv_host(int64_t rows, int64_t cols, int64_t nnz, const int32_t* h_row_offsets,
                         const int32_t* h_col_idx, const float* h_values, const float* h_x, float* h_y,
                         lb_schedule_t sched, void* d_workspace, size_t workspace_bytes, void* stream) {
  g_err.clear();
  lb_status_t st = check_shape(rows, cols, nnz);
  if (st != LB_OK) return st;
  if (!h_row_offsets || (rows > 0 && !h_y) || (nnz > 0 && (!h_col_idx || !h_values || !h_x)))
    return fail(LB_ERR_INVALID_ARG, "null host buffer");
  if (!d_workspace || workspace_bytes < lb_spmv_host_workspace_size(rows, cols, nnz))
    return fail(LB_ERR_INVALID_ARG, "workspace too small (need %zu bytes)", lb_spmv_host_workspace_size(rows, cols, nnz));
  stream_t s = S(stream);
  char* p = static_cast<char*>(d_workspace);
  int32_t* d_off = reinterpret_cast<int32_t*>(p); p += align256((rows + 1) * 4);
  int32_t* d_col = reinterpret_cast<int32_t*>(p); p += align256(nnz * 4);
  float* d_val = reinterpret_cast<float*>(p); p += align256(nnz * 4);
  float* d_x = reinterpret_cast<float*>(p); p += align256(cols * 4);
  float* d_y = reinterpret_cast<float*>(p); p += align256(rows * 4);
  lb_csr_s A;
  A.owns_scratch = false;
  if ((st = init_handle(&A, rows, cols, nnz, d_off, d_col, d_val)) != LB_OK) return st;
  carve_scratch(&A, p);
  LB_CUDA(cudaMemsetAsync(A.ticket, 0, sizeof(unsigned), s));
  LB_CUDA(cudaMemcpyAsync(d_off, h_row_offsets, (rows + 1) * 4, cudaMemcpyHostToDevice, s));
  if (nnz > 0) {
    LB_CUDA(cudaMemcpyAsync(d_col, h_col_idx, nnz * 4, cudaMemcpyHostToDevice, s));
    LB_CUDA(cudaMemcpyAsync(d_val, h_values, nnz * 4, cudaMemcpyHostToDevice, s));
  }
  if (cols > 0 && h_x) LB_CUDA(cudaMemcpyAsync(d_x, h_x, cols * 4, cudaMemcpyHostToDevice, s));
  st = spmv_impl(&A, sched, d_x, d_y, LB_SPMV_REPARTITION, s, nullptr);
  if (st != LB_OK) return st;
  if (rows > 0) LB_CUDA(cudaMemcpyAsync(h_y, d_y, rows * 4, cudaMemcpyDeviceToHost, s));
  LB_CUDA(cudaStreamSynchronize(s));
  return LB_OK;
}

lb_status_t lb_shard_bounds(const int32_t* h_row_offsets, int64_t rows, int32_t nranks, int64_t* h_bounds) {
  g_err.clear();
  if (!h_row_offsets || !h_bounds) return fail(LB_ERR_INVALID_ARG, "null argument");
  if (rows < 0 || nranks < 1) return fail(LB_ERR_INVALID_ARG, "rows < 0 or nranks < 1");
  const int64_t nnz = h_row_offsets[rows];
  h_bounds[0] = 0;
  for (int32_t g = 1; g < nranks; ++g) {
    const int64_t target = (g * nnz + nranks - 1) / nranks;  // ceil(g*nnz/G)
    // lower bound: first r in [0, rows] with off[r] >= target
    int64_t lo = 0, hi = rows;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (h_row_offsets[mid] < target) lo = mid + 1; else hi = mid;
    }
    h_bounds[g] = lo;
  }
  h_bounds[nranks] = rows;
  return LB_OK;
}

}  // extern "C"

// ============================================================================ multi-GPU (NCCL via dlopen)
namespace {

// Minimal NCCL ABI (stable since NCCL 2.0).
typedef struct { char internal[128]; } nccl_uid_t;
typedef void* nccl_comm_t;
typedef int nccl_result_t;
constexpr int kNcclFloat32 = 7;
constexpr int kNcclInt32 = 2;

struct NcclApi {
  bool loaded = false;
  nccl_result_t (*GetUniqueId)(nccl_uid_t*) = nullptr;
  nccl_result_t (*CommInitRank)(nccl_comm_t*, int, nccl_uid_t, int) = nullptr;
  nccl_result_t (*CommDestroy)(nccl_comm_t) = nullptr;
  nccl_result_t (*Broadcast)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  nccl_result_t (*GroupStart)() = nullptr;
  nccl_result_t (*GroupEnd)() = nullptr;
  nccl_result_t (*CommGetAsyncError)(nccl_comm_t, nccl_result_t*) = nullptr;
  const char* (*GetErrorString)(nccl_result_t) = nullptr;
};

NcclApi g_nccl;
std::mutex g_nccl_mu;

lb_status_t nccl_load() {
  std::lock_guard<std::mutex> g(g_nccl_mu);
  if (g_nccl.loaded) return LB_OK;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);  // PyTorch's copy, if mapped
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return fail(LB_ERR_UNSUPPORTED, "cannot load libnccl.so.2: %s", dlerror());
#define SYM(name, field)                                                                       \
  g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name));                     \
  if (!g_nccl.field) return fail(LB_ERR_UNSUPPORTED, "NCCL symbol %s missing", name);
  SYM("ncclGetUniqueId", GetUniqueId)
  SYM("ncclCommInitRank", CommInitRank)
  SYM("ncclCommDestroy", CommDestroy)
  SYM("ncclBroadcast", Broadcast)
  SYM("ncclGroupStart", GroupStart)
  SYM("ncclGroupEnd", GroupEnd)
  SYM("ncclCommGetAsyncError", CommGetAsyncError)
  SYM("ncclGetErrorString", GetErrorString)
#undef SYM
  g_nccl.loaded = true;
  return LB_OK;
}

#define LB_NCCL(call)                                                                              \
  do {                                                                                             \
    nccl_result_t r_ = (call);                                                                     \
    if (r_ != 0) return fail(LB_ERR_NCCL, "%s: %s", #call, g_nccl.GetErrorString(r_));             \
  } while (0)

}  // namespace

struct lb_comm_s {
  nccl_comm_t comm = nullptr;
  int rank = 0, nranks = 1, device = 0;
};

// A y buffer registered with every rank of a communicator: CUDA IPC handles (plus the offset of the
// buffer inside its allocation, so PyTorch caching-allocator tensors work) are exchanged over NCCL and
// the peers' buffers are mapped into this process.
struct lb_peer_s {
  lb_comm_s* comm = nullptr;
  float* y = nullptr;               // this rank's buffer (caller-owned)
  int64_t rows = 0;
  float* peer_y[8] = {nullptr};     // index = rank (nullptr for this rank)
  void* peer_base[8] = {nullptr};   // mapped allocation bases (cudaIpcCloseMemHandle)
  int* d_flag = nullptr;            // barrier scratch [8]
  char* d_slots = nullptr;          // exchange buffer (owns d_flag)
};

namespace {

// allocation base of a device pointer (driver API, loaded at run time)
lb_status_t alloc_base(const void* p, void** base) {
  typedef int (*get_range_t)(unsigned long long*, size_t*, unsigned long long);
  static get_range_t fn = nullptr;
  if (!fn) {
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libcuda.so.1", RTLD_NOW);
    if (!h) return fail(LB_ERR_UNSUPPORTED, "cannot load libcuda.so.1");
    fn = reinterpret_cast<get_range_t>(dlsym(h, "cuMemGetAddressRange_v2"));
    if (!fn) return fail(LB_ERR_UNSUPPORTED, "cuMemGetAddressRange_v2 missing");
  }
  unsigned long long b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, (unsigned long long)p) != 0) return fail(LB_ERR_CUDA, "cuMemGetAddressRange failed");
  *base = reinterpret_cast<void*>(b);
  return LB_OK;
}

constexpr int kNcclUint8 = 1;

// every rank ends the call's stream work only after every rank reached it (NCCL group of 4-byte broadcasts)
lb_status_t peer_barrier(lb_peer_s* p, stream_t s) {
  lb_comm_s* c = p->comm;
  LB_NCCL(g_nccl.GroupStart());
  for (int k = 0; k < c->nranks; ++k) {
    nccl_result_t r = g_nccl.Broadcast(p->d_flag + k, p->d_flag + k, 4, kNcclUint8, k, c->comm, s);
    if (r != 0) { g_nccl.GroupEnd(); return fail(LB_ERR_NCCL, "ncclBroadcast: %s", g_nccl.GetErrorString(r)); }
  }
  LB_NCCL(g_nccl.GroupEnd());
  return LB_OK;
}

}  // namespace

extern "C" {

lb_status_t lb_comm_unique_id(uint8_t id_out[128]) {
  g_err.clear();
  if (!id_out) return fail(LB_ERR_INVALID_ARG, "null id buffer");
  lb_status_t st = nccl_load();
  if (st != LB_OK) return st;
  nccl_uid_t uid;
  LB_NCCL(g_nccl.GetUniqueId(&uid));
  memcpy(id_out, uid.internal, 128);
  return LB_OK;
}

lb_status_t lb_comm_init(const uint8_t id[128], int32_t rank, int32_t nranks, int32_t device, lb_comm_t* out) {
  g_err.clear();
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) return fail(LB_ERR_INVALID_ARG, "bad comm arguments");
  lb_status_t st = nccl_load();
  if (st != LB_OK) return st;
  LB_CUDA(cudaSetDevice(device));
  nccl_uid_t uid;
  memcpy(uid.internal, id, 128);
  lb_comm_s* c = new (std::nothrow) lb_comm_s();
  if (!c) return fail(LB_ERR_OOM, "host allocation failed");
  nccl_result_t r = g_nccl.CommInitRank(&c->comm, nranks, uid, rank);
  if (r != 0) { delete c; return fail(LB_ERR_NCCL, "ncclCommInitRank: %s", g_nccl.GetErrorString(r)); }
  c->rank = rank; c->nranks = nranks; c->device = device;
  *out = c;
  return LB_OK;
}

lb_status_t lb_comm_destroy(lb_comm_t c) {
  if (!c) return LB_OK;
  if (c->comm && g_nccl.loaded) g_nccl.CommDestroy(c->comm);
  delete c;
  return LB_OK;
}

lb_status_t lb_allgather_rows(lb_comm_t c, const int64_t* h_bounds, float* d_y_full, void* stream) {
  g_err.clear();
  if (!c || !h_bounds || !d_y_full) return fail(LB_ERR_INVALID_ARG, "null argument");
  for (int k = 0; k < c->nranks; ++k)
    if (h_bounds[k + 1] < h_bounds[k]) return fail(LB_ERR_INVALID_ARG, "bounds not monotone at %d", k);
  if (c->nranks == 1) return LB_OK;
  // all-gather(v) as one group of broadcasts, root k sends y[b_k, b_{k+1}) (SURVEY 8(e) option 1)
  LB_NCCL(g_nccl.GroupStart());
  for (int k = 0; k < c->nranks; ++k) {
    const size_t n = (size_t)(h_bounds[k + 1] - h_bounds[k]);
    if (n == 0) continue;
    float* p = d_y_full + h_bounds[k];
    nccl_result_t r = g_nccl.Broadcast(p, p, n, kNcclFloat32, k, c->comm, S(stream));
    if (r != 0) { g_nccl.GroupEnd(); return fail(LB_ERR_NCCL, "ncclBroadcast: %s", g_nccl.GetErrorString(r)); }
  }
  LB_NCCL(g_nccl.GroupEnd());
  nccl_result_t ar = 0;
  LB_NCCL(g_nccl.CommGetAsyncError(c->comm, &ar));
  if (ar != 0) return fail(LB_ERR_NCCL, "NCCL async error: %s", g_nccl.GetErrorString(ar));
  return LB_OK;
}

lb_status_t lb_peer_create(lb_comm_t c, float* d_y_full, int64_t rows_global, void* stream, lb_peer_t* out) {
  g_err.clear();
  if (!c || !d_y_full || !out || rows_global < 0) return fail(LB_ERR_INVALID_ARG, "bad peer-buffer arguments");
  if (c->nranks > 8) return fail(LB_ERR_UNSUPPORTED, "fused exchange supports up to 8 ranks (one node)");
  *out = nullptr;
  stream_t s = S(stream);
  lb_peer_s* p = new (std::nothrow) lb_peer_s();
  if (!p) return fail(LB_ERR_OOM, "host allocation failed");
  p->comm = c;
  p->y = d_y_full;
  p->rows = rows_global;
  struct Slot { cudaIpcMemHandle_t h; int64_t offset; char pad[64 - sizeof(int64_t)]; };
  static_assert(sizeof(Slot) == 128, "slot size");
  char* d_slots = nullptr;
  if (cudaMalloc(&d_slots, sizeof(Slot) * c->nranks + 64) != cudaSuccess) {
    cudaGetLastError(); delete p; return fail(LB_ERR_OOM, "peer exchange buffer");
  }
  p->d_slots = d_slots;
  p->d_flag = reinterpret_cast<int*>(d_slots + sizeof(Slot) * c->nranks);
  lb_status_t st = LB_OK;
  std::vector<Slot> slots(c->nranks);
  if (c->nranks > 1) {
    void* base = nullptr;
    if ((st = alloc_base(d_y_full, &base)) != LB_OK) { cudaFree(d_slots); delete p; return st; }
    Slot mine = {};
    if (cudaIpcGetMemHandle(&mine.h, base) != cudaSuccess) {
      cudaGetLastError(); cudaFree(d_slots); delete p; return fail(LB_ERR_CUDA, "cudaIpcGetMemHandle failed");
    }
    mine.offset = reinterpret_cast<char*>(d_y_full) - static_cast<char*>(base);
    auto run = [&]() -> lb_status_t {
      LB_CUDA(cudaMemcpyAsync(d_slots + sizeof(Slot) * c->rank, &mine, sizeof(Slot), cudaMemcpyHostToDevice, s));
      LB_NCCL(g_nccl.GroupStart());
      for (int k = 0; k < c->nranks; ++k) {
        char* q = d_slots + sizeof(Slot) * k;
        nccl_result_t r = g_nccl.Broadcast(q, q, sizeof(Slot), kNcclUint8, k, c->comm, s);
        if (r != 0) { g_nccl.GroupEnd(); return fail(LB_ERR_NCCL, "ncclBroadcast: %s", g_nccl.GetErrorString(r)); }
      }
      LB_NCCL(g_nccl.GroupEnd());
      LB_CUDA(cudaMemcpyAsync(slots.data(), d_slots, sizeof(Slot) * c->nranks, cudaMemcpyDeviceToHost, s));
      LB_CUDA(cudaStreamSynchronize(s));
      for (int k = 0; k < c->nranks; ++k) {
        if (k == c->rank) continue;
        void* pb = nullptr;
        LB_CUDA(cudaIpcOpenMemHandle(&pb, slots[k].h, cudaIpcMemLazyEnablePeerAccess));
        p->peer_base[k] = pb;
        p->peer_y[k] = reinterpret_cast<float*>(static_cast<char*>(pb) + slots[k].offset);
      }
      return LB_OK;
    };
    st = run();
  }
  if (st != LB_OK) { lb_peer_destroy(p); return st; }
  *out = p;
  return LB_OK;
}

lb_status_t lb_peer_destroy(lb_peer_t p) {
  if (!p) return LB_OK;
  for (int k = 0; k < 8; ++k)
    if (p->peer_base[k]) cudaIpcCloseMemHandle(p->peer_base[k]);
  if (p->d_slots) cudaFree(p->d_slots);
  delete p;
  return LB_OK;
}

lb_status_t lb_spmv_multi_fused(lb_csr_t A_local, lb_peer_t peer, lb_schedule_t sched, const int64_t* h_bounds,
                                const float* d_x_full, uint32_t flags, void* stream) {
  g_err.clear();
  if (!A_local || !peer || !h_bounds || !d_x_full) return fail(LB_ERR_INVALID_ARG, "null argument");
  lb_comm_s* c = peer->comm;
  if ((const void*)d_x_full == (const void*)peer->y) return fail(LB_ERR_INVALID_ARG, "x and y must not alias");
  const int64_t b0 = h_bounds[c->rank], b1 = h_bounds[c->rank + 1];
  if (b1 - b0 != A_local->rows)
    return fail(LB_ERR_INVALID_ARG, "local shard has %lld rows, bounds say %lld", (long long)A_local->rows,
                (long long)(b1 - b0));
  if (h_bounds[c->nranks] != peer->rows) return fail(LB_ERR_INVALID_ARG, "bounds do not match the peer buffer");
  PeerArgs pa;
  for (int k = 0; k < c->nranks; ++k)
    if (k != c->rank) pa.y[pa.n++] = peer->peer_y[k] + b0;
  bool fused = false;
  lb_status_t st = spmv_impl(A_local, sched, d_x_full, peer->y + b0, flags, S(stream), nullptr,
                             pa.n > 0 && sched == LB_SCHED_MERGE_PATH ? &pa : nullptr, &fused);
  if (st != LB_OK) return st;
  if (c->nranks == 1) return LB_OK;
  if (!fused) return lb_allgather_rows(c, h_bounds, peer->y, stream);  // no fused kernel: NCCL exchange
  return peer_barrier(peer, S(stream));
}

lb_status_t lb_spmv_multi(lb_csr_t A_local, lb_comm_t c, lb_schedule_t sched, const int64_t* h_bounds,
                          const float* d_x_full, float* d_y_full, void* stream) {
  return lb_spmv_multi_ex(A_local, c, sched, h_bounds, d_x_full, d_y_full, 0u, stream);
}

// lb_spmv_multi_ex(LB_SPMV_CHUNKED): the rank's hot-plan merge-path SpMV as tile-range launches cut at
// clean coordinates (ensure_chunks); as soon as chunk c is done on every rank, an NCCL group of
// broadcasts (root k sends its chunk c rows) runs on the handle's exchange stream while chunk c+1
// computes (the sub-shard overlap).  Every rank learns every rank's cut rows once
// (a group of int32 broadcasts); ranks with fewer clean cuts send empty chunks.
lb_status_t multi_chunked(lb_csr_s* A, lb_comm_s* c, lb_schedule_t sched, const int64_t* h_bounds,
                          const float* d_x_full, float* d_y_full, uint32_t flags, stream_t s) {
  lb_status_t st;
  const int64_t b0 = h_bounds[c->rank];
  float* y_loc = d_y_full + b0;
  // a rank that cannot run the chunked kernel (no plan, other schedule, empty shard) computes its rows
  // in one call and sends them as chunk 0, so every rank issues the same collectives
  const bool chunkable = sched == LB_SCHED_MERGE_PATH && hot_usable(A) && A->rows > 0;
  if (chunkable) {
    const bool repart = !A->coords_valid || A->coords_kind != 0 || A->coords_L != A->L || (flags & LB_SPMV_REPARTITION);
    if ((st = launch_partition_xhot(A, A->L, repart, d_x_full, s)) != LB_OK) return st;
    if (repart) { A->coords_valid = true; A->coords_L = A->L; A->coords_kind = 0; }
    if ((st = ensure_chunks(A, s)) != LB_OK) return st;
  } else if (A->rows > 0) {
    if ((st = spmv_impl(A, sched, d_x_full, y_loc, flags, s, nullptr)) != LB_OK) return st;
  }
  constexpr int K1 = kChunks + 1;
  if (!A->mc_stream) {
    LB_CUDA(cudaStreamCreateWithFlags(&A->mc_stream, cudaStreamNonBlocking));
    LB_CUDA(cudaEventCreateWithFlags(&A->mc_done, cudaEventDisableTiming));
    for (auto& e : A->ch_ev)
      if (!e) LB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  if (A->mc_comm != (const void*)c || A->mc_L != A->L || A->mc_gen != A->plan_gen ||
      (int)A->mc_rows.size() != c->nranks * K1) {
    int32_t mine[K1];
    for (int k = 0; k < K1; ++k)  // padded with empty chunks
      mine[k] = chunkable ? (int32_t)A->ch_i[std::min(k, A->ch_n)] : (k == 0 ? 0 : (int32_t)A->rows);
    int32_t* d_all = nullptr;
    if (cudaMalloc(&d_all, (size_t)c->nranks * K1 * 4) != cudaSuccess) { cudaGetLastError(); return fail(LB_ERR_OOM, "cuts"); }
    struct Free { int32_t* p; ~Free() { cudaFree(p); } } free_all{d_all};
    LB_CUDA(cudaMemcpyAsync(d_all + (size_t)c->rank * K1, mine, sizeof mine, cudaMemcpyHostToDevice, s));
    LB_NCCL(g_nccl.GroupStart());
    for (int k = 0; k < c->nranks; ++k) {
      nccl_result_t r = g_nccl.Broadcast(d_all + (size_t)k * K1, d_all + (size_t)k * K1, K1, kNcclInt32, k, c->comm, s);
      if (r != 0) { g_nccl.GroupEnd(); return fail(LB_ERR_NCCL, "ncclBroadcast: %s", g_nccl.GetErrorString(r)); }
    }
    LB_NCCL(g_nccl.GroupEnd());
    std::vector<int32_t> all((size_t)c->nranks * K1);
    LB_CUDA(cudaMemcpyAsync(all.data(), d_all, all.size() * 4, cudaMemcpyDeviceToHost, s));
    LB_CUDA(cudaStreamSynchronize(s));
    A->mc_rows.assign(all.begin(), all.end());
    A->mc_comm = c;
    A->mc_L = A->L;
    A->mc_gen = A->plan_gen;
  }
  for (int ch = 0; ch < kChunks; ++ch) {
    if (chunkable && ch < A->ch_n) {
      A->tr_t0 = A->ch_t[ch];
      A->tr_t1 = A->ch_t[ch + 1];
      st = hot_launch(A, d_x_full, y_loc, s);
      A->tr_t0 = 0;
      A->tr_t1 = -1;
      if (st != LB_OK) return st;
    }
    LB_CUDA(cudaEventRecord(A->ch_ev[ch], s));
    LB_CUDA(cudaStreamWaitEvent(A->mc_stream, A->ch_ev[ch], 0));
    LB_NCCL(g_nccl.GroupStart());
    for (int k = 0; k < c->nranks; ++k) {
      const int64_t r0 = A->mc_rows[(size_t)k * K1 + ch], r1 = A->mc_rows[(size_t)k * K1 + ch + 1];
      if (r1 <= r0) continue;
      float* p = d_y_full + h_bounds[k] + r0;
      nccl_result_t r = g_nccl.Broadcast(p, p, (size_t)(r1 - r0), kNcclFloat32, k, c->comm, A->mc_stream);
      if (r != 0) { g_nccl.GroupEnd(); return fail(LB_ERR_NCCL, "ncclBroadcast: %s", g_nccl.GetErrorString(r)); }
    }
    LB_NCCL(g_nccl.GroupEnd());
  }
  LB_CUDA(cudaEventRecord(A->mc_done, A->mc_stream));
  LB_CUDA(cudaStreamWaitEvent(s, A->mc_done, 0));
  nccl_result_t ar = 0;
  LB_NCCL(g_nccl.CommGetAsyncError(c->comm, &ar));
  if (ar != 0) return fail(LB_ERR_NCCL, "NCCL async error: %s", g_nccl.GetErrorString(ar));
  return LB_OK;
}

lb_status_t lb_spmv_multi_ex(lb_csr_t A_local, lb_comm_t c, lb_schedule_t sched, const int64_t* h_bounds,
                             const float* d_x_full, float* d_y_full, uint32_t flags, void* stream) {
  g_err.clear();
  if (!A_local || !c || !h_bounds || !d_x_full || !d_y_full) return fail(LB_ERR_INVALID_ARG, "null argument");
  if ((const void*)d_x_full == (const void*)d_y_full) return fail(LB_ERR_INVALID_ARG, "x and y must not alias");
  const int64_t b0 = h_bounds[c->rank], b1 = h_bounds[c->rank + 1];
  if (b1 - b0 != A_local->rows)
    return fail(LB_ERR_INVALID_ARG, "local shard has %lld rows, bounds say %lld", (long long)A_local->rows,
                (long long)(b1 - b0));
  for (int k = 0; k < c->nranks; ++k)
    if (h_bounds[k + 1] < h_bounds[k]) return fail(LB_ERR_INVALID_ARG, "bounds not monotone at %d", k);
  if (flags & LB_SPMV_CHUNKED) return multi_chunked(A_local, c, sched, h_bounds, d_x_full, d_y_full, flags, S(stream));
  lb_status_t st = spmv_impl(A_local, sched, d_x_full, d_y_full + b0, flags, S(stream), nullptr);
  if (st != LB_OK) return st;
  return lb_allgather_rows(c, h_bounds, d_y_full, stream);
}

}  // extern "C"
