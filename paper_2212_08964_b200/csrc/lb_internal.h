// lb_internal.h -- host-side internals shared by the translation units of liblb.so.
// The C ABI is declared (and documented) in include/lb.h; this header holds the handle layout, the
// error / launch bookkeeping and the launch helpers one unit provides to another.
//
//   lb_core.cu      errors, device info, handle create / destroy / validate, partitions, AUTO
//   lb_spmv.cu      the SpMV schedules: tile-kernel launches (merge-path, nonzero-split), row-granular
//                   kernels, binning, the phase timer and the ceiling probes
//   lb_plan.cu      the x-reuse plan (build, drop, query)
//   lb_host.cu      host-buffer calls (lb_spmv_host, lb_spmv_host_x[_async], LB_SPMV_CHUNKED)
//   lb_multi.cu     multi-GPU: NCCL (dlopen), shard bounds, the exchange schedule, peers, checksums
//   lb_spmm.cu      SpMM (NEXT-2)
//   lb_sssp.cu      SSSP (NEXT-4)
// All compute runs in the kernels of the k_*.cuh headers; there is no CPU fallback.
#pragma once
#include "lb.h"

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

namespace lbi {

// NVTX ranges around the public entry points (compute / exchange overlap is read off an nsys
// timeline); header-only NVTX v3, a no-op unless a tool injects itself.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define LB_NVTX(name) ::lbi::NvtxRange lb_nvtx_range_(name)


using stream_t = cudaStream_t;
inline stream_t S(void* s) { return reinterpret_cast<stream_t>(s); }

// ----------------------------------------------------------------------------- errors, launches
extern thread_local std::string g_err;
extern std::atomic<uint64_t> g_launches;
lb_status_t fail(lb_status_t st, const char* fmt, ...);

#define LB_CUDA(call)                                                                               \
  do {                                                                                              \
    cudaError_t e_ = (call);                                                                        \
    if (e_ != cudaSuccess) return ::lbi::fail(LB_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

#define LB_LAUNCHED()                                                                                  \
  do {                                                                                                 \
    ::lbi::g_launches.fetch_add(1, std::memory_order_relaxed);                                         \
    cudaError_t e_ = cudaGetLastError();                                                               \
    if (e_ != cudaSuccess) return ::lbi::fail(LB_ERR_CUDA, "kernel launch (%s:%d): %s", __FILE__, __LINE__, \
                                              cudaGetErrorString(e_));                                 \
  } while (0)

// ----------------------------------------------------------------------------- constants
constexpr int kNT = 256;
// rows + nnz limit: int32 indices with 2^16 of headroom for the rounds / tiles that overshoot the last
// nonzero inside the kernels' int32 position arithmetic (reading R13)
constexpr int64_t kMaxMergeItems = (1ll << 31) - (1ll << 16) - 1;
constexpr int kMaxCtas = 8192;             // carry slots per handle (>= SMs x resident CTAs or warps)
constexpr int kCarryVals = 32 * kMaxCtas;  // carry values per handle (SpMM: up to 32 per carry slot)
constexpr int64_t kWarpSearchMax = 32768;  // partitions of <= this many boundaries: a lane group per search
constexpr int kMinTile = 504;              // smallest supported L: sizes the partition cache

// Merge-path tile lengths L = 256*R - 8 (warp-streamed tiles of R rounds) or NT*E - 8 (CTA tiles):
// a tile's 32-byte-aligned nonzero range spans <= L + 7, so every lane gets the same slots (R17).
constexpr int kNumL = 5;
constexpr int kTileL[kNumL] = {504, 1016, 2040, 3064, 4088};
inline int l_index(int L) {
  for (int i = 0; i < kNumL; ++i)
    if (kTileL[i] == L) return i;
  return -1;
}
constexpr int kNzL = 1016;       // nonzero-split tile (nonzeros per tile)
constexpr int kChunksMax = 8;    // LB_SPMV_CHUNKED: tile-range launches per call
constexpr int kMaxPeers = 7;     // fused epilogue: other ranks of one 8-GPU node

inline int64_t num_tiles(int64_t rows, int64_t nnz, int64_t L) { return (rows + nnz + L - 1) / L; }
inline int64_t num_tiles_nz(int64_t nnz, int64_t L) { return nnz > 0 ? (nnz + L - 1) / L : 1; }
inline size_t align256(size_t n) { return (n + 255) & ~size_t(255); }

// ----------------------------------------------------------------------------- device info
struct DeviceInfo {
  int sm_count = 0;
  int l2_bytes = 0;
};
lb_status_t device_info(int dev, const DeviceInfo** out);

// ----------------------------------------------------------------------------- the handle
}  // namespace lbi

// x-reuse plan (lb_csr_plan_hot_x; one device allocation at `mem`)
struct lb_plan_state {
  void* mem = nullptr;
  int32_t* hcol = nullptr;      // [nnz] col_idx with hot entries replaced by ~slot, warm by cols + w
  int32_t* hot_cols = nullptr;  // [hot_n] slot -> column
  float* x_hot = nullptr;       // [hot_n4 * 4] x of the hot columns, gathered every call
  int hot_n = 0;                // planned hot columns (0: no plan)
  int hot_n4 = 0;               // ceil(hot_n / 4)
  int64_t hot_nnz = 0;          // stored entries in hot columns
  int32_t* warm_cols = nullptr; // [warm_n] warm index -> column (ascending)
  float* x_warm = nullptr;      // [warm_n] x of the warm columns, gathered every call
  int warm_n = 0;
  int64_t warm_nnz = 0;
  bool compact = false;         // warm_cols = -2: every referenced non-hot column is warm; the tile
                                // kernel gathers from the dense x_warm as its x (TIER 1 path)
  unsigned* wmask = nullptr;    // compact: [ceil(cols/32)] bit c = column c is warm
  int* wbase = nullptr;         // compact: [ceil(cols/32)] warm index of the word's first warm column
  int gen = 0;                  // bumped by every build / drop (keys caches derived from the plan)
};

// LB_SPMV_CHUNKED: clean tile-range cuts of the merge-path tiles and the launch range of the next
// tile-kernel call
struct lb_chunk_state {
  int L = 0, n = 0;                  // tile length the cuts were computed for (0: none), chunks
  int64_t t[lbi::kChunksMax + 1] = {};  // first tile of chunk k (t[n] = T)
  int64_t i[lbi::kChunksMax + 1] = {};  // first row of chunk k (i[n] = rows)
  int64_t t0 = 0, t1 = -1;           // tile range of the next tile-kernel launch (t1 < 0: all tiles)
  int* d_cuts = nullptr;             // [2 * kChunksMax] device output of the cut kernel (first use)
  int* h_cuts = nullptr;             // [2 * kChunksMax] pinned host copy
  cudaStream_t d2h = nullptr;        // lb_spmv_host_x: y rows of finished chunks to the host
  cudaEvent_t ev[lbi::kChunksMax] = {};  // chunk k done (created on first chunked use)
};

// host-buffer calls (lb_spmv_host_x, lb_spmv_host_x_async)
// lb_spmv_host_x_async staging slots: with 3, a call's SpMV never waits for the D2H of the call two
// back (2 slots: 1.57 ms per C3 step, bound by SpMV + D2H of alternate calls; 3 slots: the H2D
// stream alone, 64 MB at ~48 GB/s when both directions run)
constexpr int kHostSlots = 3;
struct lb_host_state {
  float* stage = nullptr;  // lb_spmv_host_x: [cols | rows] device staging (x, then y)
  void* mem = nullptr;     // _async: kHostSlots staging slots [x | y]
  float* x[kHostSlots] = {};
  float* y[kHostSlots] = {};
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t xready[kHostSlots] = {};  // x of the slot is on the device
  cudaEvent_t done[kHostSlots] = {};    // the slot's SpMV finished (x slot reusable)
  cudaEvent_t out[kHostSlots] = {};     // the slot's y reached the host (y slot reusable)
  int next = 0;
};

// lb_spmv_multi_ex(LB_SPMV_CHUNKED): every rank's chunk cut rows, exchanged once per key
struct lb_multi_state {
  std::vector<int64_t> rows;   // [nranks][kChunksMax + 1] local cut rows of every rank
  const void* comm = nullptr;  // key: communicator, tile length, plan generation, cut generation
  int L = 0, plan_gen = -1, cut_gen = -1;
  cudaStream_t stream = nullptr;  // exchange stream
  cudaEvent_t done = nullptr;
};

// SSSP workspace (lb_sssp; allocated on first use)
struct lb_sssp_state {
  void* mem = nullptr;
  int* q_a = nullptr;     // [rows] frontier lists (ping-pong)
  int* q_b = nullptr;
  int* stamp = nullptr;   // [rows] round of the last push
  int* fo = nullptr;      // [rows + 1] frontier degree prefix (merge-path)
  int* bsum = nullptr;    // scan block sums
  int* counts = nullptr;  // [4] frontier size, next size, negative-weight flag
  int* tc = nullptr;      // tile boundaries of a merge-path round
};

// BINNING workspace (allocated on first use): [CTA | warp | thread] bin row ids, per-block counts
struct lb_bin_state {
  void* mem = nullptr;
  int* ids = nullptr;     // [rows]
  int* counts = nullptr;  // [3 * nb] counts, then write offsets
  int* sizes = nullptr;   // [3]
};

// lb_csr_trace_phases: per-call phase events of the next `cap` SpMV calls (bench.py's timed region)
struct lb_trace_state {
  std::vector<cudaEvent_t> ev;  // [cap][4]: start, partition done, main kernel done, fix-up done
  int cap = 0, n = 0;
};

struct lb_csr_s {
  int64_t rows = 0, cols = 0, nnz = 0;
  const int32_t* off = nullptr;
  const int32_t* col = nullptr;
  const float* val = nullptr;
  int device = 0;
  const lbi::DeviceInfo* dev = nullptr;
  bool vec = true;     // col/val 16-byte aligned -> 128-bit loads (fallback tile kernel)
  bool vec32 = true;   // col/val 32-byte aligned -> 256-bit loads (warp-streamed / CTA-tile kernels)
  int L = LB_DEFAULT_ITEMS_PER_TILE;
  // partition cache
  bool coords_valid = false;
  int coords_L = 0;     // tile length the cached partition was computed for
  int coords_kind = 0;  // 0: merge-path, 1: nonzero-split
  int cut_gen = 0;      // bumped whenever the chunk cuts are recomputed
  bool owns_scratch = true;
  int2* coords = nullptr;      // partition cache [(T_max+1)]
  int* carry_row = nullptr;    // [kMaxCtas]
  float* carry_val = nullptr;  // [kCarryVals]
  int* flags = nullptr;        // [4] validation flags
  unsigned* ticket = nullptr;  // [1] last-CTA ticket of the tile kernels (kept at 0 between launches)
  int max_row = -1;            // longest row (LB_SCHED_AUTO), -1 until computed
  lb_plan_state plan;
  lb_chunk_state chunks;
  lb_host_state host;
  lb_multi_state multi;
  lb_sssp_state sssp;
  lb_bin_state bins;
  lb_trace_state trace;
};

namespace lbi {

// ----------------------------------------------------------------------------- helpers across units
// lb_core.cu
size_t scratch_bytes(int64_t rows, int64_t nnz);
void carve_scratch(lb_csr_s* A, char* p);
int auto_tile_length(int64_t rows, int64_t nnz);
lb_status_t check_shape(int64_t rows, int64_t cols, int64_t nnz);
lb_status_t init_handle(lb_csr_s* A, int64_t rows, int64_t cols, int64_t nnz, const int32_t* off,
                        const int32_t* col, const float* val);
int offsets_l2_resident(const lb_csr_s* A);
lb_status_t launch_partition(const lb_csr_s* A, int64_t L, int2* coords, stream_t s);
lb_status_t launch_partition_nz(const lb_csr_s* A, int64_t L, int2* coords, stream_t s);
// partition (when `partition`) and the x-reuse plan's per-call gathers of x, in one launch
lb_status_t launch_partition_xhot(const lb_csr_s* A, int64_t L, bool partition, const float* x, stream_t s);
lb_status_t launch_clean_tiles(const lb_csr_s* A, int64_t T, int K, int span, int64_t step, int* d_out, stream_t s);
lb_status_t select_schedule(lb_csr_s* A, stream_t s, lb_schedule_t* out);
// merge-path partition of the handle at its L: (re)computed when stale or when `force`
lb_status_t ensure_partition(lb_csr_s* A, bool force, bool with_plan_gathers, const float* x, stream_t s);

// lb_spmv.cu
struct PhaseEvents {
  cudaEvent_t ev[4];
};
// Peer targets of the fused multi-GPU epilogue: the other ranks' y, already offset to this rank's first row.
struct PeerArgs {
  float* y[kMaxPeers];
  int n = 0;
};
lb_status_t spmv_impl(lb_csr_s* A, lb_schedule_t sched, const float* x, float* y, uint32_t flags, stream_t s,
                      PhaseEvents* pe, const PeerArgs* pa = nullptr, bool* fused = nullptr);
// the plan's tile kernel over A->chunks' tile range (all tiles when t1 < 0); the plan's gathers
// must have run for this x (launch_partition_xhot)
lb_status_t hot_launch(lb_csr_s* A, const float* x, float* y, stream_t s, const PeerArgs* pa = nullptr);
int hot_warps();
inline bool hot_usable(const lb_csr_s* A) {
  return A->plan.hot_n > 0 && A->vec32 && (A->L == 1016 || A->L == 504);
}
const char* merge_kernel_name(const lb_csr_s* A, char* buf, size_t n);

// lb_plan.cu
void drop_plan(lb_csr_s* A);

// lb_host.cu
// LB_SPMV_CHUNKED cuts of the handle's merge-path tiles (the partition must be current); recomputed
// when stale or when `force`.  Synchronises `s` when it computes.
lb_status_t ensure_chunks(lb_csr_s* A, bool force, stream_t s);
lb_status_t ensure_chunk_events(lb_csr_s* A);
void destroy_host_state(lb_csr_s* A);

// lb_multi.cu
void destroy_multi_state(lb_csr_s* A);

}  // namespace lbi
