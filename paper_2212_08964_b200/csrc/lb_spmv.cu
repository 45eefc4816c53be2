// lb_spmv.cu -- the SpMV schedules of liblb (arXiv 2212.08964 Ch.3-4): merge-path tile processors
// (a3 + a4) with and without the x-reuse plan, nonzero-split, thread / group / warp-mapped, binning,
// the per-phase timer and the stream / stream+gather ceiling probes.  C ABI in include/lb.h.
#include "k_merge.cuh"
#include "k_rowmapped.cuh"
#include "lb_internal.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>

namespace lbi {

static_assert(kMaxPeers == lbk::kMaxPeers, "peer count");

namespace {

// Shared-memory carve-out: the smallest that still fits `blocks` CTAs with `smem_per_cta` bytes, so
// the rest of the 256 KB stays L1 (the gathers' in-flight misses need it).
template <typename K>
lb_status_t set_carveout(K k, int threads, size_t dyn, int* blocks) {
  cudaFuncAttributes fa;
  LB_CUDA(cudaFuncGetAttributes(&fa, k));
  LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, k, threads, dyn));
  const double need = (double)(*blocks) * (fa.sharedSizeBytes + dyn + 1024.0);
  const int pct = std::min(100, std::max(1, (int)(100.0 * need / (228.0 * 1024.0)) + 1));
  LB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
  LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, k, threads, dyn));
  *blocks = std::max(1, *blocks);
  return LB_OK;
}

// per-device, per-kernel resident CTAs per SM (0 = not configured yet)
struct OccCache {
  std::mutex mu;
  int blocks[64] = {0};
};

template <typename K>
lb_status_t resident_ctas(OccCache& c, int dev, K k, int threads, size_t dyn, int* blocks) {
  std::lock_guard<std::mutex> g(c.mu);
  if (c.blocks[dev] == 0) {
    lb_status_t st = set_carveout(k, threads, dyn, &c.blocks[dev]);
    if (st != LB_OK) return st;
  }
  *blocks = c.blocks[dev];
  return LB_OK;
}

lbk::TileArgs tile_args(const lb_csr_s* A, const int32_t* col, const float* x, float* y, int T, int per) {
  lbk::TileArgs a = {};
  a.off = A->off; a.col = col; a.val = A->val; a.x = x; a.y = y;
  a.coords = A->coords; a.rows = (int)A->rows; a.nnz = (int)A->nnz;
  a.num_tiles = T; a.tiles_per_cta = per;
  a.carry_row = A->carry_row; a.carry_val = A->carry_val; a.ticket = A->ticket;
  a.cols = (int)A->cols;
  a.off_keep = offsets_l2_resident(A);
  return a;
}

void set_peers(lbk::TileArgs& a, const PeerArgs* pa) {
  a.npeers = pa ? pa->n : 0;
  for (int p = 0; p < lbk::kMaxPeers; ++p) a.peer_y[p] = pa && p < pa->n ? pa->y[p] : nullptr;
}

// launch with programmatic dependent launch after the partition kernel (PDL: the tile kernel's
// prologue overlaps the partition's tail; it waits on griddepcontrol.wait before reading coords)
template <typename K>
lb_status_t launch_pdl(K k, int grid, int threads, size_t dyn, stream_t s, const lbk::TileArgs& a) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  LB_CUDA(cudaLaunchKernelEx(&cfg, k, a));
  LB_LAUNCHED();
  return LB_OK;
}

// ----------------------------------------------------------------------------- plain-CSR tile kernels
// Warp-streamed tiles (merge_stream_kernel, L = 256*R - 8): persistent grid of SMs x resident CTAs of
// W warps; warp w owns ceil(T / warps) consecutive tiles.
template <int W, int R, int MINB>
lb_status_t stream_launch(lb_csr_s* A, const float* x, float* y, stream_t s) {
  auto k = lbk::merge_stream_kernel<W, R, MINB>;
  static OccCache occ;
  int blocks = 0;
  lb_status_t st = resident_ctas(occ, A->device, k, W * 32, 0, &blocks);
  if (st != LB_OK) return st;
  constexpr int L = 256 * R - 8;
  const int T = (int)num_tiles(A->rows, A->nnz, L);
  const int warps_max = std::min(A->dev->sm_count * blocks * W, kMaxCtas);
  const int tpw = (T + warps_max - 1) / warps_max;
  const int warps = (T + tpw - 1) / tpw;
  const int grid = (warps + W - 1) / W;
  return launch_pdl(k, grid, W * 32, 0, s, tile_args(A, A->col, x, y, T, tpw));
}

// CTA tiles (merge_wide_kernel, L = NT*E - 8): short rows (C2 stencil) and long tiles.
template <int NT, int E, int MINB>
lb_status_t wide_launch(lb_csr_s* A, const float* x, float* y, stream_t s) {
  auto k = lbk::merge_wide_kernel<NT, E, MINB>;
  static OccCache occ;
  int blocks = 0;
  lb_status_t st = resident_ctas(occ, A->device, k, NT, 0, &blocks);
  if (st != LB_OK) return st;
  constexpr int L = NT * E - 8;
  const int T = (int)num_tiles(A->rows, A->nnz, L);
  int grid = std::min(T, std::min(A->dev->sm_count * blocks, kMaxCtas));
  const int tpc = (T + grid - 1) / grid;
  grid = (T + tpc - 1) / tpc;  // every CTA owns >= 1 tile
  return launch_pdl(k, grid, NT, 0, s, tile_args(A, A->col, x, y, T, tpc));
}

// Short-row CTA tiles (merge_rows_kernel, L = 8*NT - 8): products staged in shared memory, rows
// summed one per thread.
template <int NT, int MINB>
lb_status_t rows_launch(lb_csr_s* A, const float* x, float* y, stream_t s) {
  auto k = lbk::merge_rows_kernel<NT, MINB>;
  static OccCache occ;
  int blocks = 0;
  lb_status_t st = resident_ctas(occ, A->device, k, NT, 0, &blocks);
  if (st != LB_OK) return st;
  constexpr int L = 8 * NT - 8;
  const int T = (int)num_tiles(A->rows, A->nnz, L);
  int grid = std::min(T, std::min(A->dev->sm_count * blocks, kMaxCtas));
  const int tpc = (T + grid - 1) / grid;
  grid = (T + tpc - 1) / tpc;  // every CTA owns >= 1 tile
  return launch_pdl(k, grid, NT, 0, s, tile_args(A, A->col, x, y, T, tpc));
}

// Fallback for col_idx / values that are not 32-byte aligned: CTA tiles with 128-bit (16-byte
// aligned) or scalar loads, and a separate fix-up kernel.
template <int L, bool VEC>
lb_status_t fallback_launch(lb_csr_s* A, const float* x, float* y, stream_t s, PhaseEvents* pe) {
  auto k = lbk::merge_tile_kernel<kNT, L, VEC>;
  constexpr size_t smem = sizeof(typename lbk::MergeCfg<kNT, L, VEC>::Smem);
  static OccCache occ;
  int blocks = 0;
  {
    std::lock_guard<std::mutex> g(occ.mu);
    if (occ.blocks[A->device] == 0) {
      LB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ.blocks[A->device], k, kNT, smem));
      occ.blocks[A->device] = std::max(1, occ.blocks[A->device]);
    }
    blocks = occ.blocks[A->device];
  }
  const int T = (int)num_tiles(A->rows, A->nnz, L);
  int grid = std::min(T, std::min(A->dev->sm_count * blocks, kMaxCtas));
  const int tpc = (T + grid - 1) / grid;
  grid = (T + tpc - 1) / tpc;
  const lbk::TileArgs a = tile_args(A, A->col, x, y, T, tpc);
  k<<<grid, kNT, smem, s>>>(a);
  LB_LAUNCHED();
  if (pe) LB_CUDA(cudaEventRecord(pe->ev[2], s));
  lbk::fixup_kernel<<<(grid + kNT - 1) / kNT, kNT, 0, s>>>(a, grid);
  LB_LAUNCHED();
  return LB_OK;
}

// The tile processor of each tile length, chosen by measurement.
struct TileKernel {
  const char* name;
  lb_status_t (*launch)(lb_csr_s*, const float*, float*, stream_t);
};
const TileKernel kTileKernels[kNumL] = {
    {"merge_stream_kernel<4,2,4>", stream_launch<4, 2, 4>},      // L = 504
    {"merge_stream_kernel<16,4,1>", stream_launch<16, 4, 1>},    // L = 1016 (long / irregular rows)
    {"merge_rows_kernel<256,4>", rows_launch<256, 4>},           // L = 2040 (short rows: C2 stencil)
    {"merge_stream_kernel<4,12,4>", stream_launch<4, 12, 4>},    // L = 3064
    {"merge_wide_kernel<256,16,2>", wide_launch<256, 16, 2>},    // L = 4088
};

template <int L>
lb_status_t launch_fallback(lb_csr_s* A, const float* x, float* y, stream_t s, PhaseEvents* pe) {
  return A->vec ? fallback_launch<L, true>(A, x, y, s, pe) : fallback_launch<L, false>(A, x, y, s, pe);
}

lb_status_t launch_merge(lb_csr_s* A, const float* x, float* y, stream_t s, PhaseEvents* pe) {
  const int li = l_index(A->L);
  if (li < 0) return fail(LB_ERR_INVALID_ARG, "unsupported tile length %d", A->L);
  if (A->vec32) {
    lb_status_t st = kTileKernels[li].launch(A, x, y, s);
    if (st != LB_OK) return st;
    if (pe) LB_CUDA(cudaEventRecord(pe->ev[2], s));
    return LB_OK;
  }
  switch (A->L) {
    case 504: return launch_fallback<504>(A, x, y, s, pe);
    case 1016: return launch_fallback<1016>(A, x, y, s, pe);
    case 2040: return launch_fallback<2040>(A, x, y, s, pe);
    case 3064: return launch_fallback<3064>(A, x, y, s, pe);
    default: return launch_fallback<4088>(A, x, y, s, pe);
  }
}

// ----------------------------------------------------------------------------- x-reuse plan tile kernels
// Tile kernel with the plan: warp-streamed, one CTA of W warps per SM, x of the hot columns staged
// in dynamic shared memory.  W and the slot budget were chosen by measurement;
// LB_HOT_W overrides W (8, 16) for sweeps.
constexpr int kHotDynMax = 45056 * 4;  // 176 KB (lb_csr_plan_hot_x's slot limit)

template <int W, int R, int TIER, bool PEERS = false>
lb_status_t hot_launch_wr(lb_csr_s* A, const float* x, float* y, stream_t s, const PeerArgs* pa = nullptr) {
  auto k = lbk::merge_stream_kernel<W, R, 1, unsigned short, TIER, PEERS>;
  static std::mutex mu;
  static int conf_dyn[64] = {0};  // dynamic smem size the carve-out was set for, per device
  const int dyn = A->plan.hot_n4 * 16;
  {
    std::lock_guard<std::mutex> g(mu);
    if (conf_dyn[A->device] != dyn) {
      LB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kHotDynMax));
      cudaFuncAttributes fa;
      LB_CUDA(cudaFuncGetAttributes(&fa, k));
      const double need = (double)fa.sharedSizeBytes + dyn + 1024.0;
      const int pct = std::min(100, std::max(1, (int)(100.0 * need / (228.0 * 1024.0)) + 1));
      LB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
      int blocks = 0;
      LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k, W * 32, dyn));
      if (blocks < 1) return fail(LB_ERR_UNSUPPORTED, "hot tile kernel does not fit with %d bytes of x_hot", dyn);
      conf_dyn[A->device] = dyn;
    }
  }
  constexpr int L = 256 * R - 8;
  const bool ranged = A->chunks.t1 >= 0;  // LB_SPMV_CHUNKED: tiles [t0, t1) only
  const int T = ranged ? (int)(A->chunks.t1 - A->chunks.t0) : (int)num_tiles(A->rows, A->nnz, L);
  if (T <= 0) return LB_OK;
  const int warps_max = std::min(A->dev->sm_count * W, kMaxCtas);
  const int tpw = (T + warps_max - 1) / warps_max;
  const int warps = (T + tpw - 1) / tpw;
  const int grid = (warps + W - 1) / W;
  lbk::TileArgs a = tile_args(A, A->plan.hcol, x, y, T, tpw);
  a.coords = A->coords + (ranged ? A->chunks.t0 : 0);
  a.x_hot = A->plan.x_hot; a.hot_n4 = A->plan.hot_n4;
  a.x_warm = A->plan.x_warm;
  set_peers(a, pa);
  return launch_pdl(k, grid, W * 32, (size_t)dyn, s, a);
}

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

// Fused epilogue without a plan: the warp-streamed kernel at L = 1016 (8 warps, 2 CTAs per SM, the
// plain default) or L = 504, with peer stores.
template <int R>
lb_status_t peers_stream_launch(lb_csr_s* A, const float* x, float* y, stream_t s, const PeerArgs* pa) {
  constexpr int W = 8, MINB = 2;
  auto k = lbk::merge_stream_kernel<W, R, MINB, unsigned short, 0, true>;
  static OccCache occ;
  int blocks = 0;
  lb_status_t st = resident_ctas(occ, A->device, k, W * 32, 0, &blocks);
  if (st != LB_OK) return st;
  constexpr int L = 256 * R - 8;
  const int T = (int)num_tiles(A->rows, A->nnz, L);
  const int warps_max = std::min(A->dev->sm_count * blocks * W, kMaxCtas);
  const int tpw = (T + warps_max - 1) / warps_max;
  const int warps = (T + tpw - 1) / tpw;
  const int grid = (warps + W - 1) / W;
  lbk::TileArgs a = tile_args(A, A->col, x, y, T, tpw);
  set_peers(a, pa);
  return launch_pdl(k, grid, W * 32, 0, s, a);
}

// ----------------------------------------------------------------------------- nonzero-split
// tiles of kNzL nonzeros on the warp-streamed processor with 32-bit row ids (a tile may hold any
// number of rows)
lb_status_t launch_nz_tiles(lb_csr_s* A, const float* x, float* y, stream_t s) {
  constexpr int W = 8, R = 4, MINB = 2;
  static_assert(256 * R - 8 == kNzL, "nonzero-split tile");
  auto k = lbk::merge_stream_kernel<W, R, MINB, unsigned>;
  static OccCache occ;
  int blocks = 0;
  lb_status_t st = resident_ctas(occ, A->device, k, W * 32, 0, &blocks);
  if (st != LB_OK) return st;
  const int T = (int)num_tiles_nz(A->nnz, kNzL);
  const int warps_max = std::min(A->dev->sm_count * blocks * W, kMaxCtas);
  const int tpw = (T + warps_max - 1) / warps_max;
  const int warps = (T + tpw - 1) / tpw;
  const int grid = (warps + W - 1) / W;
  return launch_pdl(k, grid, W * 32, 0, s, tile_args(A, A->col, x, y, T, tpw));
}

// ----------------------------------------------------------------------------- binning (Alg.4)
constexpr int kWarpRows = 4;  // WARP_MAPPED: rows per warp

// build the three bins on the device (stable compaction; no host sync)
lb_status_t launch_bins(lb_csr_s* A, stream_t s) {
  lb_bin_state& b = A->bins;
  const int nb = (int)((A->rows + lbk::kBinRows - 1) / lbk::kBinRows);
  if (!b.mem) {
    const size_t bytes = align256((size_t)A->rows * 4) + align256((size_t)3 * nb * 4) + align256(16);
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) { cudaGetLastError(); return fail(LB_ERR_OOM, "binning workspace"); }
    char* q = static_cast<char*>(p);
    b.mem = p;
    b.ids = reinterpret_cast<int*>(q); q += align256((size_t)A->rows * 4);
    b.counts = reinterpret_cast<int*>(q); q += align256((size_t)3 * nb * 4);
    b.sizes = reinterpret_cast<int*>(q);
  }
  lbk::bin_count_kernel<<<nb, 256, 0, s>>>((int)A->rows, A->off, nb, b.counts);
  LB_LAUNCHED();
  lbk::bin_scan_kernel<<<1, 1024, 0, s>>>(nb, b.counts, b.sizes);
  LB_LAUNCHED();
  lbk::bin_scatter_kernel<<<nb, 256, 0, s>>>((int)A->rows, A->off, nb, b.counts, b.ids);
  LB_LAUNCHED();
  return LB_OK;
}

// the three bin kernels (one specialised kernel per bin), persistent grids
lb_status_t launch_bin_kernels(lb_csr_s* A, const float* x, float* y, stream_t s) {
  const int sms = A->dev->sm_count;
  const lb_bin_state& b = A->bins;
  lbk::bin_cta_kernel<<<sms * 8, 256, 0, s>>>(b.ids, b.sizes, A->off, A->col, A->val, x, y);
  LB_LAUNCHED();
  lbk::bin_warp_kernel<<<sms * 8, 256, 0, s>>>(b.ids, b.sizes, A->off, A->col, A->val, x, y);
  LB_LAUNCHED();
  lbk::bin_thread_kernel<<<sms * 16, 256, 0, s>>>(b.ids, b.sizes, A->off, A->col, A->val, x, y);
  LB_LAUNCHED();
  return LB_OK;
}

// ----------------------------------------------------------------------------- probes
// stream+gather ceiling probe (lb_probe_stream_gather); TIER as in the tile kernel
template <int TIER>
lb_status_t probe_launch(lb_csr_s* A, const float* x, stream_t s) {
  auto k = lbk::probe_stream_gather_kernel<TIER>;
  const int dyn = TIER >= 1 ? A->plan.hot_n4 * 16 : 0;
  static std::mutex mu;
  static int conf_dyn[64] = {0};
  static int blocks_cache[64] = {0};  // 0: not configured yet on this device
  int blocks = 0;
  {
    std::lock_guard<std::mutex> g(mu);
    if (blocks_cache[A->device] == 0 || conf_dyn[A->device] != dyn) {
      LB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kHotDynMax));
      const int pct = TIER >= 1 ? std::min(100, (int)(100.0 * (dyn + 1024.0) / (228.0 * 1024.0)) + 1) : 0;
      LB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
      int b = 0;
      LB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, 512, dyn));
      // with a plan: one CTA (16 warps) per SM so x_hot is staged once per SM, as in the tile kernel
      blocks_cache[A->device] = TIER >= 1 ? 1 : std::max(1, b);
      conf_dyn[A->device] = dyn;
    }
    blocks = blocks_cache[A->device];
  }
  const int grid = A->dev->sm_count * blocks;
  k<<<grid, 512, dyn, s>>>((int)A->nnz, TIER >= 1 ? A->plan.hcol : A->col, A->val, x, A->plan.x_hot, A->plan.hot_n4,
                           A->plan.x_warm, (int)A->cols, 0, nullptr);
  LB_LAUNCHED();
  return LB_OK;
}

// cluster hot-tier probe (LB_PROBE_CLUSTER = C in {1, 2, 4, 8}; diagnostic): one CTA of 16
// warps per SM, clusters of C CTAs, as many clusters as fit at once
template <int C>
lb_status_t probe_cluster_launch(lb_csr_s* A, const float* x, stream_t s) {
  auto k = lbk::probe_cluster_gather_kernel<C>;
  const int per = (A->plan.hot_n + C - 1) / C;
  const int dyn = ((per + 3) / 4) * 16;
  LB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kHotDynMax));
  const int pct = std::min(100, (int)(100.0 * (dyn + 1024.0) / (228.0 * 1024.0)) + 1);
  LB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
  if (C > 1) LB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3(A->dev->sm_count / C * C);
  int nclusters = 0;
  LB_CUDA(cudaOccupancyMaxActiveClusters(&nclusters, k, &cfg));
  if (nclusters < 1) return fail(LB_ERR_UNSUPPORTED, "cluster probe C=%d does not fit", C);
  cfg.gridDim = dim3(std::min(nclusters, A->dev->sm_count / C) * C);
  LB_CUDA(cudaLaunchKernelEx(&cfg, k, (int)A->nnz, (const int*)A->plan.hcol, A->val, x, (const float*)A->plan.x_hot,
                             A->plan.hot_n, 0, (float*)nullptr));
  LB_LAUNCHED();
  return LB_OK;
}

template <typename F>
lb_status_t time_reps(F launch, int reps, stream_t s, float* ms_out) {
  lb_status_t st;
  if ((st = launch()) != LB_OK) return st;  // warm-up
  cudaEvent_t e0, e1;
  LB_CUDA(cudaEventCreate(&e0));
  LB_CUDA(cudaEventCreate(&e1));
  cudaEventRecord(e0, s);
  for (int r = 0; r < reps && st == LB_OK; ++r) st = launch();
  cudaEventRecord(e1, s);
  cudaError_t e = cudaEventSynchronize(e1);
  float ms = 0.f;
  if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (st != LB_OK) return st;
  if (e != cudaSuccess) return fail(LB_ERR_CUDA, "probe timing: %s", cudaGetErrorString(e));
  *ms_out = ms / reps;
  return LB_OK;
}

}  // namespace

int hot_warps() {
  const char* env = getenv("LB_HOT_W");
  const int w = env ? atoi(env) : 16;
  return w == 8 ? 8 : 16;
}

lb_status_t hot_launch(lb_csr_s* A, const float* x, float* y, stream_t s, const PeerArgs* pa) {
  if (A->plan.compact) return hot_launch_t<1>(A, A->plan.x_warm, y, s, pa);
  return A->plan.warm_n > 0 ? hot_launch_t<2>(A, x, y, s, pa) : hot_launch_t<1>(A, x, y, s, pa);
}

const char* merge_kernel_name(const lb_csr_s* A, char* buf, size_t n) {
  const int li = l_index(A->L);
  if (li < 0) return "";
  if (hot_usable(A)) {
    snprintf(buf, n, "merge_stream_kernel<%d,%d,1,%s>", hot_warps(), (A->L + 8) / 256,
             A->plan.warm_n > 0 ? "hot+warm" : "hot");
    return buf;
  }
  if (!A->vec32) {
    snprintf(buf, n, "merge_tile_kernel<256,%d> + fixup_kernel", A->L);
    return buf;
  }
  return kTileKernels[li].name;
}

lb_status_t spmv_impl(lb_csr_s* A, lb_schedule_t sched, const float* x, float* y, uint32_t flags, stream_t s,
                      PhaseEvents* pe, const PeerArgs* pa, bool* fused) {
  if (fused) *fused = false;
  if (!A) return fail(LB_ERR_INVALID_ARG, "null handle");
  if (A->rows == 0) return LB_OK;
  if (!y || (!x && A->nnz > 0)) return fail(LB_ERR_INVALID_ARG, "null x or y");
  if ((const void*)x == (const void*)y) return fail(LB_ERR_INVALID_ARG, "x and y must not alias");
  if (sched == LB_SCHED_AUTO) {
    lb_status_t st = select_schedule(A, s, &sched);
    if (st != LB_OK) return st;
  }
  PhaseEvents traced;
  if (!pe && A->trace.n < A->trace.cap) {  // lb_csr_trace_phases: this call's events go to the next slot
    for (int i = 0; i < 4; ++i) traced.ev[i] = A->trace.ev[(size_t)A->trace.n * 4 + i];
    ++A->trace.n;
    pe = &traced;
  }
  if (pe) LB_CUDA(cudaEventRecord(pe->ev[0], s));
  lb_status_t st = LB_OK;
  switch (sched) {
    case LB_SCHED_THREAD_MAPPED: {
      if (pe) LB_CUDA(cudaEventRecord(pe->ev[1], s));
      // Listing 3: blocks of 256 threads, grid = ceil(rows / 256)
      const int64_t grid = (A->rows + kNT - 1) / kNT;
      lbk::thread_mapped_kernel<<<(unsigned)grid, kNT, 0, s>>>((int)A->rows, A->off, A->col, A->val, x, y);
      LB_LAUNCHED();
      break;
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
      break;
    }
    case LB_SCHED_MERGE_PATH: {
      const bool force = (flags & LB_SPMV_REPARTITION) != 0;
      if (hot_usable(A)) {  // hot-column plan: partition + x gathers in one launch, then the hot tile kernel
        if ((st = ensure_partition(A, force, true, x, s)) != LB_OK) return st;
        if (pe) LB_CUDA(cudaEventRecord(pe->ev[1], s));
        if ((st = hot_launch(A, x, y, s, pa)) != LB_OK) return st;
        if (fused) *fused = pa != nullptr;
        break;
      }
      if ((st = ensure_partition(A, force, false, x, s)) != LB_OK) return st;
      if (pe) LB_CUDA(cudaEventRecord(pe->ev[1], s));
      if (pa && A->vec32 && (A->L == 1016 || A->L == 504)) {  // fused epilogue, plain CSR
        st = A->L == 1016 ? peers_stream_launch<4>(A, x, y, s, pa) : peers_stream_launch<2>(A, x, y, s, pa);
        if (st != LB_OK) return st;
        if (fused) *fused = true;
        break;
      }
      if ((st = launch_merge(A, x, y, s, pe)) != LB_OK) return st;
      if (pe) LB_CUDA(cudaEventRecord(pe->ev[3], s));
      return LB_OK;
    }
    case LB_SCHED_WARP_MAPPED: {
      if (pe) LB_CUDA(cudaEventRecord(pe->ev[1], s));
      // an equal share of rows per warp, kWarpRows rows each, with the warps
      // oversubscribed so that the hardware scheduler absorbs the imbalance
      const int64_t rpw = kWarpRows;
      const int64_t grid = ((A->rows + rpw - 1) / rpw * 32 + kNT - 1) / kNT;
      lbk::warp_mapped_kernel<<<(unsigned)grid, kNT, 0, s>>>((int)A->rows, (int)rpw, A->off, A->col, A->val, x, y);
      LB_LAUNCHED();
      break;
    }
    case LB_SCHED_BINNING: {
      if ((st = launch_bins(A, s)) != LB_OK) return st;  // bins depend only on A, rebuilt every call (Alg.4 runtime phase)
      if (pe) LB_CUDA(cudaEventRecord(pe->ev[1], s));
      if ((st = launch_bin_kernels(A, x, y, s)) != LB_OK) return st;
      break;
    }
    case LB_SCHED_NONZERO_SPLIT: {
      if (!A->vec32) return fail(LB_ERR_UNSUPPORTED, "nonzero-split needs 32-byte aligned col_idx/values");
      if (!A->coords_valid || A->coords_kind != 1 || A->coords_L != kNzL || (flags & LB_SPMV_REPARTITION)) {
        if ((st = launch_partition_nz(A, kNzL, A->coords, s)) != LB_OK) return st;
        A->coords_valid = true;
        A->coords_L = kNzL;
        A->coords_kind = 1;
      }
      if (pe) LB_CUDA(cudaEventRecord(pe->ev[1], s));
      if ((st = launch_nz_tiles(A, x, y, s)) != LB_OK) return st;
      break;
    }
    default:
      return fail(LB_ERR_INVALID_ARG, "unknown schedule id %d", (int)sched);
  }
  if (pe) { LB_CUDA(cudaEventRecord(pe->ev[2], s)); LB_CUDA(cudaEventRecord(pe->ev[3], s)); }
  return LB_OK;
}

}  // namespace lbi

using namespace lbi;

// ============================================================================ C ABI
extern "C" {

lb_status_t lb_spmv(lb_csr_t A, lb_schedule_t sched, const float* d_x, float* d_y, void* stream) {
  LB_NVTX("lb_spmv");
  g_err.clear();
  return spmv_impl(A, sched, d_x, d_y, 0u, S(stream), nullptr);
}

lb_status_t lb_spmv_ex(lb_csr_t A, lb_schedule_t sched, const float* d_x, float* d_y, uint32_t flags, void* stream) {
  LB_NVTX("lb_spmv_ex");
  g_err.clear();
  return spmv_impl(A, sched, d_x, d_y, flags, S(stream), nullptr);
}

lb_status_t lb_bins(lb_csr_t A, int32_t* d_ids, int64_t h_sizes[3], void* stream) {
  g_err.clear();
  if (!A || !h_sizes || (!d_ids && A->rows > 0)) return fail(LB_ERR_INVALID_ARG, "bad lb_bins arguments");
  h_sizes[0] = h_sizes[1] = h_sizes[2] = 0;
  if (A->rows == 0) return LB_OK;
  stream_t s = S(stream);
  lb_status_t st;
  if ((st = launch_bins(A, s)) != LB_OK) return st;
  LB_CUDA(cudaMemcpyAsync(d_ids, A->bins.ids, (size_t)A->rows * 4, cudaMemcpyDeviceToDevice, s));
  int h[3];
  LB_CUDA(cudaMemcpyAsync(h, A->bins.sizes, sizeof h, cudaMemcpyDeviceToHost, s));
  LB_CUDA(cudaStreamSynchronize(s));
  for (int q = 0; q < 3; ++q) h_sizes[q] = h[q];
  return LB_OK;
}

lb_status_t lb_spmv_peers(lb_csr_t A, const float* d_x, float* d_y, float* const* h_peer_y, int32_t npeers,
                          uint32_t flags, void* stream) {
  g_err.clear();
  if (!A) return fail(LB_ERR_INVALID_ARG, "null handle");
  if (npeers < 0 || npeers > kMaxPeers) return fail(LB_ERR_INVALID_ARG, "npeers %d not in [0, %d]", npeers, kMaxPeers);
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
    cudaError_t e = cudaEventSynchronize(pe.ev[3]);
    for (int i = 0; i < 3 && e == cudaSuccess; ++i) e = cudaEventElapsedTime(&ms_out[i], pe.ev[i], pe.ev[i + 1]);
    if (e != cudaSuccess) st = fail(LB_ERR_CUDA, "phase timing: %s", cudaGetErrorString(e));
  } else if (st == LB_OK) {
    ms_out[0] = ms_out[1] = ms_out[2] = 0.f;
  }
  for (auto& e : pe.ev) cudaEventDestroy(e);
  return st;
}

lb_status_t lb_csr_trace_phases(lb_csr_t A, int32_t capacity) {
  g_err.clear();
  if (!A || capacity < 0) return fail(LB_ERR_INVALID_ARG, "bad trace arguments");
  lb_trace_state& t = A->trace;
  for (cudaEvent_t e : t.ev) cudaEventDestroy(e);
  t.ev.clear();
  t.cap = t.n = 0;
  if (capacity == 0) return LB_OK;
  t.ev.resize((size_t)capacity * 4, nullptr);
  for (auto& e : t.ev) {
    if (cudaEventCreate(&e) != cudaSuccess) {
      cudaGetLastError();
      e = nullptr;
      for (cudaEvent_t q : t.ev)
        if (q) cudaEventDestroy(q);
      t.ev.clear();
      return fail(LB_ERR_CUDA, "cudaEventCreate (trace)");
    }
  }
  t.cap = capacity;
  return LB_OK;
}

lb_status_t lb_csr_trace_read(lb_csr_t A, int32_t* n_out, float* ms_out) {
  g_err.clear();
  if (!A || !n_out) return fail(LB_ERR_INVALID_ARG, "bad trace arguments");
  lb_trace_state& t = A->trace;
  *n_out = t.n;
  if (t.n > 0) {
    if (!ms_out) return fail(LB_ERR_INVALID_ARG, "null ms_out");
    LB_CUDA(cudaEventSynchronize(t.ev[(size_t)(t.n - 1) * 4 + 3]));
    for (int c = 0; c < t.n; ++c)
      for (int i = 0; i < 3; ++i)
        LB_CUDA(cudaEventElapsedTime(&ms_out[(size_t)c * 3 + i], t.ev[(size_t)c * 4 + i], t.ev[(size_t)c * 4 + i + 1]));
  }
  t.n = 0;
  return LB_OK;
}

lb_status_t lb_probe_stream_gather(lb_csr_t A, const float* d_x, int32_t reps, void* stream, float* ms_out) {
  g_err.clear();
  if (!A || !ms_out || reps < 1 || (!d_x && A->nnz > 0)) return fail(LB_ERR_INVALID_ARG, "bad probe arguments");
  if (!A->vec32) return fail(LB_ERR_UNSUPPORTED, "probe needs 32-byte aligned col_idx/values");
  stream_t s = S(stream);
  const lb_plan_state& p = A->plan;
  const int tier = p.hot_n > 0 ? (p.warm_n > 0 && !p.compact ? 2 : 1) : 0;
  lb_status_t st;
  if (tier > 0 && (st = launch_partition_xhot(A, 0, false, d_x, s)) != LB_OK) return st;  // x_hot / x_warm of this x
  const float* xg = p.compact ? p.x_warm : d_x;
  const char* env = getenv("LB_PROBE_CLUSTER");
  const int ccl = env ? atoi(env) : 0;
  if (ccl > 0 && (tier != 1 || (ccl != 1 && ccl != 2 && ccl != 4 && ccl != 8)))
    return fail(LB_ERR_UNSUPPORTED, "LB_PROBE_CLUSTER needs a hot-only plan and C in {1,2,4,8}");
  auto launch = [&]() {
    if (ccl == 1) return probe_cluster_launch<1>(A, xg, s);
    if (ccl == 2) return probe_cluster_launch<2>(A, xg, s);
    if (ccl == 4) return probe_cluster_launch<4>(A, xg, s);
    if (ccl == 8) return probe_cluster_launch<8>(A, xg, s);
    return tier == 2 ? probe_launch<2>(A, d_x, s) : tier == 1 ? probe_launch<1>(A, xg, s) : probe_launch<0>(A, d_x, s);
  };
  return time_reps(launch, reps, s, ms_out);
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
  return time_reps(launch, reps, s, ms_out);
}

}  // extern "C"
