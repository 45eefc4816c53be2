// lb_host.cu -- the host-buffer calls of liblb: lb_spmv_host (whole CSR uploaded per call),
// lb_spmv_host_x (resident matrix, host x / y; LB_SPMV_CHUNKED overlaps the y download with the next
// chunk's tiles) and lb_spmv_host_x_async / _wait (three staging slots, copies of neighbouring calls
// overlapped).  DESIGN.md 8.  C ABI in include/lb.h.
#include "lb_internal.h"

#include <algorithm>

namespace lbi {

// Clean chunk cuts of A's merge-path tiles at its tile length: for k = 1 .. K-1 the first tile at or
// after k * step whose start coordinate does not split a row (j == off[i]).  Computed on first use,
// after a tile-length or plan change, and when `force` (LB_SPMV_REPARTITION: the row offsets may have
// changed).  The partition must be current.  Synchronises `s` when it computes.
lb_status_t ensure_chunks(lb_csr_s* A, bool force, stream_t s) {
  lb_chunk_state& c = A->chunks;
  if (c.L == A->L && !force) return LB_OK;
  const int64_t T = num_tiles(A->rows, A->nnz, A->L);
  if (!c.d_cuts) {
    if (cudaMalloc(&c.d_cuts, 2 * kChunksMax * sizeof(int)) != cudaSuccess) { cudaGetLastError(); return fail(LB_ERR_OOM, "chunks"); }
    if (cudaMallocHost(&c.h_cuts, 2 * kChunksMax * sizeof(int)) != cudaSuccess) { cudaGetLastError(); return fail(LB_ERR_OOM, "chunks"); }
  }
  // a hot tile-kernel launch has `wave` warps and takes ceil(tiles / wave) tiles per warp: cut after
  // q whole waves minus a slack of 32 tiles, so a clean cut found within the slack (a clean start
  // every ~1 + nnz/rows merge items) keeps the chunk at q waves
  const int64_t wave = std::min(A->dev->sm_count * hot_warps(), kMaxCtas), slack = 32;
  const int64_t q = T / ((int64_t)kChunksMax * wave);
  const int64_t step = q >= 1 && q * wave > 4 * slack ? q * wave - slack : T / kChunksMax;
  lb_status_t st = launch_clean_tiles(A, T, kChunksMax, 4096, step, c.d_cuts, s);
  if (st != LB_OK) return st;
  LB_CUDA(cudaMemcpyAsync(c.h_cuts, c.d_cuts, 2 * kChunksMax * sizeof(int), cudaMemcpyDeviceToHost, s));
  LB_CUDA(cudaStreamSynchronize(s));
  const int* h = c.h_cuts;
  int n = 0;
  c.t[0] = 0;
  c.i[0] = 0;
  for (int k = 1; k < kChunksMax; ++k)
    if (h[k] > c.t[n] && h[k] < T) { ++n; c.t[n] = h[k]; c.i[n] = h[kChunksMax + k]; }
  ++n;
  c.t[n] = T;
  c.i[n] = A->rows;
  c.n = n;
  c.L = A->L;
  ++A->cut_gen;
  return LB_OK;
}

lb_status_t ensure_chunk_events(lb_csr_s* A) {
  for (auto& e : A->chunks.ev)
    if (!e) LB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return LB_OK;
}

void destroy_host_state(lb_csr_s* A) {
  lb_host_state& h = A->host;
  if (h.stage) cudaFree(h.stage);
  if (h.mem) {
    if (h.h2d) cudaStreamSynchronize(h.h2d);
    if (h.d2h) cudaStreamSynchronize(h.d2h);
    for (int i = 0; i < kHostSlots; ++i) {
      if (h.xready[i]) cudaEventDestroy(h.xready[i]);
      if (h.done[i]) cudaEventDestroy(h.done[i]);
      if (h.out[i]) cudaEventDestroy(h.out[i]);
    }
    if (h.h2d) cudaStreamDestroy(h.h2d);
    if (h.d2h) cudaStreamDestroy(h.d2h);
    cudaFree(h.mem);
  }
  h = lb_host_state();
  lb_chunk_state& c = A->chunks;
  if (c.d2h) {
    cudaStreamSynchronize(c.d2h);
    cudaStreamDestroy(c.d2h);
    c.d2h = nullptr;
  }
  for (auto& e : c.ev)
    if (e) { cudaEventDestroy(e); e = nullptr; }
  if (c.d_cuts) cudaFree(c.d_cuts);
  if (c.h_cuts) cudaFreeHost(c.h_cuts);
  c.d_cuts = nullptr;
  c.h_cuts = nullptr;
}

namespace {

// LB_SPMV_CHUNKED: the merge-path step with the hot plan as up to kChunksMax tile-kernel launches over
// tile ranges that start and end on clean merge-path coordinates (no row split across a boundary, so
// each launch's rows are final when it ends); the D2H copy of chunk k's rows overlaps chunk k+1.
lb_status_t host_x_chunked(lb_csr_s* A, const float* d_x, float* d_y, float* h_y, uint32_t flags, stream_t s) {
  lb_status_t st;
  const bool force = (flags & LB_SPMV_REPARTITION) != 0;
  if ((st = ensure_partition(A, force, true, d_x, s)) != LB_OK) return st;
  if (!A->chunks.d2h) LB_CUDA(cudaStreamCreateWithFlags(&A->chunks.d2h, cudaStreamNonBlocking));
  if ((st = ensure_chunk_events(A)) != LB_OK) return st;
  if ((st = ensure_chunks(A, force, s)) != LB_OK) return st;
  lb_chunk_state& c = A->chunks;
  for (int k = 0; k < c.n; ++k) {
    c.t0 = c.t[k];
    c.t1 = c.t[k + 1];
    st = hot_launch(A, d_x, d_y, s);
    c.t0 = 0;
    c.t1 = -1;
    if (st != LB_OK) return st;
    LB_CUDA(cudaEventRecord(c.ev[k], s));
    LB_CUDA(cudaStreamWaitEvent(c.d2h, c.ev[k], 0));
    const int64_t r0 = c.i[k], r1 = c.i[k + 1];
    if (r1 > r0) LB_CUDA(cudaMemcpyAsync(h_y + r0, d_y + r0, (size_t)(r1 - r0) * 4, cudaMemcpyDeviceToHost, c.d2h));
  }
  LB_CUDA(cudaStreamSynchronize(c.d2h));
  LB_CUDA(cudaStreamSynchronize(s));
  return LB_OK;
}

}  // namespace
}  // namespace lbi

using namespace lbi;

// ============================================================================ C ABI
extern "C" {

lb_status_t lb_spmv_host_x(lb_csr_t A, lb_schedule_t sched, const float* h_x, float* h_y, uint32_t flags,
                           void* stream) {
  LB_NVTX("lb_spmv_host_x");
  g_err.clear();
  if (!A) return fail(LB_ERR_INVALID_ARG, "null handle");
  if (A->rows == 0) return LB_OK;
  if (!h_y || (!h_x && A->cols > 0)) return fail(LB_ERR_INVALID_ARG, "null host x or y");
  lb_host_state& h = A->host;
  if (!h.stage) {
    void* p = nullptr;
    // x and y separately aligned (256 B) inside one allocation
    if (cudaMalloc(&p, align256((size_t)A->cols * 4) + (size_t)A->rows * 4) != cudaSuccess) {
      cudaGetLastError();
      return fail(LB_ERR_OOM, "lb_spmv_host_x staging");
    }
    h.stage = static_cast<float*>(p);
  }
  stream_t s = S(stream);
  float* d_x = h.stage;
  float* d_y = reinterpret_cast<float*>(reinterpret_cast<char*>(h.stage) + align256((size_t)A->cols * 4));
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
  LB_NVTX("lb_spmv_host_x_async");
  g_err.clear();
  if (!A) return fail(LB_ERR_INVALID_ARG, "null handle");
  if (A->rows == 0) return LB_OK;
  if (!h_y || (!h_x && A->cols > 0)) return fail(LB_ERR_INVALID_ARG, "null host x or y");
  lb_host_state& h = A->host;
  if (!h.mem) {
    const size_t xb = align256((size_t)A->cols * 4), yb = align256((size_t)A->rows * 4);
    void* p = nullptr;
    if (cudaMalloc(&p, kHostSlots * (xb + yb)) != cudaSuccess) {
      cudaGetLastError();
      return fail(LB_ERR_OOM, "lb_spmv_host_x_async staging");
    }
    h.mem = p;
    char* b = static_cast<char*>(p);
    for (int i = 0; i < kHostSlots; ++i) {
      h.x[i] = reinterpret_cast<float*>(b + i * (xb + yb));
      h.y[i] = reinterpret_cast<float*>(b + i * (xb + yb) + xb);
      LB_CUDA(cudaEventCreateWithFlags(&h.xready[i], cudaEventDisableTiming));
      LB_CUDA(cudaEventCreateWithFlags(&h.done[i], cudaEventDisableTiming));
      LB_CUDA(cudaEventCreateWithFlags(&h.out[i], cudaEventDisableTiming));
    }
    LB_CUDA(cudaStreamCreateWithFlags(&h.h2d, cudaStreamNonBlocking));
    LB_CUDA(cudaStreamCreateWithFlags(&h.d2h, cudaStreamNonBlocking));
  }
  const int k = h.next;
  stream_t s = S(stream);
  // x slot k is free once the SpMV of the call kHostSlots back (same slot) has read it
  LB_CUDA(cudaStreamWaitEvent(h.h2d, h.done[k], 0));
  if (A->cols > 0) LB_CUDA(cudaMemcpyAsync(h.x[k], h_x, (size_t)A->cols * 4, cudaMemcpyHostToDevice, h.h2d));
  LB_CUDA(cudaEventRecord(h.xready[k], h.h2d));
  // the SpMV waits for its x and for y slot k to have been copied out by the call kHostSlots back
  LB_CUDA(cudaStreamWaitEvent(s, h.xready[k], 0));
  LB_CUDA(cudaStreamWaitEvent(s, h.out[k], 0));
  lb_status_t st = spmv_impl(A, sched, h.x[k], h.y[k], flags, s, nullptr);
  if (st != LB_OK) return st;
  LB_CUDA(cudaEventRecord(h.done[k], s));
  LB_CUDA(cudaStreamWaitEvent(h.d2h, h.done[k], 0));
  LB_CUDA(cudaMemcpyAsync(h_y, h.y[k], (size_t)A->rows * 4, cudaMemcpyDeviceToHost, h.d2h));
  LB_CUDA(cudaEventRecord(h.out[k], h.d2h));
  h.next = (k + 1) % kHostSlots;
  return LB_OK;
}

lb_status_t lb_spmv_host_x_wait(lb_csr_t A) {
  LB_NVTX("lb_spmv_host_x_wait");
  g_err.clear();
  if (!A) return fail(LB_ERR_INVALID_ARG, "null handle");
  if (!A->host.mem) return LB_OK;
  LB_CUDA(cudaStreamSynchronize(A->host.h2d));
  LB_CUDA(cudaStreamSynchronize(A->host.d2h));
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
  LB_NVTX("lb_spmv_host");
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
  if (A.bins.mem) cudaFree(A.bins.mem);  // the transient handle's lazily allocated workspace
  return LB_OK;
}

}  // extern "C"
