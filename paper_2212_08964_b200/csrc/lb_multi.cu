// lb_multi.cu -- the multi-GPU layer of liblb (a7; the paper's multi-GPU future work,
// P:2187-2192): equal-nnz row shards, the y exchange between iterated SpMVs over NCCL (dlopen'ed) --
// all-gather(v) as a group of broadcasts, its chunked form overlapped with the SpMV, the padded
// ncclAllGather layout -- the fused peer-store epilogue over CUDA IPC, and the replica checksum of
// SURVEY 8(c) p10.  The exchange schedule is a plain host function (lb_exchange_schedule) used by every
// exchange path, so the CPU tests run the same code at any world size.  C ABI in include/lb.h.
#include "k_multi.cuh"
#include "lb_internal.h"

#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

namespace lbi {
namespace {

// Minimal NCCL ABI (stable since NCCL 2.0).
typedef struct { char internal[128]; } nccl_uid_t;
typedef void* nccl_comm_t;
typedef int nccl_result_t;
constexpr int kNcclUint8 = 1;
constexpr int kNcclInt64 = 4;
constexpr int kNcclUint64 = 5;
constexpr int kNcclFloat32 = 7;
constexpr int kNcclMax = 2;
constexpr int kNcclMin = 3;

struct NcclApi {
  bool loaded = false;
  nccl_result_t (*GetUniqueId)(nccl_uid_t*) = nullptr;
  nccl_result_t (*CommInitRank)(nccl_comm_t*, int, nccl_uid_t, int) = nullptr;
  nccl_result_t (*CommDestroy)(nccl_comm_t) = nullptr;
  nccl_result_t (*Broadcast)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  nccl_result_t (*AllGather)(const void*, void*, size_t, int, nccl_comm_t, cudaStream_t) = nullptr;
  nccl_result_t (*AllReduce)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
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
  SYM("ncclAllGather", AllGather)
  SYM("ncclAllReduce", AllReduce)
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
}  // namespace lbi

struct lb_comm_s {
  lbi::nccl_comm_t comm = nullptr;
  int rank = 0, nranks = 1, device = 0;
  unsigned long long* d_hash = nullptr;  // replica checksum scratch [3]
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

namespace lbi {
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

// every rank's stream passes this point only after every rank reached it (NCCL group of 4-byte
// broadcasts: a broadcast from root k completes on a rank only once rank k issued it)
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

lb_status_t async_error(lb_comm_s* c) {
  nccl_result_t ar = 0;
  LB_NCCL(g_nccl.CommGetAsyncError(c->comm, &ar));
  if (ar != 0) return fail(LB_ERR_NCCL, "NCCL async error: %s", g_nccl.GetErrorString(ar));
  return LB_OK;
}

// One chunk of the exchange: an NCCL group of broadcasts, root k sends y_full[off[k], off[k] + cnt[k]).
lb_status_t broadcast_chunk(lb_comm_s* c, float* d_y_full, const int64_t* off, const int64_t* cnt, stream_t s) {
  LB_NCCL(g_nccl.GroupStart());
  for (int k = 0; k < c->nranks; ++k) {
    if (cnt[k] == 0) continue;
    float* p = d_y_full + off[k];
    nccl_result_t r = g_nccl.Broadcast(p, p, (size_t)cnt[k], kNcclFloat32, k, c->comm, s);
    if (r != 0) { g_nccl.GroupEnd(); return fail(LB_ERR_NCCL, "ncclBroadcast: %s", g_nccl.GetErrorString(r)); }
  }
  LB_NCCL(g_nccl.GroupEnd());
  return LB_OK;
}

lb_status_t check_bounds(int nranks, const int64_t* h_bounds) {
  if (h_bounds[0] != 0) return fail(LB_ERR_INVALID_ARG, "bounds[0] must be 0");
  for (int k = 0; k < nranks; ++k)
    if (h_bounds[k + 1] < h_bounds[k]) return fail(LB_ERR_INVALID_ARG, "bounds not monotone at %d", k);
  return LB_OK;
}

// the handle's LB_SPMV_CHUNKED cut rows padded with empty chunks to K + 1 entries; a handle that cannot
// chunk (no plan, another schedule, empty shard) sends its rows as chunk 0
void padded_cuts(const lb_csr_s* A, bool chunkable, int K, int64_t* out) {
  for (int k = 0; k <= K; ++k)
    out[k] = chunkable ? A->chunks.i[std::min(k, A->chunks.n)] : (k == 0 ? 0 : A->rows);
}

}  // namespace

void destroy_multi_state(lb_csr_s* A) {
  lb_multi_state& m = A->multi;
  if (m.stream) {
    cudaStreamSynchronize(m.stream);
    cudaStreamDestroy(m.stream);
  }
  if (m.done) cudaEventDestroy(m.done);
  m = lb_multi_state();
}

}  // namespace lbi

using namespace lbi;

extern "C" {

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

lb_status_t lb_exchange_schedule(int32_t nranks, const int64_t* h_bounds, int32_t nchunks, const int64_t* h_cut_rows,
                                 int64_t* h_offsets, int64_t* h_counts) {
  g_err.clear();
  if (nranks < 1 || nchunks < 1 || !h_bounds || !h_offsets || !h_counts) return fail(LB_ERR_INVALID_ARG, "bad schedule arguments");
  lb_status_t st = check_bounds(nranks, h_bounds);
  if (st != LB_OK) return st;
  for (int k = 0; k < nranks; ++k) {
    const int64_t n = h_bounds[k + 1] - h_bounds[k];
    const int64_t* cut = h_cut_rows ? h_cut_rows + (size_t)k * (nchunks + 1) : nullptr;
    if (cut) {
      if (cut[0] != 0 || cut[nchunks] != n) return fail(LB_ERR_INVALID_ARG, "rank %d: cuts must run from 0 to its %lld rows", k, (long long)n);
      for (int c = 0; c < nchunks; ++c)
        if (cut[c + 1] < cut[c]) return fail(LB_ERR_INVALID_ARG, "rank %d: cuts not monotone at %d", k, c);
    }
    for (int c = 0; c < nchunks; ++c) {
      const int64_t r0 = cut ? cut[c] : (c == 0 ? 0 : n), r1 = cut ? cut[c + 1] : n;
      h_offsets[(size_t)c * nranks + k] = h_bounds[k] + r0;
      h_counts[(size_t)c * nranks + k] = r1 - r0;
    }
  }
  return LB_OK;
}

int64_t lb_padded_rows(int32_t nranks, const int64_t* h_bounds) {
  if (nranks < 1 || !h_bounds) return -1;
  int64_t P = 0;
  for (int k = 0; k < nranks; ++k) P = std::max(P, h_bounds[k + 1] - h_bounds[k]);
  return P;
}

lb_status_t lb_remap_cols_padded(int32_t nranks, const int64_t* h_bounds, const int32_t* d_col_in, int64_t nnz,
                                 int32_t* d_col_out, void* stream) {
  g_err.clear();
  if (nranks < 1 || !h_bounds || nnz < 0 || (nnz > 0 && (!d_col_in || !d_col_out)))
    return fail(LB_ERR_INVALID_ARG, "bad remap arguments");
  lb_status_t st = check_bounds(nranks, h_bounds);
  if (st != LB_OK) return st;
  const int64_t P = lb_padded_rows(nranks, h_bounds);
  if ((int64_t)nranks * P >= (int64_t)INT32_MAX) return fail(LB_ERR_INVALID_ARG, "padded column space exceeds int32");
  if (nnz == 0) return LB_OK;
  stream_t s = S(stream);
  int64_t* d_b = nullptr;
  if (cudaMalloc(&d_b, (size_t)(nranks + 1) * 8) != cudaSuccess) { cudaGetLastError(); return fail(LB_ERR_OOM, "bounds"); }
  cudaError_t e = cudaMemcpyAsync(d_b, h_bounds, (size_t)(nranks + 1) * 8, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    lbk::remap_cols_padded_kernel<<<sms * 8, 256, 0, s>>>(d_col_in, nnz, d_b, nranks, P, d_col_out);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // d_b is freed below
  cudaFree(d_b);
  if (e != cudaSuccess) return fail(LB_ERR_CUDA, "padded remap: %s", cudaGetErrorString(e));
  return LB_OK;
}

lb_status_t lb_y_checksum(const float* d_y, int64_t n, void* stream, uint64_t* h_out) {
  g_err.clear();
  if (!h_out || n < 0 || (n > 0 && !d_y)) return fail(LB_ERR_INVALID_ARG, "bad checksum arguments");
  stream_t s = S(stream);
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, 8) != cudaSuccess) { cudaGetLastError(); return fail(LB_ERR_OOM, "checksum"); }
  cudaError_t e = cudaMemsetAsync(d, 0, 8, s);
  if (e == cudaSuccess && n > 0) {
    lbk::checksum_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, s>>>(d_y, n, d);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    e = cudaGetLastError();
  }
  unsigned long long h = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(d);
  if (e != cudaSuccess) return fail(LB_ERR_CUDA, "checksum: %s", cudaGetErrorString(e));
  *h_out = h;
  return LB_OK;
}

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
  if (cudaMalloc(&c->d_hash, 3 * sizeof(unsigned long long)) != cudaSuccess) {
    cudaGetLastError(); delete c; return fail(LB_ERR_OOM, "comm scratch");
  }
  nccl_result_t r = g_nccl.CommInitRank(&c->comm, nranks, uid, rank);
  if (r != 0) { cudaFree(c->d_hash); delete c; return fail(LB_ERR_NCCL, "ncclCommInitRank: %s", g_nccl.GetErrorString(r)); }
  c->rank = rank; c->nranks = nranks; c->device = device;
  *out = c;
  return LB_OK;
}

lb_status_t lb_comm_destroy(lb_comm_t c) {
  if (!c) return LB_OK;
  if (c->comm && g_nccl.loaded) g_nccl.CommDestroy(c->comm);
  if (c->d_hash) cudaFree(c->d_hash);
  delete c;
  return LB_OK;
}

lb_status_t lb_comm_check_replicas(lb_comm_t c, const float* d_y, int64_t n, void* stream, int32_t* h_equal,
                                   uint64_t* h_hash) {
  g_err.clear();
  if (!c || !h_equal || n < 0 || (n > 0 && !d_y)) return fail(LB_ERR_INVALID_ARG, "bad replica-check arguments");
  stream_t s = S(stream);
  LB_CUDA(cudaMemsetAsync(c->d_hash, 0, 8, s));
  if (n > 0) {
    lbk::checksum_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, s>>>(d_y, n, c->d_hash);
    LB_LAUNCHED();
  }
  // min and max of the hash over the ranks: equal iff every rank holds the same bits
  LB_NCCL(g_nccl.GroupStart());
  nccl_result_t r1 = g_nccl.AllReduce(c->d_hash, c->d_hash + 1, 1, kNcclUint64, kNcclMin, c->comm, s);
  nccl_result_t r2 = r1 == 0 ? g_nccl.AllReduce(c->d_hash, c->d_hash + 2, 1, kNcclUint64, kNcclMax, c->comm, s) : r1;
  LB_NCCL(g_nccl.GroupEnd());
  if (r2 != 0) return fail(LB_ERR_NCCL, "ncclAllReduce: %s", g_nccl.GetErrorString(r2));
  unsigned long long h[3];
  LB_CUDA(cudaMemcpyAsync(h, c->d_hash, sizeof h, cudaMemcpyDeviceToHost, s));
  LB_CUDA(cudaStreamSynchronize(s));
  *h_equal = h[1] == h[2] && h[0] == h[1];
  if (h_hash) *h_hash = h[0];
  return async_error(c);
}

lb_status_t lb_allgather_rows(lb_comm_t c, const int64_t* h_bounds, float* d_y_full, void* stream) {
  LB_NVTX("lb_allgather_rows");
  g_err.clear();
  if (!c || !h_bounds || !d_y_full) return fail(LB_ERR_INVALID_ARG, "null argument");
  std::vector<int64_t> off(c->nranks), cnt(c->nranks);
  lb_status_t st = lb_exchange_schedule(c->nranks, h_bounds, 1, nullptr, off.data(), cnt.data());
  if (st != LB_OK) return st;
  // all-gather(v) as one group of broadcasts, root k sends y[b_k, b_{k+1}) (SURVEY 8(e) option 1); at
  // world size 1 the group holds one in-place broadcast (the same code path)
  if ((st = broadcast_chunk(c, d_y_full, off.data(), cnt.data(), S(stream))) != LB_OK) return st;
  return async_error(c);
}

lb_status_t lb_allgather_padded(lb_comm_t c, int64_t padded_rows, float* d_y_pad, void* stream) {
  LB_NVTX("lb_allgather_padded");
  g_err.clear();
  if (!c || !d_y_pad || padded_rows < 0) return fail(LB_ERR_INVALID_ARG, "bad padded all-gather arguments");
  if (padded_rows == 0) return LB_OK;
  // SURVEY 8(e) option 2: one ncclAllGather of equal max-shard-sized slots, in place (rank r's slot
  // is d_y_pad + r * P); the columns of every shard were remapped once to the padded ids
  LB_NCCL(g_nccl.AllGather(d_y_pad + (size_t)c->rank * padded_rows, d_y_pad, (size_t)padded_rows, kNcclFloat32,
                           c->comm, S(stream)));
  return async_error(c);
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
  LB_NVTX("lb_spmv_multi_fused");
  g_err.clear();
  if (!A_local || !peer || !h_bounds || !d_x_full) return fail(LB_ERR_INVALID_ARG, "null argument");
  lb_comm_s* c = peer->comm;
  if ((const void*)d_x_full == (const void*)peer->y) return fail(LB_ERR_INVALID_ARG, "x and y must not alias");
  lb_status_t st = check_bounds(c->nranks, h_bounds);
  if (st != LB_OK) return st;
  const int64_t b0 = h_bounds[c->rank], b1 = h_bounds[c->rank + 1];
  if (b1 - b0 != A_local->rows)
    return fail(LB_ERR_INVALID_ARG, "local shard has %lld rows, bounds say %lld", (long long)A_local->rows,
                (long long)(b1 - b0));
  if (h_bounds[c->nranks] != peer->rows) return fail(LB_ERR_INVALID_ARG, "bounds do not match the peer buffer");
  PeerArgs pa;
  for (int k = 0; k < c->nranks; ++k)
    if (k != c->rank) pa.y[pa.n++] = peer->peer_y[k] + b0;
  const bool try_fused = pa.n > 0 && sched == LB_SCHED_MERGE_PATH;
  // entry barrier: no rank stores into a peer's y before every rank's stream has finished the work
  // queued before this call (e.g. reading last iteration's y into its x) -- write-after-read order
  if (try_fused && (st = peer_barrier(peer, S(stream))) != LB_OK) return st;
  bool fused = false;
  st = spmv_impl(A_local, sched, d_x_full, peer->y + b0, flags, S(stream), nullptr, try_fused ? &pa : nullptr, &fused);
  if (st != LB_OK) return st;
  if (c->nranks == 1) return LB_OK;
  if (!fused) return lb_allgather_rows(c, h_bounds, peer->y, stream);  // no fused kernel: NCCL exchange
  // exit barrier: every rank's peer stores are complete before any rank reads its y (read-after-write)
  return peer_barrier(peer, S(stream));
}

}  // extern "C"

namespace lbi {
namespace {

// lb_spmv_multi_ex(LB_SPMV_CHUNKED): the rank's hot-plan merge-path SpMV as tile-range launches cut at
// clean coordinates (ensure_chunks); as soon as chunk c is done on every rank, an NCCL group of
// broadcasts (root k sends its chunk c rows) runs on the handle's exchange stream while chunk c+1
// computes (the sub-shard overlap).  Every rank learns every rank's cut rows (a
// group of int64 broadcasts) on the first call, after a plan or tile-length change, and on every
// LB_SPMV_REPARTITION call (all ranks pass the same flags, so the collectives match).
lb_status_t multi_chunked(lb_csr_s* A, lb_comm_s* c, lb_schedule_t sched, const int64_t* h_bounds,
                          const float* d_x_full, float* d_y_full, uint32_t flags, stream_t s) {
  lb_status_t st;
  const int64_t b0 = h_bounds[c->rank];
  float* y_loc = d_y_full + b0;
  const bool force = (flags & LB_SPMV_REPARTITION) != 0;
  const bool chunkable = sched == LB_SCHED_MERGE_PATH && hot_usable(A) && A->rows > 0;
  if (chunkable) {
    if ((st = ensure_partition(A, force, true, d_x_full, s)) != LB_OK) return st;
    if ((st = ensure_chunks(A, force, s)) != LB_OK) return st;
  } else if (A->rows > 0) {
    if ((st = spmv_impl(A, sched, d_x_full, y_loc, flags, s, nullptr)) != LB_OK) return st;
  }
  constexpr int K = kChunksMax, K1 = kChunksMax + 1;
  lb_multi_state& m = A->multi;
  if (!m.stream) {
    LB_CUDA(cudaStreamCreateWithFlags(&m.stream, cudaStreamNonBlocking));
    LB_CUDA(cudaEventCreateWithFlags(&m.done, cudaEventDisableTiming));
  }
  if ((st = ensure_chunk_events(A)) != LB_OK) return st;
  if (force || m.comm != (const void*)c || m.L != A->L || m.plan_gen != A->plan.gen || m.cut_gen != A->cut_gen ||
      (int)m.rows.size() != c->nranks * K1) {
    int64_t mine[K1];
    padded_cuts(A, chunkable, K, mine);
    int64_t* d_all = nullptr;
    if (cudaMalloc(&d_all, (size_t)c->nranks * K1 * 8) != cudaSuccess) { cudaGetLastError(); return fail(LB_ERR_OOM, "cuts"); }
    struct Free { int64_t* p; ~Free() { cudaFree(p); } } free_all{d_all};
    LB_CUDA(cudaMemcpyAsync(d_all + (size_t)c->rank * K1, mine, sizeof mine, cudaMemcpyHostToDevice, s));
    LB_NCCL(g_nccl.GroupStart());
    for (int k = 0; k < c->nranks; ++k) {
      nccl_result_t r = g_nccl.Broadcast(d_all + (size_t)k * K1, d_all + (size_t)k * K1, K1, kNcclInt64, k, c->comm, s);
      if (r != 0) { g_nccl.GroupEnd(); return fail(LB_ERR_NCCL, "ncclBroadcast: %s", g_nccl.GetErrorString(r)); }
    }
    LB_NCCL(g_nccl.GroupEnd());
    m.rows.assign((size_t)c->nranks * K1, 0);
    LB_CUDA(cudaMemcpyAsync(m.rows.data(), d_all, m.rows.size() * 8, cudaMemcpyDeviceToHost, s));
    LB_CUDA(cudaStreamSynchronize(s));
    m.comm = c;
    m.L = A->L;
    m.plan_gen = A->plan.gen;
    m.cut_gen = A->cut_gen;
  }
  std::vector<int64_t> off((size_t)K * c->nranks), cnt((size_t)K * c->nranks);
  if ((st = lb_exchange_schedule(c->nranks, h_bounds, K, m.rows.data(), off.data(), cnt.data())) != LB_OK) return st;
  lb_chunk_state& ch = A->chunks;
  for (int k = 0; k < K; ++k) {
    if (chunkable && k < ch.n) {
      ch.t0 = ch.t[k];
      ch.t1 = ch.t[k + 1];
      st = hot_launch(A, d_x_full, y_loc, s);
      ch.t0 = 0;
      ch.t1 = -1;
      if (st != LB_OK) return st;
    }
    LB_CUDA(cudaEventRecord(ch.ev[k], s));
    LB_CUDA(cudaStreamWaitEvent(m.stream, ch.ev[k], 0));
    if ((st = broadcast_chunk(c, d_y_full, &off[(size_t)k * c->nranks], &cnt[(size_t)k * c->nranks], m.stream)) != LB_OK)
      return st;
  }
  LB_CUDA(cudaEventRecord(m.done, m.stream));
  LB_CUDA(cudaStreamWaitEvent(s, m.done, 0));
  return async_error(c);
}

}  // namespace
}  // namespace lbi

extern "C" {

lb_status_t lb_csr_chunk_rows(lb_csr_t A, int32_t nchunks, int64_t* h_rows_out, void* stream) {
  g_err.clear();
  if (!A || !h_rows_out || nchunks != kChunksMax) return fail(LB_ERR_INVALID_ARG, "bad chunk-rows arguments (nchunks must be %d)", kChunksMax);
  const bool chunkable = hot_usable(A) && A->rows > 0;
  if (chunkable) {
    lb_status_t st;
    stream_t s = S(stream);
    if ((st = ensure_partition(A, false, false, nullptr, s)) != LB_OK) return st;
    if ((st = ensure_chunks(A, false, s)) != LB_OK) return st;
  }
  padded_cuts(A, chunkable, nchunks, h_rows_out);
  return LB_OK;
}

lb_status_t lb_spmv_multi(lb_csr_t A_local, lb_comm_t c, lb_schedule_t sched, const int64_t* h_bounds,
                          const float* d_x_full, float* d_y_full, void* stream) {
  return lb_spmv_multi_ex(A_local, c, sched, h_bounds, d_x_full, d_y_full, 0u, stream);
}

lb_status_t lb_spmv_multi_ex(lb_csr_t A_local, lb_comm_t c, lb_schedule_t sched, const int64_t* h_bounds,
                             const float* d_x_full, float* d_y_full, uint32_t flags, void* stream) {
  LB_NVTX("lb_spmv_multi_ex");
  g_err.clear();
  if (!A_local || !c || !h_bounds || !d_x_full || !d_y_full) return fail(LB_ERR_INVALID_ARG, "null argument");
  if ((const void*)d_x_full == (const void*)d_y_full) return fail(LB_ERR_INVALID_ARG, "x and y must not alias");
  lb_status_t st = check_bounds(c->nranks, h_bounds);
  if (st != LB_OK) return st;
  const int64_t b0 = h_bounds[c->rank], b1 = h_bounds[c->rank + 1];
  if (b1 - b0 != A_local->rows)
    return fail(LB_ERR_INVALID_ARG, "local shard has %lld rows, bounds say %lld", (long long)A_local->rows,
                (long long)(b1 - b0));
  if ((flags & LB_SPMV_PADDED) && (flags & LB_SPMV_CHUNKED))
    return fail(LB_ERR_INVALID_ARG, "LB_SPMV_PADDED and LB_SPMV_CHUNKED are exclusive");
  if (flags & LB_SPMV_PADDED) {  // y_full (and x_full) in the padded layout: slot r at r * P
    const int64_t P = lb_padded_rows(c->nranks, h_bounds);
    if ((st = spmv_impl(A_local, sched, d_x_full, d_y_full + (size_t)c->rank * P, flags, S(stream), nullptr)) != LB_OK)
      return st;
    return lb_allgather_padded(c, P, d_y_full, stream);
  }
  if (flags & LB_SPMV_CHUNKED) return multi_chunked(A_local, c, sched, h_bounds, d_x_full, d_y_full, flags, S(stream));
  st = spmv_impl(A_local, sched, d_x_full, d_y_full + b0, flags, S(stream), nullptr);
  if (st != LB_OK) return st;
  return lb_allgather_rows(c, h_bounds, d_y_full, stream);
}

}  // extern "C"
