// Probe: where can a random 4-byte x gather be served from, and at what rate, beyond the one
// L1TEX line per clock per SM of a global miss?  R-MAT-like column distribution (popcount classes
// of a 24-bit column id with P(bit) = 0.24, i.e. Graph500 b + d), 2^28 nonzeros, x = 64 MB.
//   hot  : the H most referenced columns in shared memory (H = 16384 per CTA); with a cluster of
//          CL CTAs the hot set is CL x 16384 slots spread over the cluster (DSMEM reads)
//   warm : the next KW columns packed into a dense copy xw, read with an L1 eviction priority
//   cold : x[col] with an L1 eviction / no-allocate flavour
// Question answered: do L1-resident packed warm columns or a cluster-wide DSMEM hot set raise
// GNZ/s over the per-SM shared-memory hot tier of merge_stream_kernel?
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull; z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; return z ^ (z >> 31);
}
constexpr int NC = 1 << 24;
constexpr int SLOTS = 16384;  // per CTA
// column classes by popcount: pc <= 4 -> 12951 columns (28.3% of nnz), pc 5 -> 42504 (18.4%),
// pc 6 -> 134596 (18.4%).  hot: the H top columns; warm: the next KW.
__global__ void k_fill(int* col, size_t n, int H, int KW, uint64_t seed) {
  const int c4 = 12951, c5 = 42504, c6 = 134596;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t c = 0;
    for (int b = 0; b < 24; ++b) { uint32_t u = (uint32_t)(mix64(seed + i * 64 + b) >> 40); c |= (u < (uint32_t)(0.24 * 16777216.0)) ? (1u << b) : 0u; }
    const int pc = __popc(c);
    // rank of this column in degree order (approximate within a class: a hash index)
    long rank;
    if (pc <= 4) rank = (long)(mix64(c) % c4);
    else if (pc == 5) rank = c4 + (long)(mix64(c) % c5);
    else if (pc == 6) rank = c4 + c5 + (long)(mix64(c) % c6);
    else rank = 1L << 40;
    uint32_t p = (c * 0x9E3779B1u) & (NC - 1); p ^= p >> 12; p = (p * 0x85EBCA77u) & (NC - 1);
    int v;
    if (rank < H) v = ~(int)(mix64(c ^ 77) % (uint64_t)H);
    else if (rank < (long)H + KW) v = NC + (int)(mix64(c ^ 99) % (uint64_t)KW);
    else v = (int)p;
    col[i] = v;
  }
}
__device__ __forceinline__ void ld8(const int* p, int (&r)[8]) {
  asm volatile("ld.global.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "l"(p));
}
__device__ __forceinline__ void ld8(const float* p, float (&r)[8]) {
  asm volatile("ld.global.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7]) : "l"(p));
}
template <int M> __device__ __forceinline__ float ldg_flavour(const float* p) {
  float v;
  if (M == 0) asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(p));
  else if (M == 1) asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  else if (M == 2) asm volatile("ld.global.nc.L1::evict_first.f32 %0, [%1];" : "=f"(v) : "l"(p));
  else asm volatile("ld.global.nc.L1::evict_last.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
// CM: cold flavour, WM: warm flavour, CL: cluster size for the hot set
template <int CM, int WM, int CL>
__global__ void __launch_bounds__(512, 1) k_tiers(const int* __restrict__ col, const float* __restrict__ val,
                                                  const float* __restrict__ x, const float* __restrict__ xw,
                                                  size_t n, float* out) {
  extern __shared__ float sm[];
  for (int s = threadIdx.x; s < SLOTS; s += blockDim.x) sm[s] = __ldg(x + s * 97);
  uint32_t rank_self = 0;
  if (CL > 1) {
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank_self));
    asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
  } else {
    __syncthreads();
  }
  const uint32_t smb = (uint32_t)__cvta_generic_to_shared(sm);
  float s = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x * 8;
  for (size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 8; i + 8 <= n; i += stride) {
    int c[8]; float v[8], xv[8];
    ld8(col + i, c); ld8(val + i, v);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int ce = c[e];
      if (ce < 0) {
        const uint32_t slot = (uint32_t)~ce;
        if (CL == 1) {
          xv[e] = sm[slot];
        } else {
          const uint32_t r = slot / SLOTS, off = slot % SLOTS;
          uint32_t ra;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smb + 4 * off), "r"(r));
          asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(xv[e]) : "r"(ra));
        }
      } else if (ce >= NC) {
        xv[e] = ldg_flavour<WM>(xw + (ce - NC));
      } else {
        xv[e] = ldg_flavour<CM>(x + ce);
      }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) s = fmaf(v[e], xv[e], s);
  }
  if (CL > 1) asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
  if (s == 1234.5f) out[0] = s + (float)rank_self;
}
template <typename F> float time_ms(F f, int reps = 7) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b)); f(); CK(cudaDeviceSynchronize());
  std::vector<float> t;
  for (int r = 0; r < reps; ++r) { CK(cudaEventRecord(a)); f(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b)); float ms; CK(cudaEventElapsedTime(&ms, a, b)); t.push_back(ms); }
  std::sort(t.begin(), t.end()); return t[t.size() / 2];
}
template <int CM, int WM, int CL>
void run(const char* tag, const int* col, const float* val, const float* x, const float* xw, size_t G, float* out, int sms,
         double hf, double wf) {
  auto k = k_tiers<CM, WM, CL>;
  const int smem = SLOTS * 4;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 30));
  if (CL > 1) CK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms / CL * CL);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  float ms = time_ms([&] { CK(cudaLaunchKernelEx(&cfg, k, col, val, x, xw, G, out)); });
  CK(cudaGetLastError());
  printf("%-34s hot %.3f warm %.3f cold %.3f  cold=%d warm=%d cluster=%d: %6.1f GNZ/s\n", tag, hf, wf, 1 - hf - wf, CM,
         WM, CL, G / ms / 1e6);
  fflush(stdout);
}
int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0)); const int sms = p.multiProcessorCount;
  const size_t G = 1ull << 28;
  int* col; float *val, *x, *xw, *out;
  CK(cudaMalloc(&col, G * 4)); CK(cudaMalloc(&val, G * 4)); CK(cudaMalloc(&x, (size_t)NC * 4)); CK(cudaMalloc(&xw, 1 << 24));
  CK(cudaMalloc(&out, 4));
  CK(cudaMemset(val, 0, G * 4)); CK(cudaMemset(x, 0, (size_t)NC * 4)); CK(cudaMemset(xw, 0, 1 << 24));
  int* hcol; CK(cudaMallocHost(&hcol, 1 << 22));
  struct Case { int H, KW; };
  const Case cases[] = {{16384, 0}, {16384, 8192}, {16384, 16384}, {16384, 24576}, {16384, 40000}, {32768, 0}, {65536, 0},
                        {32768, 16384}};
  for (const Case& cs : cases) {
    k_fill<<<sms * 8, 256>>>(col, G, cs.H, cs.KW, 12345); CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(hcol, col, 1 << 22, cudaMemcpyDeviceToHost));
    int nh = 0, nw = 0; for (int i = 0; i < (1 << 20); ++i) { nh += hcol[i] < 0; nw += hcol[i] >= NC; }
    const double hf = nh / double(1 << 20), wf = nw / double(1 << 20);
    char tag[64];
    snprintf(tag, sizeof tag, "H %d KW %d", cs.H, cs.KW);
    if (cs.H == 16384) {
      if (cs.KW == 0) {
        run<0, 0, 1>(tag, col, val, x, xw, G, out, sms, hf, wf);
        run<1, 0, 1>(tag, col, val, x, xw, G, out, sms, hf, wf);
        run<2, 0, 1>(tag, col, val, x, xw, G, out, sms, hf, wf);
      } else {
        run<0, 0, 1>(tag, col, val, x, xw, G, out, sms, hf, wf);
        run<0, 3, 1>(tag, col, val, x, xw, G, out, sms, hf, wf);
        run<1, 3, 1>(tag, col, val, x, xw, G, out, sms, hf, wf);
        run<2, 3, 1>(tag, col, val, x, xw, G, out, sms, hf, wf);
        run<1, 0, 1>(tag, col, val, x, xw, G, out, sms, hf, wf);
      }
    } else if (cs.H == 32768) {
      if (cs.KW == 0) {
        run<0, 0, 2>(tag, col, val, x, xw, G, out, sms, hf, wf);
        run<1, 0, 2>(tag, col, val, x, xw, G, out, sms, hf, wf);
      } else {
        run<1, 3, 2>(tag, col, val, x, xw, G, out, sms, hf, wf);
      }
    } else {
      run<0, 0, 4>(tag, col, val, x, xw, G, out, sms, hf, wf);
      run<1, 0, 4>(tag, col, val, x, xw, G, out, sms, hf, wf);
    }
  }
  printf("done\n");
}
