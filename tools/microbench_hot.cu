// Probe: stream+gather where a fraction of the x gathers is served from a shared-memory copy of
// the hottest columns (R-MAT-like column distribution, 2^24 columns, 2^28 nonzeros).
// Question answered: does moving hot gathers from L1TEX global misses to LDS raise GNZ/s, and how
// does that trade against the L1 capacity the shared-memory carve-out takes away?
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull; z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; return z ^ (z >> 31);
}
// col < 0 encodes a hot slot ~col; otherwise a global column
__global__ void k_fill(int* col, size_t n, uint32_t mask, int bits, uint64_t seed, int thr, int ks, int half5) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t c = 0;
    for (int b = 0; b < bits; ++b) { uint32_t u = (uint32_t)(mix64(seed + i * 64 + b) >> 40); c |= (u < (uint32_t)(0.24 * 16777216.0)) ? (1u << b) : 0u; }
    const int pc = __popc(c);
    const bool hot = ks > 0 && (pc <= thr || (half5 && pc == thr + 1 && (mix64(c) & 1023) < (uint64_t)half5));
    uint32_t p = (c * 0x9E3779B1u) & mask; p ^= p >> (bits / 2); p = (p * 0x85EBCA77u) & mask;
    col[i] = hot ? ~(int)(mix64(c ^ 77) % (uint64_t)ks) : (int)p;
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
template <bool HOT>
__global__ void k_stream(const int* __restrict__ col, const float* __restrict__ val, const float* __restrict__ x,
                         size_t n, int ks, float* out) {
  extern __shared__ float sm[];
  if (HOT) {
    for (int s = threadIdx.x; s < ks; s += blockDim.x) sm[s] = __ldg(x + s * 97);
    __syncthreads();
  }
  float s = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x * 8;
  for (size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 8; i + 8 <= n; i += stride) {
    int c[8]; float v[8], xv[8];
    ld8(col + i, c); ld8(val + i, v);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      if (HOT) xv[e] = c[e] < 0 ? sm[~c[e]] : __ldg(x + c[e]);
      else xv[e] = __ldg(x + c[e]);
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) s = fmaf(v[e], xv[e], s);
  }
  if (s == 1234.5f) out[0] = s;
}
template <typename F> float time_ms(F f, int reps = 7) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b)); f(); CK(cudaDeviceSynchronize());
  std::vector<float> t;
  for (int r = 0; r < reps; ++r) { CK(cudaEventRecord(a)); f(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b)); float ms; CK(cudaEventElapsedTime(&ms, a, b)); t.push_back(ms); }
  std::sort(t.begin(), t.end()); return t[t.size() / 2];
}
int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0)); const int sms = p.multiProcessorCount;
  const size_t G = 1ull << 28; const int bits = 24; const uint32_t mask = (1u << bits) - 1;
  int* col; float *val, *x, *out;
  CK(cudaMalloc(&col, G * 4)); CK(cudaMalloc(&val, G * 4)); CK(cudaMalloc(&x, (mask + 1) * 4ull)); CK(cudaMalloc(&out, 4));
  CK(cudaMemset(val, 0, G * 4)); CK(cudaMemset(x, 0, (mask + 1) * 4ull));
  int* hcol; CK(cudaMallocHost(&hcol, 1 << 22));
  struct Case { int thr, ks, half5; };
  const Case cases[] = {{-1, 0, 0}, {2, 512, 0}, {3, 4096, 0}, {4, 8192, 0}, {4, 16384, 0}, {4, 16384, 256}, {4, 24576, 512}, {4, 32768, 1023}};
  for (const Case& cs : cases) {
    k_fill<<<sms * 8, 256>>>(col, G, mask, bits, 12345, cs.thr, cs.ks, cs.half5); CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(hcol, col, 1 << 22, cudaMemcpyDeviceToHost));
    int nh = 0; for (int i = 0; i < (1 << 20); ++i) nh += hcol[i] < 0;
    const double hf = nh / double(1 << 20);
    for (int nt : {256, 512, 1024}) for (int bpsm : {1, 2, 4, 8}) {
      if (nt * bpsm > 2048) continue;
      const size_t smem = (size_t)cs.ks * 4;
      if (smem * bpsm > 220 * 1024) continue;
      float ms;
      if (cs.ks == 0) {
        auto k = k_stream<false>;
        CK(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
        ms = time_ms([&] { k<<<sms * bpsm, nt, 0>>>(col, val, x, G, 0, out); });
      } else {
        auto k = k_stream<true>;
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int pct = (int)(100.0 * (smem + 1024) * bpsm / (228.0 * 1024)) + 1;
        CK(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, std::min(100, pct)));
        int occ = 0; CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, nt, smem));
        if (occ < bpsm) continue;
        ms = time_ms([&] { k<<<sms * bpsm, nt, smem>>>(col, val, x, G, cs.ks, out); });
      }
      CK(cudaGetLastError());
      printf("hot_frac %.3f slots %6d (smem/SM %3zu KB) nt %4d ctas/sm %d: %6.1f GNZ/s\n", hf, cs.ks,
             smem * bpsm / 1024, nt, bpsm, G / ms / 1e6);
      fflush(stdout);
    }
  }
  printf("done\n");
}
