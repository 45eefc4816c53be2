// Probe: SpMV-like stream+gather throughput vs shared-memory carve-out (L1 left) and load flavour.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull; z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; return z ^ (z >> 31);
}
template <int MODE> __device__ __forceinline__ float ldx(const float* p) {
  float v;
  if (MODE == 0) v = __ldg(p);
  else if (MODE == 1) asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  else asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
template <int MODE, int U>
__global__ void k_stream_gather(const int* __restrict__ col, const float* __restrict__ val, const float* __restrict__ x, size_t n, float* out) {
  extern __shared__ float sm[];
  float s = 0.f;
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = tid; i + (U - 1) * stride < n; i += stride * U) {
    int c[U]; float v[U], xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { c[u] = __ldcs(col + i + u * stride); v[u] = __ldcs(val + i + u * stride); }
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = ldx<MODE>(x + c[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) s = fmaf(v[u], xv[u], s);
  }
  if (s == 1234.5f) { sm[threadIdx.x] = s; out[0] = sm[threadIdx.x ^ 1]; }
}
__global__ void k_fill_idx(int* col, size_t n, uint32_t mask, int bits, uint64_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t c = 0;
    for (int b = 0; b < bits; ++b) { uint32_t u = (uint32_t)(mix64(seed + i * 64 + b) >> 40); c |= (u < (uint32_t)(0.24 * 16777216.0)) ? (1u << b) : 0u; }
    c = (c * 0x9E3779B1u) & mask; c ^= c >> (bits / 2); c = (c * 0x85EBCA77u) & mask;
    col[i] = (int)c;
  }
}
template <typename F> float time_ms(F f, int reps = 7) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b)); f(); CK(cudaDeviceSynchronize());
  std::vector<float> t;
  for (int r = 0; r < reps; ++r) { CK(cudaEventRecord(a)); f(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b)); float ms; CK(cudaEventElapsedTime(&ms, a, b)); t.push_back(ms); }
  std::sort(t.begin(), t.end()); return t[t.size() / 2];
}
template <int MODE> void run(const int* col, const float* val, const float* x, size_t G, float* out, int sms) {
  auto k = k_stream_gather<MODE, 8>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  for (int bpsm : {4, 8}) for (int smkb : {0, 8, 16, 24, 28, 40}) {
    if (bpsm * smkb > 220) continue;
    size_t smem = smkb * 1024;
    float ms = time_ms([&] { k<<<sms * bpsm, 256, smem>>>(col, val, x, G, out); });
    CK(cudaGetLastError());
    printf("mode %d ctas/sm %d smem/cta %3d KB (smem/SM %3d KB): %.1f GNZ/s\n", MODE, bpsm, smkb, bpsm * smkb, G / ms / 1e6);
  }
}
int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0)); int sms = p.multiProcessorCount;
  const size_t G = 1ull << 28; const int bits = 24; const uint32_t mask = (1u << bits) - 1;
  int* col; float *val, *x, *out;
  CK(cudaMalloc(&col, G * 4)); CK(cudaMalloc(&val, G * 4)); CK(cudaMalloc(&x, (mask + 1) * 4ull)); CK(cudaMalloc(&out, 4));
  CK(cudaMemset(val, 0, G * 4)); CK(cudaMemset(x, 0, (mask + 1) * 4ull));
  k_fill_idx<<<sms * 8, 256>>>(col, G, mask, bits, 12345); CK(cudaDeviceSynchronize());
  run<0>(col, val, x, G, out, sms); run<1>(col, val, x, G, out, sms); run<2>(col, val, x, G, out, sms);
  printf("done\n");
}
