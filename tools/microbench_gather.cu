// Microbenchmark: HBM stream bandwidth vs random 4-byte gather throughput on B200.
// Purpose: decide how the SpMV tile processor should issue its x[col] gathers.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/mb tools/microbench_gather.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_read_f4(const float4* __restrict__ a, size_t n4, float* out) {
  float s = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = a[i];
    s += v.x + v.y + v.z + v.w;
  }
  if (s == 1234.5f) out[0] = s;
}

__global__ void k_copy_f4(const float4* __restrict__ a, float4* __restrict__ b, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

template <int MODE>
__device__ __forceinline__ float ldx(const float* p) {
  float v;
  if (MODE == 0) v = *p;
  else if (MODE == 1) v = __ldg(p);
  else if (MODE == 2) asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  else if (MODE == 3) asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
  else asm volatile("ld.global.nc.L1::evict_last.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}

// Pure gather: indices from a hash in registers (no index stream).
template <int MODE, int U>
__global__ void k_gather_hash(const float* __restrict__ x, uint32_t mask, size_t n, float* out) {
  float s = 0.f;
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = tid * U; i < n; i += stride * U) {
    float v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldx<MODE>(x + ((uint32_t)mix64(i + u) & mask));
#pragma unroll
    for (int u = 0; u < U; ++u) s += v[u];
  }
  if (s == 1234.5f) out[0] = s;
}

// SpMV-like stream: sum += val[k] * x[col[k]] over a coalesced (col,val) stream.
template <int MODE, int U>
__global__ void k_stream_gather(const int* __restrict__ col, const float* __restrict__ val,
                                const float* __restrict__ x, size_t n, float* out) {
  float s = 0.f;
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = tid;
  for (; i + (U - 1) * stride < n; i += stride * U) {
    int c[U];
    float v[U], xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { c[u] = __ldcs(col + i + u * stride); v[u] = __ldcs(val + i + u * stride); }
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = ldx<MODE>(x + c[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) s = fmaf(v[u], xv[u], s);
  }
  for (; i < n; i += stride) s += val[i] * x[col[i]];
  if (s == 1234.5f) out[0] = s;
}

__global__ void k_fill_idx(int* col, size_t n, uint32_t mask, int rmat_bits, uint64_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t c;
    if (rmat_bits == 0) {
      c = (uint32_t)mix64(seed + i) & mask;
    } else {
      // R-MAT column marginal: each of rmat_bits bits is 1 w.p. 0.24, then a bijective scramble.
      c = 0;
      for (int b = 0; b < rmat_bits; ++b) {
        uint32_t u = (uint32_t)(mix64(seed + i * 64 + b) >> 40);
        c |= (u < (uint32_t)(0.24 * 16777216.0)) ? (1u << b) : 0u;
      }
      c = (c * 0x9E3779B1u) & mask; c ^= c >> (rmat_bits / 2); c = (c * 0x85EBCA77u) & mask;
    }
    col[i] = (int)c;
  }
}

__global__ void k_fill_f(float* a, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) a[i] = 1.0f;
}

template <typename F>
float time_ms(F f, int reps = 10) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); CK(cudaDeviceSynchronize());
  std::vector<float> t;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a)); f(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b)); t.push_back(ms);
  }
  std::sort(t.begin(), t.end());
  return t[t.size() / 2];
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  printf("device %s sms=%d l2=%d MB smem/sm=%zu\n", p.name, sms, p.l2CacheSize >> 20, p.sharedMemPerMultiprocessor);
  float* out; CK(cudaMalloc(&out, 4));
  const size_t N = 1ull << 29;  // 512 Mi floats = 2 GiB
  float *a, *b; CK(cudaMalloc(&a, N * 4)); CK(cudaMalloc(&b, N * 4));
  k_fill_f<<<sms * 8, 256>>>(a, N); k_fill_f<<<sms * 8, 256>>>(b, N);
  for (int bpsm : {4, 8, 16}) {
    float ms = time_ms([&] { k_read_f4<<<sms * bpsm, 256>>>((float4*)a, N / 4, out); });
    printf("read_f4   grid=%d*%d: %.3f ms  %.1f GB/s\n", sms, bpsm, ms, N * 4 / ms / 1e6);
    ms = time_ms([&] { k_copy_f4<<<sms * bpsm, 256>>>((float4*)a, (float4*)b, N / 4); });
    printf("copy_f4   grid=%d*%d: %.3f ms  %.1f GB/s (r+w)\n", sms, bpsm, ms, N * 8 / ms / 1e6);
  }
  const size_t G = 1ull << 28;  // gathers per launch
  for (uint32_t logm : {10u, 12u, 14u, 15u, 16u, 20u, 24u}) {
    uint32_t mask = (1u << logm) - 1;
    float t0 = time_ms([&] { k_gather_hash<0, 8><<<sms * 8, 256>>>(a, mask, G, out); });
    float t1 = time_ms([&] { k_gather_hash<1, 8><<<sms * 8, 256>>>(a, mask, G, out); });
    float t2 = time_ms([&] { k_gather_hash<2, 8><<<sms * 8, 256>>>(a, mask, G, out); });
    float t3 = time_ms([&] { k_gather_hash<3, 8><<<sms * 8, 256>>>(a, mask, G, out); });
    float t4 = time_ms([&] { k_gather_hash<4, 8><<<sms * 8, 256>>>(a, mask, G, out); });
    printf("gather_hash x=%8u KB: G/s default %.1f  ldg %.1f  na %.1f  cg %.1f  evl %.1f\n", (1u << logm) * 4 >> 10,
           G / t0 / 1e6, G / t1 / 1e6, G / t2 / 1e6, G / t3 / 1e6, G / t4 / 1e6);
  }
  int* col; CK(cudaMalloc(&col, G * 4));
  for (int rm : {0, 24}) {
    for (uint32_t logm : {24u, 26u}) {
      uint32_t mask = (1u << logm) - 1;
      k_fill_idx<<<sms * 8, 256>>>(col, G, mask, rm ? (int)logm : 0, 12345);
      CK(cudaDeviceSynchronize());
      for (int bpsm : {4, 8}) {
        float t0 = time_ms([&] { k_stream_gather<0, 8><<<sms * bpsm, 256>>>(col, b, a, G, out); });
        float t1 = time_ms([&] { k_stream_gather<1, 8><<<sms * bpsm, 256>>>(col, b, a, G, out); });
        float t2 = time_ms([&] { k_stream_gather<2, 8><<<sms * bpsm, 256>>>(col, b, a, G, out); });
        float t4 = time_ms([&] { k_stream_gather<4, 8><<<sms * bpsm, 256>>>(col, b, a, G, out); });
        double bytes = G * 8.0 + (1ull << logm) * 4.0;
        printf("stream_gather %s x=%4u MB bpsm=%d: GNZ/s default %.1f ldg %.1f na %.1f evl %.1f | alg GB/s best %.0f\n",
               rm ? "rmat" : "unif", (1u << logm) * 4 >> 20, bpsm, G / t0 / 1e6, G / t1 / 1e6, G / t2 / 1e6,
               G / t4 / 1e6, bytes / std::min(std::min(t0, t1), std::min(t2, t4)) / 1e6);
      }
    }
  }
  CK(cudaDeviceSynchronize());
  printf("done\n");
  return 0;
}
