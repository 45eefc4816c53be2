// Probe: can x[col] gathers issued as 4-byte cp.async (LDGSTS, global -> shared) keep more misses in
// flight than LDG gathers, whose in-flight misses hold L1 lines (profiles/r01_microbench_l1.txt)?
// Stream col/val with 256-bit loads, gather x[col] (R-MAT-like columns, x = 64 MB, 2^28 nonzeros).
//  mode 0: LDG gathers into registers, depth-2 software pipeline (like the tile kernel)
//  mode 1: cp.async.ca 4-byte gathers into a per-warp shared ring of S stages, wait_group S-1
// plus a shared-memory ballast to emulate the tile kernel's hot-x cache (smem/SM grows).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull; z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; return z ^ (z >> 31);
}
__global__ void k_fill(int* col, size_t n, uint32_t mask, int bits, uint64_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t c = 0;
    for (int b = 0; b < bits; ++b) { uint32_t u = (uint32_t)(mix64(seed + i * 64 + b) >> 40); c |= (u < (uint32_t)(0.24 * 16777216.0)) ? (1u << b) : 0u; }
    uint32_t p = (c * 0x9E3779B1u) & mask; p ^= p >> (bits / 2); p = (p * 0x85EBCA77u) & mask;
    col[i] = (int)p;
  }
}
__device__ __forceinline__ void ld8(const int* p, int (&r)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "l"(p));
}
__device__ __forceinline__ void ld8(const float* p, float (&r)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7]) : "l"(p));
}
// mode 0: per warp round = 256 nonzeros (8 per lane); gathers of round r+1 in flight while r is summed
__global__ void k_ldg(const int* __restrict__ col, const float* __restrict__ val, const float* __restrict__ x,
                      size_t n, float* out) {
  extern __shared__ float ballast[];
  float s = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x * 8;
  size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 8;
  int c[8]; float v[8], xv[8], vn[8], xn[8];
  if (i + 8 <= n) { ld8(col + i, c); ld8(val + i, v);
#pragma unroll
    for (int e = 0; e < 8; ++e) xv[e] = __ldg(x + c[e]); }
  for (; i + 8 <= n; i += stride) {
    const size_t j = i + stride;
    if (j + 8 <= n) { ld8(col + j, c); ld8(val + j, vn);
#pragma unroll
      for (int e = 0; e < 8; ++e) xn[e] = __ldg(x + c[e]); }
#pragma unroll
    for (int e = 0; e < 8; ++e) s = fmaf(v[e], xv[e], s);
#pragma unroll
    for (int e = 0; e < 8; ++e) { v[e] = vn[e]; xv[e] = xn[e]; }
  }
  if (s == 1234.5f) { ballast[threadIdx.x] = s; out[0] = ballast[threadIdx.x ^ 1]; }
}
// mode 1: cp.async 4-byte gathers into a shared ring of S stages per thread (8 floats per stage)
template <int S>
__global__ void k_cpasync(const int* __restrict__ col, const float* __restrict__ val, const float* __restrict__ x,
                          size_t n, float* out) {
  extern __shared__ float sm[];  // [S][blockDim][8] ring, then ballast
  float s = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x * 8;
  const size_t i0 = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 8;
  float vr[S][8];
  auto slot = [&](int st, int e) { return (uint32_t)__cvta_generic_to_shared(&sm[(st * blockDim.x + threadIdx.x) * 8 + e]); };
  // prologue: S-1 stages in flight
#pragma unroll
  for (int st = 0; st < S - 1; ++st) {
    const size_t i = i0 + st * stride;
    if (i + 8 <= n) {
      int c[8]; ld8(col + i, c); ld8(val + i, vr[st]);
#pragma unroll
      for (int e = 0; e < 8; ++e)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(slot(st, e)), "l"(x + c[e]) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  size_t i = i0;
  while (true) {
#pragma unroll
    for (int st = 0; st < S; ++st) {  // consume stage st, refill stage (st + S - 1) % S
      if (i + 8 > n) goto done;
      const size_t j = i + (S - 1) * stride;
      constexpr int dummy = 0; (void)dummy;
      const int sj = (st + S - 1) % S;
      if (j + 8 <= n) {
        int c[8]; ld8(col + j, c); ld8(val + j, vr[sj]);
#pragma unroll
        for (int e = 0; e < 8; ++e)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(slot(sj, e)), "l"(x + c[e]) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group %0;" :: "n"(S - 1) : "memory");
#pragma unroll
      for (int e = 0; e < 8; ++e) s = fmaf(vr[st][e], sm[(st * blockDim.x + threadIdx.x) * 8 + e], s);
      i += stride;
    }
  }
done:
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (s == 1234.5f) out[0] = s;
}
template <typename F> float time_ms(F f, int reps = 5) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b)); f(); CK(cudaDeviceSynchronize());
  std::vector<float> t;
  for (int r = 0; r < reps; ++r) { CK(cudaEventRecord(a)); f(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b)); float ms; CK(cudaEventElapsedTime(&ms, a, b)); t.push_back(ms); }
  std::sort(t.begin(), t.end()); return t[t.size() / 2];
}
template <typename K> void run(const char* name, K k, size_t ring_per_thread, const int* col, const float* val,
                               const float* x, size_t G, float* out, int sms) {
  for (int nt : {256, 512}) for (int bpsm : {1, 2, 4}) for (int ballast_kb : {0, 32, 64, 96, 128}) {
    if (nt * bpsm > 1024) continue;
    const size_t smem = ring_per_thread * nt + (size_t)ballast_kb * 1024 / bpsm;
    if (smem * bpsm > 220 * 1024) continue;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    int pct = std::min(100, (int)(100.0 * (smem + 1024) * bpsm / (228.0 * 1024)) + 1);
    CK(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
    int occ = 0; CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, nt, smem));
    if (occ < bpsm) continue;
    float ms = time_ms([&] { k<<<sms * bpsm, nt, smem>>>(col, val, x, G, out); });
    CK(cudaGetLastError());
    printf("%-10s nt %3d ctas/sm %d smem/SM %3zu KB (ballast %3d KB): %6.1f GNZ/s\n", name, nt, bpsm,
           smem * bpsm / 1024, ballast_kb, G / ms / 1e6);
    fflush(stdout);
  }
}
int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0)); const int sms = p.multiProcessorCount;
  const size_t G = 1ull << 28; const int bits = 24; const uint32_t mask = (1u << bits) - 1;
  int* col; float *val, *x, *out;
  CK(cudaMalloc(&col, G * 4)); CK(cudaMalloc(&val, G * 4)); CK(cudaMalloc(&x, (mask + 1) * 4ull)); CK(cudaMalloc(&out, 4));
  CK(cudaMemset(val, 0, G * 4)); CK(cudaMemset(x, 0, (mask + 1) * 4ull));
  k_fill<<<sms * 8, 256>>>(col, G, mask, bits, 12345); CK(cudaDeviceSynchronize());
  run("ldg", k_ldg, 0, col, val, x, G, out, sms);
  run("cpasync2", k_cpasync<2>, 2 * 32, col, val, x, G, out, sms);
  run("cpasync3", k_cpasync<3>, 3 * 32, col, val, x, G, out, sms);
  run("cpasync4", k_cpasync<4>, 4 * 32, col, val, x, G, out, sms);
  printf("done\n");
}
