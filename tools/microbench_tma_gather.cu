// Microbenchmark: can TMA (tile::gather4 / cp.async.bulk) beat the ~1 line/clk/SM L1tex
// gather rate for random 4-byte x[col] reads?  (Design probe for the SpMV tile kernel.)
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n"
      :: "r"(smem_u32(b)), "r"(parity) : "memory");
}

// Each warp: lane 0 issues NB gather4 per batch (4*NB random 16-byte rows), waits, repeats.
template <int NB>
__global__ void k_tma_gather4(const __grid_constant__ CUtensorMap tm, uint32_t rows_mask, int batches, float* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm) + warp;
  uint8_t* dst = sm + 1024 + warp * NB * 128;
  if (lane == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncwarp();
  float s = 0.f;
  uint64_t base = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) << 32;
  for (int b = 0; b < batches; ++b) {
    if (lane == 0) {
      mbar_expect(bar, NB * 64);
      for (int q = 0; q < NB; ++q) {
        uint64_t h = mix64(base + b * NB + q);
        int r0 = (int)(h & rows_mask), r1 = (int)((h >> 16) & rows_mask), r2 = (int)((h >> 32) & rows_mask),
            r3 = (int)((h >> 40) & rows_mask);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
            :: "r"(smem_u32(dst + q * 128)), "l"(&tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
            : "memory");
      }
      mbar_wait(bar, b & 1);
      s += reinterpret_cast<float*>(dst)[b & 15];
    }
    __syncwarp();
  }
  if (s == 1234.5f) out[0] = s;
}

// Each warp: lane 0 issues NB cp.async.bulk of 16 bytes at random 16B-aligned offsets.
template <int NB>
__global__ void k_bulk16(const float* x, uint32_t rows_mask, int batches, float* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm) + warp;
  uint8_t* dst = sm + 1024 + warp * NB * 16;
  if (lane == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncwarp();
  float s = 0.f;
  uint64_t base = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) << 32;
  for (int b = 0; b < batches; ++b) {
    // lanes split the issue work
    if (lane == 0) mbar_expect(bar, NB * 16);
    __syncwarp();
    for (int q = lane; q < NB; q += 32) {
      uint64_t h = mix64(base + b * NB + q);
      const float* src = x + 4 * (h & rows_mask);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];"
          :: "r"(smem_u32(dst + q * 16)), "l"(src), "r"(smem_u32(bar)) : "memory");
    }
    mbar_wait(bar, b & 1);
    s += reinterpret_cast<float*>(dst)[b & 15];
    __syncwarp();
  }
  if (s == 1234.5f) out[0] = s;
}

template <typename F>
float time_ms(F f, int reps = 7) {
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
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  float* out; CK(cudaMalloc(&out, 4));
  for (int logm : {24, 26}) {
    size_t M = 1ull << logm;  // floats
    float* x; CK(cudaMalloc(&x, M * 4)); CK(cudaMemset(x, 0, M * 4));
    CUtensorMap tm;
    cuuint64_t dims[2] = {4, M / 4};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {4, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    uint32_t rmask = (uint32_t)(M / 4 - 1);
    for (int wpb : {4, 8}) for (int bpsm : {1, 2, 4}) {
      const int NB = 32, batches = 256;
      int grid = sms * bpsm, threads = wpb * 32;
      size_t smem = 1024 + wpb * NB * 128;
      CK(cudaFuncSetAttribute(k_tma_gather4<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      float ms = time_ms([&] { k_tma_gather4<NB><<<grid, threads, smem>>>(tm, rmask, batches, out); });
      CK(cudaGetLastError());
      double rowsg = (double)grid * wpb * batches * NB * 4;
      printf("tma_gather4 x=%4zu MB warps/cta=%d cta/sm=%d: %.1f G rows(16B)/s\n", M * 4 >> 20, wpb, bpsm, rowsg / ms / 1e6);
    }
    for (int wpb : {4, 8}) for (int bpsm : {2, 4}) {
      const int NB = 64, batches = 256;
      int grid = sms * bpsm, threads = wpb * 32;
      size_t smem = 1024 + wpb * NB * 16;
      CK(cudaFuncSetAttribute(k_bulk16<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      float ms = time_ms([&] { k_bulk16<NB><<<grid, threads, smem>>>(x, rmask, batches, out); });
      CK(cudaGetLastError());
      double n = (double)grid * wpb * batches * NB;
      printf("bulk16      x=%4zu MB warps/cta=%d cta/sm=%d: %.1f G copies/s\n", M * 4 >> 20, wpb, bpsm, n / ms / 1e6);
    }
    CK(cudaFree(x));
  }
  printf("done\n");
  return 0;
}
