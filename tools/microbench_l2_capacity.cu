// Effective L2 capacity for data gathered by ALL SMs (B200: two dies, one L2 per die).
// Random 4-byte gathers over an x of S MB (index = hash(i) mod n, no index stream), every SM touching
// all of x.  Per size: gathers/s of a warm launch (CUDA events) -- when S outgrows what the L2 keeps
// for all-SM-shared data, the gathers start missing to DRAM and the rate drops.  ncu's dram bytes per
// launch of the same binary (run under ncu --cache-control none) give the miss traffic directly.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_l2cap tools/microbench_l2_capacity.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint32_t v) {
  v ^= v >> 16; v *= 0x7feb352dU; v ^= v >> 15; v *= 0x846ca68bU; v ^= v >> 16; return v;
}

__global__ void gather_kernel(const float* __restrict__ x, uint32_t n, int per_thread, uint32_t salt,
                              float* __restrict__ out) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  float acc = 0.f;
#pragma unroll 8
  for (int k = 0; k < per_thread; ++k) {
    const uint32_t h = mix(t * 0x9E3779B9u + k * 0x85EBCA6Bu + salt);
    acc += __ldg(x + (uint32_t)(((uint64_t)h * n) >> 32));
  }
  out[t] = acc;
}

int main() {
  const int sizes_mb[] = {8, 16, 24, 32, 40, 48, 56, 64, 72, 80, 96, 112, 128, 192, 256};
  const int blocks = 148 * 8, threads = 256, per_thread = 512;
  const double gathers = (double)blocks * threads * per_thread;
  float* x; float* out;
  cudaMalloc(&x, 256ull << 20);
  cudaMalloc(&out, blocks * threads * 4);
  cudaMemset(x, 0, 256ull << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  printf("# random 4-byte gathers by all 148 SMs, %.0f M gathers per launch, warm (2 launches before)\n",
         gathers / 1e6);
  printf("%8s %12s %10s\n", "x_MB", "Ggathers/s", "ms");
  for (int mb : sizes_mb) {
    const uint32_t n = (uint32_t)((size_t)mb << 20) / 4;
    for (int w = 0; w < 2; ++w) gather_kernel<<<blocks, threads>>>(x, n, per_thread, 17u * w, out);
    cudaEventRecord(a);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) gather_kernel<<<blocks, threads>>>(x, n, per_thread, 101u + r, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    ms /= reps;
    printf("%8d %12.1f %10.4f\n", mb, gathers / (ms * 1e-3) / 1e9, ms);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
