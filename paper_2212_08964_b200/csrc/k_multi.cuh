// k_multi.cuh -- sm_100a device code of the multi-GPU layer (arXiv 2212.08964 P:2187-2192).
// The replica checksum of SURVEY 8(c) p10 and the column remap of the padded all-gather layout.
#pragma once
#include "dev_common.cuh"

namespace lbk {

// splitmix64 finaliser (Steele et al.): a bijective 64-bit mixer
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// out += sum_i mix64(i * 0x9E3779B97F4A7C15 + bits(y_i)) mod 2^64 (order-free, so the parallel sum is
// deterministic; position-dependent, so permuted values differ; bitwise, so -0 != +0).  *out zeroed
// by the caller.  lb_y_checksum documents the same formula for host-side checks.
__global__ void __launch_bounds__(256) checksum_kernel(const float* __restrict__ y, int64_t n,
                                                       unsigned long long* __restrict__ out) {
  uint64_t h = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    h += mix64((uint64_t)i * 0x9E3779B97F4A7C15ull + (uint64_t)__float_as_uint(__ldg(y + i)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(kFull, h, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, (unsigned long long)h);
}

// Padded all-gather layout (SURVEY 8(e) option 2): global column c of shard k = the largest k with
// bounds[k] <= c becomes k * P + (c - bounds[k]).  bounds: int64[nranks + 1] in device memory.
__global__ void __launch_bounds__(256) remap_cols_padded_kernel(const int* __restrict__ col, int64_t nnz,
                                                                const int64_t* __restrict__ bounds, int nranks,
                                                                int64_t P, int* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += stride) {
    const int64_t c = __ldg(col + k);
    int lo = 0, hi = nranks - 1;  // last shard whose first row is <= c
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (__ldg(bounds + mid) <= c) lo = mid; else hi = mid - 1;
    }
    out[k] = (int)(lo * P + (c - __ldg(bounds + lo)));
  }
}

}  // namespace lbk
