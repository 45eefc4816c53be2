// Probe: does this B200 box support NVSwitch multicast (NVLS) objects, and does a kernel's
// multimem.st through a multicast mapping land in the bound (unicast) buffer?  One device in the
// multicast group (the gpurun box has one GPU); with N ranks the same store reaches N buffers.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#define DR(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s = nullptr; cuGetErrorString(r, &s); \
  printf("FAIL %s -> %d %s\n", #x, (int)r, s ? s : "?"); return 1; } } while (0)
#define RT(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("FAIL %s -> %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void mc_store(float* mc, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) asm volatile("multimem.st.global.f32 [%0], %1;" ::"l"(mc + i), "f"(1.5f * i) : "memory");
}

int main() {
  DR(cuInit(0));
  CUdevice dev;
  DR(cuDeviceGet(&dev, 0));
  CUcontext ctx;
  RT(cudaSetDevice(0));
  RT(cudaFree(0));
  DR(cuCtxGetCurrent(&ctx));
  int mc = 0, fab = 0, vmm = 0, posix = 0;
  DR(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  DR(cuDeviceGetAttribute(&vmm, CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED, dev));
  DR(cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev));
  DR(cuDeviceGetAttribute(&posix, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, dev));
  printf("multicast_supported=%d vmm=%d fabric_handles=%d posix_fd_handles=%d\n", mc, vmm, fab, posix);
  if (!mc) return 0;
  const int n = 1 << 20;
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  mp.size = (size_t)n * 4;
  DR(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  mp.size = (mp.size + gran - 1) / gran * gran;
  printf("mc granularity %zu size %zu\n", gran, mp.size);
  size_t gmin = 0;
  DR(cuMulticastGetGranularity(&gmin, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
  printf("mc minimum granularity %zu\n", gmin);
  CUmemGenericAllocationHandle mch;
  const unsigned types[3] = {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_FABRIC, CU_MEM_HANDLE_TYPE_NONE};
  CUresult cr = CUDA_ERROR_UNKNOWN;
  for (unsigned t : types) {
    for (size_t szc : {(size_t)gmin, mp.size}) {
      CUmulticastObjectProp q = mp;
      q.handleTypes = t;
      q.size = (((size_t)n * 4) + szc - 1) / szc * szc;
      cr = cuMulticastCreate(&mch, &q);
      const char* es = nullptr; cuGetErrorString(cr, &es);
      printf("cuMulticastCreate(numDevices=1, handleTypes=%u, size=%zu) -> %d %s\n", t, q.size, (int)cr, es ? es : "?");
      if (cr == CUDA_SUCCESS) { mp = q; break; }
    }
    if (cr == CUDA_SUCCESS) break;
  }
  if (cr != CUDA_SUCCESS) return 1;
  gran = mp.size;
  DR(cuMulticastAddDevice(mch, dev));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = dev;
  ap.requestedHandleTypes = (CUmemAllocationHandleType)mp.handleTypes;
  size_t ug = 0;
  DR(cuMemGetAllocationGranularity(&ug, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  const size_t sz = (mp.size + ug - 1) / ug * ug;
  CUmemGenericAllocationHandle uh;
  DR(cuMemCreate(&uh, sz, &ap, 0));
  DR(cuMulticastBindMem(mch, 0, uh, 0, mp.size, 0));
  CUdeviceptr uva, mva;
  DR(cuMemAddressReserve(&uva, sz, ug, 0, 0));
  DR(cuMemMap(uva, sz, 0, uh, 0));
  CUmemAccessDesc ad = {};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = dev;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  DR(cuMemSetAccess(uva, sz, &ad, 1));
  DR(cuMemAddressReserve(&mva, mp.size, gran, 0, 0));
  DR(cuMemMap(mva, mp.size, 0, mch, 0));
  DR(cuMemSetAccess(mva, mp.size, &ad, 1));
  RT(cudaMemset((void*)uva, 0, (size_t)n * 4));
  mc_store<<<(n + 255) / 256, 256>>>((float*)mva, n);
  RT(cudaGetLastError());
  RT(cudaDeviceSynchronize());
  float* h = new float[n];
  RT(cudaMemcpy(h, (void*)uva, (size_t)n * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int i = 0; i < n; ++i) bad += h[i] != 1.5f * i;
  printf("multimem.st through the multicast mapping: %d of %d values wrong\n", bad, n);
  // bandwidth of multimem.st (1 device)
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 20; ++r) mc_store<<<(n + 255) / 256, 256>>>((float*)mva, n);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  printf("multimem.st 4 MB x 20: %.3f ms per pass (%.1f GB/s)\n", ms / 20, 4.0 * n / (ms / 20) / 1e6);
  return bad != 0;
}
