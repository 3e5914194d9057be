// nvls_probe.cu — does this box support NVLink SHARP multicast objects for ONE device?
// Creates a multicast object over this GPU, binds a physical allocation, and checks
// multimem.st / multimem.ld_reduce through the multicast address against plain loads.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#define CKD(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char *s; cuGetErrorString(r, &s); printf("FAIL %s: %s\n", #x, s); return 1; } } while (0)

__global__ void mm_kernel(float *mc, float *uc, float *out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n / 4) return;
  float4 v = make_float4(1.f * i, 2.f * i, 3.f * i, 4.f * i);
  asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + 4 * i), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
  asm volatile("fence.proxy.alias;" ::: "memory");
  __syncthreads();
  float4 r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(mc + 4 * i) : "memory");
  reinterpret_cast<float4 *>(out)[i] = r;
}

int main() {
  CKD(cuInit(0));
  CUdevice dev; CKD(cuDeviceGet(&dev, 0));
  int mcs = 0; CKD(cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  printf("MULTICAST_SUPPORTED %d\n", mcs);
  CUcontext ctx; CKD(cuDevicePrimaryCtxRetain(&ctx, dev)); CKD(cuCtxSetCurrent(ctx));
  const size_t n = 1 << 20, bytes = n * 4;
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1; mp.size = bytes; mp.handleTypes = (CUmemAllocationHandleType)(getenv("MC_HT") ? atoi(getenv("MC_HT")) : 0);
  size_t gran = 0; CKD(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  mp.size = ((bytes + gran - 1) / gran) * gran;
  printf("granularity %zu size %zu\n", gran, mp.size);
  CUmemGenericAllocationHandle mch; CKD(cuMulticastCreate(&mch, &mp));
  CKD(cuMulticastAddDevice(mch, dev));
  CUmemAllocationProp ap = {}; ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ap.location.id = 0;
  ap.requestedHandleTypes = mp.handleTypes;
  size_t ag = 0; CKD(cuMemGetAllocationGranularity(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  CUmemGenericAllocationHandle ph; CKD(cuMemCreate(&ph, mp.size, &ap, 0));
  CKD(cuMulticastBindMem(mch, 0, ph, 0, mp.size, 0));
  CUdeviceptr uc, mc;
  CKD(cuMemAddressReserve(&uc, mp.size, ag, 0, 0)); CKD(cuMemMap(uc, mp.size, 0, ph, 0));
  CKD(cuMemAddressReserve(&mc, mp.size, gran, 0, 0)); CKD(cuMemMap(mc, mp.size, 0, mch, 0));
  CUmemAccessDesc ad = {}; ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ad.location.id = 0; ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CKD(cuMemSetAccess(uc, mp.size, &ad, 1)); CKD(cuMemSetAccess(mc, mp.size, &ad, 1));
  float *out; cudaMalloc(&out, bytes);
  mm_kernel<<<(n / 4 + 255) / 256, 256>>>((float *)mc, (float *)uc, out, n);
  cudaError_t e = cudaDeviceSynchronize(); printf("kernel: %s\n", cudaGetErrorString(e));
  float *h = new float[n], *hu = new float[n];
  cudaMemcpy(h, out, bytes, cudaMemcpyDeviceToHost); cudaMemcpy(hu, (void *)uc, bytes, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (size_t i = 0; i < n; ++i) { float want = (float)((i % 4) + 1) * (float)(i / 4); if (h[i] != want || hu[i] != want) ++bad; }
  printf("multimem st/ld_reduce mismatches: %d of %zu  (e.g. %g %g)\n", bad, n, h[12], hu[12]);
  printf("NVLS_PROBE %s\n", bad == 0 && e == cudaSuccess ? "OK" : "FAIL");
  return 0;
}
