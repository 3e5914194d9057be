// lsa_probe.cu — NCCL 2.28 device API on a 1-rank communicator: symmetric window (ncclMemAlloc +
// ncclCommWindowRegister), ncclDevComm with LSA barriers, in-kernel ncclGetLsaPointer loads/stores
// and ncclLsaBarrierSession; then whether lsaMultimem (NVLS) can be requested.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>
#include <cstdio>
#define NKC(x) do { ncclResult_t r = (x); if (r != ncclSuccess) { printf("FAIL %s: %s\n", #x, ncclGetErrorString(r)); } else printf("ok   %s\n", #x); } while (0)

__global__ void k(ncclDevComm dc, ncclWindow_t win, int n, float *out) {
  ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), blockIdx.x);
  bar.sync(ncclCoopCta(), cuda::memory_order_relaxed);
  float *p = (float *)ncclGetLsaPointer(win, 0, dc.lsaRank);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = 2.f * i;
  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
  float s = 0.f;
  for (int peer = 0; peer < dc.lsaSize; ++peer) {
    const float *q = (const float *)ncclGetLsaPointer(win, 0, peer);
    s += q[blockIdx.x * blockDim.x + threadIdx.x];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (blockIdx.x == 0 && threadIdx.x == 0) printf("device: rank %d nRanks %d lsaRank %d lsaSize %d\n", dc.rank, dc.nRanks, dc.lsaRank, dc.lsaSize);
}

int main() {
  ncclUniqueId id; NKC(ncclGetUniqueId(&id));
  ncclComm_t comm; NKC(ncclCommInitRank(&comm, 1, id, 0));
  const int n = 16 * 256;
  void *buf = nullptr; NKC(ncclMemAlloc(&buf, 1 << 20));
  ncclWindow_t win; NKC(ncclCommWindowRegister(comm, buf, 1 << 20, &win, NCCL_WIN_COLL_SYMMETRIC));
  ncclDevCommRequirements reqs = {}; reqs.lsaBarrierCount = 16;
  ncclDevComm dc; NKC(ncclDevCommCreate(comm, &reqs, &dc));
  float *out; cudaMalloc(&out, n * 4);
  k<<<16, 256>>>(dc, win, n, out);
  cudaError_t e = cudaDeviceSynchronize(); printf("kernel: %s\n", cudaGetErrorString(e));
  float h[8]; cudaMemcpy(h, out + 100, 32, cudaMemcpyDeviceToHost);
  printf("out[100..] %g %g (want %g %g)\n", h[0], h[1], 200.f, 202.f);
  ncclDevCommRequirements r2 = {}; r2.lsaBarrierCount = 4; r2.lsaMultimem = true;
  ncclDevComm dc2; NKC(ncclDevCommCreate(comm, &r2, &dc2));
  printf("LSA_PROBE %s\n", (e == cudaSuccess && h[0] == 200.f && h[1] == 202.f) ? "OK" : "FAIL");
  return 0;
}
