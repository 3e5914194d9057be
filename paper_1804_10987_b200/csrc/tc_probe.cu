// tc_probe.cu — experiment harness for the tcgen05 helpers (not part of libdp.so):
// D[64][64] = A[64][K] * B[64][K]^T with kind::tf32 UMMA, operands staged in the
// interleaved K-major layout of tcgen05.cuh.  mode bit 0 swaps LBO/SBO (convention probe).
#include "tcgen05.cuh"

__global__ void probe_kernel(const float *A, const float *B, float *D, int K, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  uint8_t *sa = sm, *sb = sm + 64 * K * 4;
  for (int i = threadIdx.x; i < 64 * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<uint32_t *>(sa + tc::kmaj_off(64, r, k)) = tc::to_tf32(A[i]);
    *reinterpret_cast<uint32_t *>(sb + tc::kmaj_off(64, r, k)) = tc::to_tf32(B[i]);
  }
  tc::fence_proxy_async();
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (w == 0) {
    tc::tmem_alloc(&tbase, 64);
    tc::tmem_relinquish();
  }
  if (threadIdx.x == 32) {
    tc::mbar_init(&mbar, 1);
    tc::fence_mbar_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tm = tbase;
  const uint32_t lbo = (mode & 1) ? 128u : 64u * 16u, sbo = (mode & 1) ? 64u * 16u : 128u;
  if (threadIdx.x == 0) {
    for (int t = 0; t < K / 8; ++t) {
      const uint64_t ad = tc::smem_desc(tc::smem_u32(sa) + 2 * t * 64 * 16, lbo, sbo);
      const uint64_t bd = tc::smem_desc(tc::smem_u32(sb) + 2 * t * 64 * 16, lbo, sbo);
      tc::mma_tf32(tm, ad, bd, tc::idesc_tf32(64, 64), t > 0 ? 1u : 0u);
    }
    tc::mma_commit(&mbar);
  }
  tc::mbar_wait(&mbar, 0);
  tc::fence_after_sync();
  if (w < 4) {
    for (int c = 0; c < 64; c += 16) {
      float v[16];
      tc::tmem_ld16(tm + ((uint32_t)(32 * w) << 16) + c, v);
      for (int j = 0; j < 16; ++j) D[(size_t)(64 * 64) * 1 * (lane >= 16) + (16 * w + (lane & 15)) * 64 + c + j] = v[j];
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (w == 0) tc::tmem_dealloc(tm, 64);
}

extern "C" int tc_probe(const float *A, const float *B, float *D, int K, int mode) {
  const size_t sm = (size_t)2 * 64 * K * 4;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  probe_kernel<<<1, 128, sm>>>(A, B, D, K, mode);
  cudaError_t e = cudaDeviceSynchronize();
  return (int)e;
}
