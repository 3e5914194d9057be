// tma_probe.cu — experiment (not part of libdp.so): TMA 2-D SWIZZLE_128B tile of a
// fp32 [R][64] matrix used directly as a tf32 K-major UMMA operand (M = 128, K = 32),
// optionally with a 3xTF32-style residual plane A_s = A - trunc_tf32(A).
#include <cuda.h>
#include <cudaTypedefs.h>
#include "tcgen05.cuh"

__global__ void probe(const __grid_constant__ CUtensorMap tmap, const float *B, float *D, int row0, int col0,
                      int split) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sa = sm;                 // 128 rows x 128 B, swizzled (16 KB)
  uint8_t *ss = sm + 16384;         // residual plane, same layout
  uint8_t *sb = sm + 32768;         // B: 64 rows x 32 K, interleaved K-major (8 KB)
  __shared__ __align__(8) uint64_t bar, mbar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, w = tid / 32, lane = tid % 32;
  if (w == 0) { tc::tmem_alloc(&tbase, 64); tc::tmem_relinquish(); }
  if (tid == 32) { tc::mbar_init(&bar, 1); tc::mbar_init(&mbar, 1); tc::fence_mbar_init(); }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (tid == 0) {
    tc::mbar_arrive_expect_tx(&bar, 16384);
    tc::tma_load_2d(sa, &tmap, col0, row0, &bar);
  }
  for (int i = tid; i < 64 * 32; i += blockDim.x) {
    const int r = i / 32, k = i % 32;
    *reinterpret_cast<float *>(sb + tc::kmaj_off(64, r, k)) = B[i];
  }
  tc::mbar_wait(&bar, 0);
  for (int i = tid; i < 16384 / 4; i += blockDim.x) {   // residual, elementwise (layout-agnostic)
    const float x = reinterpret_cast<const float *>(sa)[i];
    const float big = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
    reinterpret_cast<float *>(ss)[i] = x - big;
  }
  tc::fence_proxy_async();
  __syncthreads();
  const uint32_t tm = tbase;
  if (tid == 0) {
    tc::fence_after_sync();
    const uint32_t idesc = tc::idesc_tf32(128, 64);
    for (int t = 0; t < 4; ++t) {
      const uint64_t bd = tc::smem_desc(tc::smem_u32(sb) + t * 2 * 64 * 16, 64 * 16, 128);
      tc::mma_tf32(tm, tc::smem_desc_sw128(tc::smem_u32(sa) + 32 * t, 1024), bd, idesc, t > 0);
      if (split) tc::mma_tf32(tm, tc::smem_desc_sw128(tc::smem_u32(ss) + 32 * t, 1024), bd, idesc, 1);
    }
    tc::mma_commit(&mbar);
  }
  tc::mbar_wait(&mbar, 0);
  tc::fence_after_sync();
  for (int c = 0; c < 64; c += 16) {
    float v[16];
    tc::tmem_ld16(tm + ((uint32_t)(32 * w) << 16) + c, v);
    for (int j = 0; j < 16; ++j) D[(32 * w + lane) * 64 + c + j] = v[j];
  }
  tc::fence_before_sync();
  __syncthreads();
  if (w == 0) tc::tmem_dealloc(tm, 64);
}

extern "C" int tma_probe(const float *A, int R, const float *B, float *D, int row0, int col0, int split) {
  PFN_cuTensorMapEncodeTiled encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&encode, cudaEnableDefault, &q) != cudaSuccess ||
      !encode)
    return -1;
  CUtensorMap tmap;
  cuuint64_t dims[2] = {64, (cuuint64_t)R};
  cuuint64_t strides[1] = {64 * 4};
  cuuint32_t box[2] = {32, 128};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)A, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return -2 - (int)r;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  probe<<<1, 128, 48 * 1024>>>(tmap, B, D, row0, col0, split);
  return (int)cudaDeviceSynchronize();
}
