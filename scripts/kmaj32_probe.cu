// kmaj32_probe.cu — does a K-major tf32 UMMA operand accept the SWIZZLE_128B_BASE32B smem layout
// (descriptor layout type 1) that the TMA writes with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B?
// If yes, one shared-memory copy of an H tile is both the MN-major Gram operand (fd_tc.cuh) and the
// K-major precode operand (contraction over the users).  Not part of libdp.so.
//
// X [128][32] fp32 (rows = M, 32 = K), Y [32][32] (rows = N); both TMA-loaded with ATOM_32B into smem;
// D = X Y^T with 4 UMMAs (M = 128, N = 32, K = 8 each, start address + 32 B per K step), layout type
// `lt`, SBO `sbo`, LBO `lbo`.  Build / run: scripts/kmaj32_probe.sh (GPU box).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include "tcgen05.cuh"

__global__ void kprobe_kernel(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap ty, float *D,
                              int lt, int lbo, int sbo) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t *sm = smraw + ((1024u - (tc::smem_u32(smraw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full, done;
  __shared__ uint32_t tbase;
  uint8_t *sx = sm, *sy = sm + 16384;
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    tc::mbar_init(&full, 1);
    tc::mbar_init(&done, 1);
    tc::fence_mbar_init();
    tc::mbar_arrive_expect_tx(&full, 16384 + 4096);
    tc::tma_load_2d(sx, &tx, 0, 0, &full);
    tc::tma_load_2d(sy, &ty, 0, 0, &full);
  }
  if (w == 0) {
    tc::tmem_alloc(&tbase, 32);
    tc::tmem_relinquish();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    tc::mbar_wait(&full, 0);
    for (int t = 0; t < 4; ++t) {
      auto desc = [&](uint32_t a) {
        uint64_t d = 0;
        d |= (uint64_t)((a >> 4) & 0x3FFF);
        d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
        d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
        d |= (uint64_t)1 << 46;
        d |= (uint64_t)(lt & 7) << 61;
        return d;
      };
      tc::mma_tf32(tm, desc(tc::smem_u32(sx) + 32 * t), desc(tc::smem_u32(sy) + 32 * t), tc::idesc_tf32(128, 32),
                   t > 0 ? 1u : 0u);
    }
    tc::mma_commit(&done);
  }
  __syncwarp();
  tc::mbar_wait(&done, 0);
  tc::fence_after_sync();
  float v[16];
  for (int c = 0; c < 32; c += 16) {
    tc::tmem_ld16(tm + ((uint32_t)(32 * w) << 16) + c, v);
    for (int j = 0; j < 16; ++j) D[(32 * w + lane) * 32 + c + j] = v[j];
  }
  tc::fence_before_sync();
  __syncthreads();
  if (w == 0) tc::tmem_dealloc(tm, 32);
}

static PFN_cuTensorMapEncodeTiled enc() {
  static PFN_cuTensorMapEncodeTiled f = nullptr;
  if (!f) {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&f, cudaEnableDefault, &q);
  }
  return f;
}
static void tmap(CUtensorMap *m, const float *p, int rows, CUtensorMapSwizzle sw) {
  cuuint64_t dims[2] = {32, (cuuint64_t)rows};
  cuuint64_t strides[1] = {32 * 4};
  cuuint32_t box[2] = {32, (cuuint32_t)rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     sw, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
}

// swz: 0 = SWIZZLE_128B_ATOM_32B (TMA), 1 = SWIZZLE_128B
extern "C" int kprobe(const float *X, const float *Y, float *D, int swz, int lt, int lbo, int sbo) {
  CUtensorMap tx, ty;
  const CUtensorMapSwizzle sw = swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
  tmap(&tx, X, 128, sw);
  tmap(&ty, Y, 32, sw);
  cudaFuncSetAttribute(kprobe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 24576);
  kprobe_kernel<<<1, 128, 24576>>>(tx, ty, D, lt, lbo, sbo);
  return (int)cudaDeviceSynchronize();
}
