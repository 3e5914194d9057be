// tc_probe.cu — experiment harness for the tcgen05 helpers (not part of libdp.so):
// D[64][64] = A[64][K] * B[64][K]^T with kind::tf32 UMMA, operands staged in the
// interleaved K-major layout of tcgen05.cuh.  mode bit 0 swaps LBO/SBO (convention probe).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -I paper_1804_10987_b200/csrc
//        scripts/tc_probe.cu -o paper_1804_10987_b200/libtcprobe.so -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
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

// MN-major SWIZZLE_128B probe: X [32 rows][64] fp32 row-major placed like the TMA
// SW128 boxes (cols 0..31 at +0, 32..63 at +4096; row r at 128 r; 16-byte chunk c at
// (c ^ r % 8)); D = X^T X via 4 UMMAs (M = N = 64, K = 8), A = B = MN-major desc.
// mode bit 0: swap LBO/SBO; bit 1: clear the transpose bits.
__global__ void mn_probe_kernel(const float *X, float *D, int mode) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 32 * 64; i += blockDim.x) {
    const int r = i / 64, col = i % 64, box = col / 32, cc = col % 32, ch = cc / 4;
    *reinterpret_cast<float *>(sm + box * 4096 + r * 128 + ((ch ^ (r & 7)) << 4) + (cc & 3) * 4) = X[i];
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
  const uint32_t lbo = (mode & 1) ? 1024u : 4096u, sbo = (mode & 1) ? 4096u : 1024u;
  uint32_t idesc = tc::idesc_tf32(64, 64);
  if (!(mode & 2)) idesc |= (1u << 15) | (1u << 16);
  if (threadIdx.x == 0) {
    for (int t = 0; t < 4; ++t) {
      uint64_t d = 0;
      const uint32_t sa = tc::smem_u32(sm) + 1024 * t;
      d |= (uint64_t)((sa >> 4) & 0x3FFF);
      d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
      d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
      d |= (uint64_t)1 << 46;
      d |= (uint64_t)2 << 61;
      tc::mma_tf32(tm, d, d, idesc, t > 0 ? 1u : 0u);
    }
    tc::mma_commit(&mbar);
  }
  tc::mbar_wait(&mbar, 0);
  tc::fence_after_sync();
  if (w < 4) {
    for (int c = 0; c < 64; c += 16) {
      float v[16];
      tc::tmem_ld16(tm + ((uint32_t)(32 * w) << 16) + c, v);
      for (int j = 0; j < 16; ++j) D[(32 * w + lane) * 64 + c + j] = v[j];   // all 128 lanes
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (w == 0) tc::tmem_dealloc(tm, 64);
}

extern "C" int mn_probe(const float *X, float *D, int mode) {
  cudaFuncSetAttribute(mn_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  mn_probe_kernel<<<1, 128, 16384>>>(X, D, mode);
  return (int)cudaDeviceSynchronize();
}

// MN-major tf32 probe #2: TMA (swizzle mode `sw`) two boxes {32 fp32, 32 rows} of X
// [32][64] into smem, dump the smem bytes, then D = X^T X with UMMA layout type `lt`,
// LBO/SBO given.
__global__ void mn_probe2_kernel(const __grid_constant__ CUtensorMap tm_x, float *dump, float *D, int lt,
                                 uint32_t lbo, uint32_t sbo, int kgrp) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full, mbar;
  __shared__ uint32_t tbase;
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (w == 0) {
    tc::tmem_alloc(&tbase, 64);
    tc::tmem_relinquish();
  }
  if (threadIdx.x == 32) {
    tc::mbar_init(&mbar, 1);
    tc::mbar_init(&full, 1);
    tc::fence_mbar_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (threadIdx.x == 0) {
    tc::mbar_arrive_expect_tx(&full, 8192);
    tc::tma_load_2d(sm, &tm_x, 0, 0, &full);
    tc::tma_load_2d(sm + 4096, &tm_x, 32, 0, &full);
  }
  tc::mbar_wait(&full, 0);
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) dump[i] = reinterpret_cast<const float *>(sm)[i];
  const uint32_t tm = tbase;
  uint32_t idesc = tc::idesc_tf32(64, 64) | (1u << 15) | (1u << 16);
  if (threadIdx.x == 0) {
    for (int t = 0; t < 4; ++t) {       // K = 8 per UMMA: rows 8t .. 8t+7 start at 8t * 128 bytes
      uint64_t d = 0;
      const uint32_t sa = tc::smem_u32(sm) + 1024 * t;
      d |= (uint64_t)((sa >> 4) & 0x3FFF);
      d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
      d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
      d |= (uint64_t)1 << 46;
      d |= (uint64_t)(lt & 7) << 61;
      tc::mma_tf32(tm + ((uint32_t)kgrp << 16), d, d, idesc, t > 0 ? 1u : 0u);
    }
    tc::mma_commit(&mbar);
  }
  tc::mbar_wait(&mbar, 0);
  tc::fence_after_sync();
  if (w < 4) {
    for (int c = 0; c < 64; c += 16) {
      float v[16];
      tc::tmem_ld16(tm + ((uint32_t)(32 * w) << 16) + c, v);
      for (int j = 0; j < 16; ++j) D[(32 * w + lane) * 64 + c + j] = v[j];
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (w == 0) tc::tmem_dealloc(tm, 64);
}

extern "C" int mn_probe2(const float *X, float *dump, float *D, int sw, int lt, unsigned lbo, unsigned sbo, int lane_off) {
  static PFN_cuTensorMapEncodeTiled encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&encode, cudaEnableDefault, &q) != cudaSuccess) return -1;
  }
  CUtensorMap tm;
  cuuint64_t dims[2] = {64, 32};
  cuuint64_t strides[1] = {64 * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)X, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, (CUtensorMapSwizzle)sw, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return -2;
  cudaFuncSetAttribute(mn_probe2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  mn_probe2_kernel<<<1, 128, 16384>>>(tm, dump, D, lt, lbo, sbo, lane_off);
  return (int)cudaDeviceSynchronize();
}

extern "C" int tc_probe(const float *A, const float *B, float *D, int K, int mode) {
  const size_t sm = (size_t)2 * 64 * K * 4;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  probe_kernel<<<1, 128, sm>>>(A, B, D, K, mode);
  cudaError_t e = cudaDeviceSynchronize();
  return (int)e;
}
