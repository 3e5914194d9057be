// gram_tc2.cuh — batched Gram G = H_g H_g^H on the tensor cores for U = 32 (sm_100a),
// reading H straight from HBM into UMMA operands (TMA, no SIMT operand build).
//
// Work item = (subcarrier, group): G = sum_{b in group} h_b h_b^H; PD groups are
// all local antennas (the first levels of the adder tree), FD groups are clusters.  With
// X = the fp32 rows of H viewed as nb x 64 reals (j = 2u + {0: re, 1: im}) and
// P = X^T X (64 x 64):
//     Re G[u][v] = P[2u][2v] + P[2u+1][2v+1],   Im G[u][v] = P[2u+1][2v] - P[2u][2v+1].
// 3xTF32:  P = Xb^T Xb + Xs^T Xb + (Xs^T Xb)^T  with Xb the raw fp32 tile read as tf32
// and Xs = X - trunc_tf32(X).  One kind::tf32 UMMA per 8 antennas computes the first two
// products: M = 128 with A = [Xb^T ; Xs^T], N = 64 with B = Xb^T.
//
// Operand layout: a chunk of CH antennas arrives by TMA as two boxes (reals 0..31 and
// 32..63) of CH rows x 128 B with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, which is directly
// an MN-major SWIZZLE_128B_BASE32B operand (M = reals, K = antennas; LBO = CH * 128 B
// between the 32-real atoms, SBO = 512 B between 4-antenna K groups).  The residual
// plane Xs is written right behind it in the same layout, so A = [Xb^T; Xs^T] is four
// equally spaced atoms and B = Xb^T the first two (only the residual plane is computed
// with SIMT instructions; an earlier version converted both planes).
//
// Persistent, warp-specialised, one CTA per SM (10 warps):
//   warp 8     TMA: CH-antenna chunks into an NS-stage ring (tx-count mbarriers);
//   warps 4-7  residual plane of each chunk;
//   warp 9     UMMA issue: CH/8 UMMAs per chunk into a double-buffered TMEM accumulator;
//   warps 0-3  epilogue per item: TMEM -> staging -> P = D1 + D2 + D2^T -> packed G.
#pragma once
#include "tcgen05.cuh"

// diagnostics only (scripts, never the shipped build): 1 = no UMMAs, 2 = no UMMAs and no residual math,
// 3 = 2 and no epilogue work (TMEM load, staging, G stores)
#ifndef DP_GRAM_DIAG
#define DP_GRAM_DIAG 0
#endif

namespace dpk {

// U = 32: 2 atoms of 32 reals per antenna row, M = 128, N = 64 (D rows = TMEM lanes);
// U = 16: 1 atom, M = 64, N = 32 (an M = 64 accumulator: D row r in lane 32 (r / 16) + r % 16).
template <int CH, int U> struct GT2 {
  static constexpr int NA = U / 16;                        // 32-real atoms per antenna row
  static constexpr int BOX = CH * 128;                     // one TMA box: CH rows x 32 fp32
  static constexpr int STAGE = 2 * NA * BOX;               // Xb (NA atoms) + Xs (NA atoms)
  static constexpr int NS = (U == 32 ? (CH == 64 ? 5 : 8) : (CH == 64 ? 10 : 16));   // 160 / 128 KB
  static constexpr int M = 4 * U, N = 2 * U;               // UMMA shape: A = [Xb^T; Xs^T], B = Xb^T
  static constexpr int LD = N + 4;                         // staging row stride (floats)
  static constexpr int THREADS = 320;
  static constexpr size_t SMEM = (size_t)NS * STAGE + M * LD * 4 + 1024;
};

template <int CH, int U>
__global__ void __launch_bounds__(GT2<CH, U>::THREADS, 1) gram_tc2_kernel(const __grid_constant__ CUtensorMap tmH, Args a) {
  pdl_trigger();   // early: the next kernel may launch once every CTA of this grid has started
                   // (it still waits for this grid's completion in griddepcontrol.wait)
  using T = GT2<CH, U>;
  extern __shared__ __align__(1024) uint8_t smem_dyn[];
  uint8_t *sm = smem_dyn + ((1024u - (tc::smem_u32(smem_dyn) & 1023u)) & 1023u);
  float *stg = reinterpret_cast<float *>(sm + (size_t)T::NS * T::STAGE);
  __shared__ __align__(8) uint64_t full[T::NS], prep_done[T::NS], stage_free[T::NS], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_items = a.n_sc * a.nchunks;          // (subcarrier, group); group = S antennas
  const int nck = a.S / CH;                        // chunks per item
  if (warp == 0) {
    tc::tmem_alloc(&tmem_base, 128);
    tc::tmem_relinquish();
  }
  if (tid == 32) {
    for (int i = 0; i < T::NS; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&prep_done[i], 128);
      tc::mbar_init(&stage_free[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&acc_full[i], 1);
      tc::mbar_init(&acc_empty[i], 128);
    }
    tc::fence_mbar_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tm = tmem_base;

  if (warp == 8) {
    // ------------------------------------------------------------ TMA producer
    // H is an input of the call (no predecessor kernel writes it): no griddepcontrol.wait
    if (lane == 0) {
      int s = 0, ph = 0, g = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        for (int c = 0; c < nck; ++c, ++g) {
          if (g >= T::NS) tc::mbar_wait(&stage_free[s], ph ^ 1);
          uint8_t *st = sm + (size_t)s * T::STAGE;
          const int row0 = item * a.S + c * CH;
          tc::mbar_arrive_expect_tx(&full[s], T::NA * T::BOX);
#pragma unroll
          for (int at = 0; at < T::NA; ++at) tc::tma_load_2d(st + at * T::BOX, &tmH, 32 * at, row0, &full[s]);
          if (++s == T::NS) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ UMMA issuer
    if (lane == 0) {
      constexpr uint32_t IDESC = tc::idesc_tf32(T::M, T::N) | (1u << 15) | (1u << 16);   // A, B MN-major
      int s = 0, ph = 0, g = 0, n = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++n) {
        const int b = n & 1;
        if (n >= 2) tc::mbar_wait(&acc_empty[b], ((n >> 1) - 1) & 1);
        const uint32_t d = tm + T::N * b;
        for (int c = 0; c < nck; ++c, ++g) {
          tc::mbar_wait(&prep_done[s], ph);
          tc::fence_after_sync();
          const uint32_t base = tc::smem_u32(sm + (size_t)s * T::STAGE);
#pragma unroll
          for (int t = 0; t < CH / 8; ++t) {                 // antennas 8t .. 8t+7
            const uint64_t dsc = smem_desc_mn_sw128b32(base + 1024 * t, T::BOX, 512);
            if (DP_GRAM_DIAG < 1) tc::mma_tf32(d, dsc, dsc, IDESC, (c > 0 || t > 0) ? 1u : 0u);
          }
          tc::mma_commit(&stage_free[s]);
          if (++s == T::NS) { s = 0; ph ^= 1; }
        }
        tc::mma_commit(&acc_full[b]);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ residual plane (warps 4-7)
    const int ptid = tid - 128;
    int s = 0, ph = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      for (int c = 0; c < nck; ++c) {
        tc::mbar_wait(&full[s], ph);
        uint8_t *st = sm + (size_t)s * T::STAGE;
        const uint4 *src = reinterpret_cast<const uint4 *>(st);
        uint4 *dst = reinterpret_cast<uint4 *>(st + T::NA * T::BOX);
        constexpr int NV = (DP_GRAM_DIAG >= 2) ? 0 : T::NA * T::BOX / 16 / 128;
        uint4 v[NV > 0 ? NV : 1];
#pragma unroll
        for (int i = 0; i < NV; ++i) v[i] = src[ptid + 128 * i];
#pragma unroll
        for (int i = 0; i < NV; ++i) {                        // Xs = X - trunc_tf32(X), same positions
          float4 f;
          f.x = __uint_as_float(v[i].x) - __uint_as_float(v[i].x & 0xFFFFE000u);
          f.y = __uint_as_float(v[i].y) - __uint_as_float(v[i].y & 0xFFFFE000u);
          f.z = __uint_as_float(v[i].z) - __uint_as_float(v[i].z & 0xFFFFE000u);
          f.w = __uint_as_float(v[i].w) - __uint_as_float(v[i].w & 0xFFFFE000u);
          dst[ptid + 128 * i] = *reinterpret_cast<uint4 *>(&f);
        }
        tc::fence_proxy_async();
        mbar_arrive(&prep_done[s]);
        if (++s == T::NS) { s = 0; ph ^= 1; }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 0-3)
    // D row r: r < 2U -> (Xb^T Xb)[r], r >= 2U -> (Xs^T Xb)[r - 2U]; TMEM lane of row r:
    // r (M = 128) or 32 (r / 16) + r % 16 (M = 64: lanes 16..31 of each quarter unused)
    pdl_wait();                                       // Gout may still be read by the predecessor
    constexpr int N = T::N;
    const int myrow = (T::M == 128) ? tid : (lane < 16 ? 16 * warp + lane : -1);
    int n = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++n) {
      const int b = n & 1;
      tc::mbar_wait(&acc_full[b], (n >> 1) & 1);
      tc::fence_after_sync();
      float d[N];
      const uint32_t ta = tm + N * b + ((uint32_t)(32 * warp) << 16);
#pragma unroll
      for (int cb = 0; cb < N / 16; ++cb) tc::tmem_ld16_nowait(ta + 16 * cb, *reinterpret_cast<float(*)[16]>(d + 16 * cb));
      tc::tmem_wait_ld();
      tc::fence_before_sync();
      mbar_arrive(&acc_empty[b]);                     // accumulator free for item n + 2
      named_sync(1, 128);                             // previous item done with the staging
      if (myrow >= 0) {
        float4 *row = reinterpret_cast<float4 *>(stg + myrow * T::LD);
#pragma unroll
        for (int j = 0; j < N / 4; ++j) row[j] = make_float4(d[4 * j], d[4 * j + 1], d[4 * j + 2], d[4 * j + 3]);
      }
      named_sync(1, 128);
      // P = D1 + D2 + D2^T ; D1 = stg rows 0..N-1, D2 = stg rows N..2N-1
      auto P = [&](int r, int q) {
        return stg[r * T::LD + q] + stg[(N + r) * T::LD + q] + stg[(N + q) * T::LD + r];
      };
      float2 *out = a.Gout + (size_t)item * npacked(U);
#pragma unroll 2
      for (int e = tid; e < (DP_GRAM_DIAG >= 3 ? 0 : U * U); e += 128) {
        const int u = e / U, v = e % U;
        if (u <= v) {
          const float gr = P(2 * u, 2 * v) + P(2 * u + 1, 2 * v + 1);
          const float gi = P(2 * u + 1, 2 * v) - P(2 * u, 2 * v + 1);
          out[pidx(U, u, v)] = make_float2(gr, gi);
        }
      }
    }
  }
  pdl_trigger();
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tm, 128);
}

}  // namespace dpk
