// precode_tc.cuh — tensor-core (tcgen05 / TMEM / TMA) precode x_c = H_c^H z for U = 32.
//
// Per antenna b and symbol k:  x[k][b] = sum_u conj(H[b][u]) z[k][u].
// With the interleaved real index j = 2u + {0: re, 1: im}, H's fp32 row is used as is:
//     Re x[k][b] = sum_j H[b][j] Zr[k][j],  Zr[k][2u] = Re z[k][u],  Zr[k][2u+1] = Im z[k][u]
//     Im x[k][b] = sum_j H[b][j] Zi[k][j],  Zi[k][2u] = Im z[k][u],  Zi[k][2u+1] = -Re z[k][u]
// so D = Z H^T is one real GEMM: A = Z (16 Re-rows, 16 Im-rows), K = 64, B = the 32
// antenna rows of one block (N = 32).  3xTF32 (all 4 products, summed by the tensor
// core): A = [Zb ; Zs] (M = 64: big rows 0..31, small rows 32..63) and B = Hb + Hs,
// where Hb is the raw fp32 H row consumed as tf32 (the tensor core reads its top 19
// bits) and Hs = H - trunc_tf32(H) is computed elementwise; both UMMAs accumulate
// into one TMEM tile and x = D[0:32] + D[32:64].
//
// A work item is 64 antennas (2 blocks of 32) of one subcarrier; block j uses z
// group zg (PD: the subcarrier's z; FD: cluster 2 item + j, S = 32).  Stage layout
// (x2): H raw boxes (2 K-halves, 64 rows x 128 B, SWIZZLE_128B by TMA), H residual,
// the z rows (TMA bulk copy), two Z operands.
// Warp roles (10 warps, 1 CTA per SM): 0-3 epilogue (their TMEM lane quarters),
// 4-7 operand prep (residual + Z), 8 TMA, 9 UMMA issue.  Hand-offs are mbarriers:
// full (TMA tx bytes) -> prep_done (128) -> stage_free (UMMA commit), and
// acc_full (commit) / acc_empty (128) for the double-buffered TMEM accumulators.
#pragma once
#include "tcgen05.cuh"

namespace dpk {

constexpr int TCP_ROWS = 64;                            // antennas per item
constexpr int TCP_NS = 3;                               // stages
constexpr int TCP_HB = TCP_ROWS * 128;                  // one TMA box: 64 rows x 128 B = 8 KB
constexpr int TCP_ZRAW = 2 * 16 * 32 * 8;               // z rows of up to 2 groups, K <= 16: 8 KB
constexpr int TCP_Z = 64 * 64 * 4;                      // one Z operand (64 rows x 64 K, interleaved) = 16 KB
constexpr int TCP_STAGE = 4 * TCP_HB + TCP_ZRAW + 2 * TCP_Z;   // 72 KB
constexpr int TCP_STG_LD = 33;
constexpr int TCP_THREADS = 320;
constexpr size_t TCP_SMEM = (size_t)TCP_NS * TCP_STAGE + 64 * TCP_STG_LD * 4 + 1024;

__global__ void __launch_bounds__(TCP_THREADS, 1) precode_tc_kernel(const __grid_constant__ CUtensorMap tmH, Args a) {
  pdl_wait();
  extern __shared__ __align__(1024) uint8_t smem_dyn[];
  // align by an offset (not integer casts) so the compiler keeps the shared state space: LDS, not LD
  uint8_t *sm = smem_dyn + ((1024u - (tc::smem_u32(smem_dyn) & 1023u)) & 1023u);
  float *stg = reinterpret_cast<float *>(sm + (size_t)TCP_NS * TCP_STAGE);
  __shared__ __align__(8) uint64_t full[TCP_NS], prep_done[TCP_NS], stage_free[TCP_NS], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base;
  __shared__ float pw_part[2][4];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int items_per_sc = a.Bl / TCP_ROWS;
  const int n_items = a.n_sc * items_per_sc;
  const bool per_block = a.zgroups > 1;
  const int nz = per_block ? 2 : 1;
  const uint32_t zbytes = (uint32_t)nz * a.K * 32 * 8;
  if (warp == 0) {
    tc::tmem_alloc(&tmem_base, 128);
    tc::tmem_relinquish();
  }
  if (tid == 32) {
    for (int i = 0; i < TCP_NS; ++i) {
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
  auto stage = [&](int s) { return sm + (size_t)s * TCP_STAGE; };

  if (warp == 8) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int s = 0, ph = 0, n = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++n) {
        if (n >= TCP_NS) tc::mbar_wait_sleep(&stage_free[s], ph ^ 1);
        const int sc = item / items_per_sc, blk = item % items_per_sc;
        const int row0 = sc * a.Bl + blk * TCP_ROWS;
        uint8_t *st = stage(s);
        tc::mbar_arrive_expect_tx(&full[s], 2 * TCP_HB + zbytes);
        tc::tma_load_2d(st, &tmH, 0, row0, &full[s]);
        tc::tma_load_2d(st + TCP_HB, &tmH, 32, row0, &full[s]);
        const float2 *z = a.zin + ((size_t)sc * a.zgroups + (per_block ? 2 * blk : 0)) * a.K * 32;
        tc::bulk_g2s(st + 4 * TCP_HB, z, zbytes, &full[s]);
        if (++s == TCP_NS) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ UMMA issuer
    if (lane == 0) {
      constexpr uint32_t IDESC = tc::idesc_tf32(64, 32);
      int s = 0, ph = 0, n = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++n) {
        const int b = n & 1;
        if (n >= 2) tc::mbar_wait_sleep(&acc_empty[b], ((n >> 1) - 1) & 1);
        tc::mbar_wait_sleep(&prep_done[s], ph);
        tc::fence_after_sync();
        const uint32_t hb = tc::smem_u32(stage(s));
        const uint32_t zb = hb + 4 * TCP_HB + TCP_ZRAW;
#pragma unroll
        for (int j = 0; j < 2; ++j) {                     // 32-antenna block j -> TMEM columns 64 b + 32 j
          const uint32_t za = zb + (uint32_t)(per_block ? j : 0) * TCP_Z;
          const uint32_t d = tm + 64 * b + 32 * j;
#pragma unroll
          for (int t = 0; t < 8; ++t) {                   // K = 64 reals in 8 steps of 8
            const uint64_t ad = tc::smem_desc(za + t * 2 * 64 * 16, 64 * 16, 128);
            const uint32_t koff = (uint32_t)(t >> 2) * TCP_HB + (uint32_t)(t & 3) * 32 + (uint32_t)j * 32 * 128;
            tc::mma_tf32(d, ad, tc::smem_desc_sw128(hb + koff, 1024), IDESC, t > 0 ? 1u : 0u);
            tc::mma_tf32(d, ad, tc::smem_desc_sw128(hb + 2 * TCP_HB + koff, 1024), IDESC, 1u);
          }
        }
        tc::mma_commit(&stage_free[s]);
        tc::mma_commit(&acc_full[b]);
        if (++s == TCP_NS) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ operand prep (warps 4-7)
    const int ptid = tid - 128;
    int s = 0, ph = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      tc::mbar_wait(&full[s], ph);
      uint8_t *st = stage(s);
      {  // residual plane Hs = H - trunc_tf32(H) (elementwise on the swizzled boxes)
        const uint4 *src = reinterpret_cast<const uint4 *>(st);
        uint4 *dst = reinterpret_cast<uint4 *>(st + 2 * TCP_HB);
#pragma unroll
        for (int i = 0; i < 2 * TCP_HB / 16 / 128; ++i) {
          const int e = ptid + 128 * i;
          const uint4 v = src[e];
          float4 f;
          f.x = __uint_as_float(v.x) - __uint_as_float(v.x & 0xFFFFE000u);
          f.y = __uint_as_float(v.y) - __uint_as_float(v.y & 0xFFFFE000u);
          f.z = __uint_as_float(v.z) - __uint_as_float(v.z & 0xFFFFE000u);
          f.w = __uint_as_float(v.w) - __uint_as_float(v.w & 0xFFFFE000u);
          dst[e] = *reinterpret_cast<uint4 *>(&f);
        }
      }
      {  // Z operands: rows 0..15 Re-rows k, 16..31 Im-rows k (big), +32 small; cols j = 2u + {0,1}
        const float2 *zr = reinterpret_cast<const float2 *>(st + 4 * TCP_HB);
        for (int jz = 0; jz < nz; ++jz) {
          uint8_t *zo = st + 4 * TCP_HB + TCP_ZRAW + (size_t)jz * TCP_Z;
#pragma unroll 2
          for (int i = 0; i < 8; ++i) {
            const int e = ptid + 128 * i, r = e >> 5, u = e & 31, k = r & 15;
            const float2 v = (k < a.K) ? zr[((size_t)jz * a.K + k) * 32 + u] : make_float2(0.f, 0.f);
            const float c0 = (r < 16) ? v.x : v.y, c1 = (r < 16) ? v.y : -v.x;
            const uint32_t b0 = tc::to_tf32(c0), b1 = tc::to_tf32(c1);
            const uint32_t s0 = tc::to_tf32(c0 - __uint_as_float(b0)), s1 = tc::to_tf32(c1 - __uint_as_float(b1));
            *reinterpret_cast<uint2 *>(zo + tc::kmaj_off(64, r, 2 * u)) = make_uint2(b0, b1);
            *reinterpret_cast<uint2 *>(zo + tc::kmaj_off(64, 32 + r, 2 * u)) = make_uint2(s0, s1);
          }
        }
      }
      tc::fence_proxy_async();
      mbar_arrive(&prep_done[s]);
      if (++s == TCP_NS) { s = 0; ph ^= 1; }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 0-3)
    // D rows: 0..15 Re(big) k, 16..31 Im(big) k, 32..47 Re(small), 48..63 Im(small);
    // M = 64 layout: D row 16 w + i lives in TMEM lane 32 w + i.
    const int c = tid & 31, kg = tid >> 5;
    int n = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++n) {
      const int sc = item / items_per_sc, blk = item % items_per_sc, b = n & 1;
      tc::mbar_wait(&acc_full[b], (n >> 1) & 1);
      tc::fence_after_sync();
#pragma unroll 1
      for (int j = 0; j < 2; ++j) {
        named_sync(1, 128);                               // staging free
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          float v[16];
          tc::tmem_ld16(tm + ((uint32_t)(32 * warp) << 16) + 64 * b + 32 * j + 16 * h2, v);
          if (lane < 16) {
#pragma unroll
            for (int q = 0; q < 16; ++q) stg[(16 * warp + lane) * TCP_STG_LD + 16 * h2 + q] = v[q];
          }
        }
        if (j == 1) {
          tc::fence_before_sync();
          mbar_arrive(&acc_empty[b]);
        }
        named_sync(1, 128);
        float2 *x = a.x + (size_t)sc * a.K * a.Bl + blk * TCP_ROWS + 32 * j + c;
        float pw = 0.f;
        for (int k = kg; k < a.K; k += 4) {
          const float re = stg[k * TCP_STG_LD + c] + stg[(32 + k) * TCP_STG_LD + c];
          const float im = stg[(16 + k) * TCP_STG_LD + c] + stg[(48 + k) * TCP_STG_LD + c];
          x[(size_t)k * a.Bl] = make_float2(re, im);
          pw = fmaf(re, re, fmaf(im, im, pw));
        }
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) pw += __shfl_xor_sync(0xffffffffu, pw, m);
        if (c == 0) pw_part[j][kg] = pw;
      }
      named_sync(1, 128);
      if (tid < 2)
        a.pw[(size_t)sc * a.nchunks + blk * 2 + tid] =
            ((pw_part[tid][0] + pw_part[tid][1]) + pw_part[tid][2]) + pw_part[tid][3];
    }
  }
  pdl_trigger();
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tm, 128);
}

}  // namespace dpk
