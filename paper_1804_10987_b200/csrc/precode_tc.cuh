// precode_tc.cuh — tensor-core (tcgen05 / TMEM / TMA) precode x_c = H_c^H z for U = 32.
//
// Per antenna b and symbol k:  x[k][b] = sum_u conj(H[b][u]) z[k][u].
// With the interleaved real index j = 2u + {0: re, 1: im}, H's fp32 row is used as is:
//     Re x[k][b] = sum_j H[b][j] Zr[k][j],  Zr[k][2u] = Re z[k][u],  Zr[k][2u+1] = Im z[k][u]
//     Im x[k][b] = sum_j H[b][j] Zi[k][j],  Zi[k][2u] = Im z[k][u],  Zi[k][2u+1] = -Re z[k][u]
// so D = Z H^T is one real GEMM: A = Z (rows: 16 Re-rows k, 16 Im-rows k), K = 64,
// B = the 32 antenna rows of one block (N = 32).  3xTF32 (4 products, summed by the
// tensor core): A = [Zb ; Zs] (M = 64: big rows 0..31, small rows 32..63) and
// B = Hb + Hs, where Hb is the raw fp32 row consumed as tf32 (the tensor core reads
// its top 19 bits) and Hs = H - trunc_tf32(H) is computed in place; both UMMAs
// accumulate into one TMEM tile, and x = D[0:32] + D[32:64].
//
// H tiles arrive by TMA (2-D tensor map over [rows][64] fp32, 128 rows x 32 floats
// boxes, SWIZZLE_128B, which is the canonical K-major SW128 UMMA layout).  A work item
// is 128 antennas (4 blocks of 32) of one subcarrier; block j uses z group
// zg(j) (PD: the subcarrier's z for every block; FD: cluster j's z, S = 32).
//
// Warp roles (6 warps, 1 CTA per SM): warp 4 TMA, warp 5 UMMA issue, warps 0-3 build
// the residual plane and the Z operands, then run the epilogue (TMEM -> shared
// staging -> coalesced x stores + power partial per 32-antenna block).
#pragma once
#include "tcgen05.cuh"

namespace dpk {

constexpr int TCP_NS = 2;                               // H stages
constexpr int TCP_HB = 128 * 128;                       // one TMA box: 128 rows x 128 B = 16 KB
constexpr int TCP_HSTAGE = 4 * TCP_HB;                  // raw (2 K-halves) + residual (2 K-halves) = 64 KB
constexpr int TCP_Z = 64 * 64 * 4;                      // one Z operand (64 rows x 64 K, interleaved) = 16 KB
constexpr int TCP_STG_LD = 33;                          // staging: [64 rows][33]
constexpr int TCP_THREADS = 192;
constexpr size_t TCP_SMEM = (size_t)TCP_NS * TCP_HSTAGE + 4 * TCP_Z + 64 * TCP_STG_LD * 4 + 1024;

__global__ void __launch_bounds__(TCP_THREADS, 1) precode_tc_kernel(const __grid_constant__ CUtensorMap tmH, Args a) {
  pdl_wait();
  extern __shared__ __align__(1024) uint8_t smem_dyn[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  uint8_t *hst = sm;                                      // [NS][raw h0, raw h1, res h0, res h1]
  uint8_t *zop = sm + (size_t)TCP_NS * TCP_HSTAGE;        // 4 Z operands
  float *stg = reinterpret_cast<float *>(zop + 4 * TCP_Z);
  __shared__ __align__(8) uint64_t h_full[TCP_NS], h_empty[TCP_NS], op_full[TCP_NS], z_empty, acc_full, acc_empty;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int blocks_per_sc = a.Bl / 128;                  // items per subcarrier
  const int n_items = a.n_sc * blocks_per_sc;
  if (warp == 0) {
    tc::tmem_alloc(&tmem_base, 128);
    tc::tmem_relinquish();
  }
  if (tid == 32) {
    for (int i = 0; i < TCP_NS; ++i) {
      tc::mbar_init(&h_full[i], 1);
      tc::mbar_init(&h_empty[i], 1);
      tc::mbar_init(&op_full[i], 128);
    }
    tc::mbar_init(&z_empty, 1);
    tc::mbar_init(&acc_full, 1);
    tc::mbar_init(&acc_empty, 128);
    tc::fence_mbar_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tm = tmem_base;

  if (warp == 4) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int s = 0, ph = 0, n = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++n) {
        if (n >= TCP_NS) tc::mbar_wait_sleep(&h_empty[s], ph ^ 1);
        const int row0 = (item / blocks_per_sc) * a.Bl + (item % blocks_per_sc) * 128;
        uint8_t *dst = hst + (size_t)s * TCP_HSTAGE;
        tc::mbar_arrive_expect_tx(&h_full[s], 2 * TCP_HB);
        tc::tma_load_2d(dst, &tmH, 0, row0, &h_full[s]);
        tc::tma_load_2d(dst + TCP_HB, &tmH, 32, row0, &h_full[s]);
        if (++s == TCP_NS) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ UMMA issuer
    if (lane == 0) {
      constexpr uint32_t IDESC = tc::idesc_tf32(64, 32);
      int s = 0, ph = 0, n = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++n) {
        if (n >= 1) tc::mbar_wait_sleep(&acc_empty, (n - 1) & 1);
        tc::mbar_wait_sleep(&op_full[s], ph);
        tc::fence_after_sync();
        const uint32_t hb = tc::smem_u32(hst + (size_t)s * TCP_HSTAGE);
#pragma unroll
        for (int j = 0; j < 4; ++j) {                     // 32-antenna block j -> TMEM columns 32 j
          const uint32_t za = tc::smem_u32(zop + (size_t)(a.zgroups > 1 ? j : 0) * TCP_Z);   // PD: one Z
          const uint32_t d = tm + 32 * j;
#pragma unroll
          for (int t = 0; t < 8; ++t) {                   // K = 64 reals in 8 steps of 8
            const uint64_t ad = tc::smem_desc(za + t * 2 * 64 * 16, 64 * 16, 128);
            const uint32_t koff = (uint32_t)(t >> 2) * TCP_HB + (uint32_t)(t & 3) * 32 + (uint32_t)j * 32 * 128;
            tc::mma_tf32(d, ad, tc::smem_desc_sw128(hb + koff, 1024), IDESC, t > 0 ? 1u : 0u);
            tc::mma_tf32(d, ad, tc::smem_desc_sw128(hb + 2 * TCP_HB + koff, 1024), IDESC, 1u);
          }
        }
        tc::mma_commit(&h_empty[s]);
        tc::mma_commit(&z_empty);
        tc::mma_commit(&acc_full);
        if (++s == TCP_NS) { s = 0; ph ^= 1; }
      }
    }
  } else {
    // ------------------------------------------------------------ operands + epilogue (warps 0-3)
    const int zs_K = a.K;
    int s = 0, ph = 0, n = 0, zsc = -1;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++n) {
      const int sc = item / blocks_per_sc, blk = item % blocks_per_sc;
      // -- Z operands (rebuilt when the subcarrier or the groups change); wait until the
      //    previous item's UMMAs stopped reading them
      const bool per_block = a.zgroups > 1;
      if (per_block || sc != zsc) {
        if (n >= 1) tc::mbar_wait(&z_empty, (n - 1) & 1);
        const int nz = per_block ? 4 : 1;
        for (int jz = 0; jz < nz; ++jz) {
          const int g = per_block ? blk * 4 + jz : 0;
          const float2 *z = a.zin + ((size_t)sc * a.zgroups + g) * zs_K * 32;
          uint8_t *zo = zop + (size_t)jz * TCP_Z;
          // rows r: 0..15 Re-rows k=r, 16..31 Im-rows k=r-16 (big); +32: small. cols j = 2u + {0,1}
          for (int e = tid; e < 32 * 32; e += 128) {
            const int r = e >> 5, u = e & 31;
            const int k = r & 15;
            float2 v = (k < zs_K) ? z[(size_t)k * 32 + u] : make_float2(0.f, 0.f);
            float c0, c1;
            if (r < 16) { c0 = v.x; c1 = v.y; } else { c0 = v.y; c1 = -v.x; }
            const uint32_t b0 = tc::to_tf32(c0), b1 = tc::to_tf32(c1);
            const uint32_t s0 = tc::to_tf32(c0 - __uint_as_float(b0)), s1 = tc::to_tf32(c1 - __uint_as_float(b1));
            *reinterpret_cast<uint32_t *>(zo + tc::kmaj_off(64, r, 2 * u)) = b0;
            *reinterpret_cast<uint32_t *>(zo + tc::kmaj_off(64, r, 2 * u + 1)) = b1;
            *reinterpret_cast<uint32_t *>(zo + tc::kmaj_off(64, 32 + r, 2 * u)) = s0;
            *reinterpret_cast<uint32_t *>(zo + tc::kmaj_off(64, 32 + r, 2 * u + 1)) = s1;
          }
        }
        zsc = sc;
      } else if (n >= 1) {
        tc::mbar_wait(&z_empty, (n - 1) & 1);
      }
      // -- residual plane Hs = H - trunc_tf32(H) (elementwise on the swizzled tiles)
      tc::mbar_wait(&h_full[s], ph);
      {
        const uint4 *src = reinterpret_cast<const uint4 *>(hst + (size_t)s * TCP_HSTAGE);
        uint4 *dst = reinterpret_cast<uint4 *>(hst + (size_t)s * TCP_HSTAGE + 2 * TCP_HB);
#pragma unroll 4
        for (int e = tid; e < 2 * TCP_HB / 16; e += 128) {
          uint4 v = src[e];
          float4 f;
          f.x = __uint_as_float(v.x) - __uint_as_float(v.x & 0xFFFFE000u);
          f.y = __uint_as_float(v.y) - __uint_as_float(v.y & 0xFFFFE000u);
          f.z = __uint_as_float(v.z) - __uint_as_float(v.z & 0xFFFFE000u);
          f.w = __uint_as_float(v.w) - __uint_as_float(v.w & 0xFFFFE000u);
          dst[e] = *reinterpret_cast<uint4 *>(&f);
        }
      }
      tc::fence_proxy_async();
      mbar_arrive(&op_full[s]);
      // -- epilogue, one 32-antenna block at a time: D rows = output rows (r < 32 big,
      //    r >= 32 small), columns = antennas; M = 64 layout: D row 16 w + i lives in
      //    TMEM lane 32 w + i
      tc::mbar_wait(&acc_full, n & 1);
      tc::fence_after_sync();
      __shared__ float pw_part[4][4];
      const int c = tid & 31, kg = tid >> 5;             // column c, symbols k = kg, kg + 4, ...
#pragma unroll 1
      for (int j = 0; j < 4; ++j) {
        named_sync(1, 128);                               // staging free
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          float v[16];
          tc::tmem_ld16(tm + ((uint32_t)(32 * warp) << 16) + 32 * j + 16 * h2, v);
          if (lane < 16) {
            const int r = 16 * warp + lane;
#pragma unroll
            for (int q = 0; q < 16; ++q) stg[r * TCP_STG_LD + 16 * h2 + q] = v[q];
          }
        }
        if (j == 3) {
          tc::fence_before_sync();
          mbar_arrive(&acc_empty);                        // accumulator free for the next item
        }
        named_sync(1, 128);
        const int b = blk * 128 + 32 * j + c;            // antenna within the rank
        float2 *x = a.x + (size_t)sc * a.K * a.Bl + b;
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
      if (tid < 4) {
        const int j = tid;
        a.pw[(size_t)sc * a.nchunks + blk * 4 + j] = ((pw_part[j][0] + pw_part[j][1]) + pw_part[j][2]) + pw_part[j][3];
      }
      if (++s == TCP_NS) { s = 0; ph ^= 1; }
    }
  }
  pdl_trigger();
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tm, 128);
}

}  // namespace dpk
