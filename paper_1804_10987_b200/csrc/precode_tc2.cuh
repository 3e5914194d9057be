// precode_tc2.cuh — PD precode x = H_c^H z on the tensor cores (tcgen05 / TMEM / TMA),
// U = 32, one z per subcarrier (PD: every GPU precodes its antennas
// with the common whitened symbols), K <= 16, local antennas a multiple of 128.
//
// Per antenna b and symbol k:  x[k][b] = sum_u conj(H[b][u]) z[k][u].  With the fp32
// row of H read as 64 reals j = 2u + {0: re, 1: im}:
//     Re x[k][b] = sum_j H[b][j] Z'[k][j],       Z'[k][2u] = Re z_k[u],   Z'[k][2u+1] = Im z_k[u]
//     Im x[k][b] = sum_j H[b][j] Z'[16+k][j],    Z'[16+k][2u] = Im z_k[u], Z'[16+k][2u+1] = -Re z_k[u]
// so a block of 128 antennas is ONE real GEMM  D (128 x 32) = H (128 x 64) Z'^T  with H
// as the K-major A operand exactly as it sits in HBM (TMA, SWIZZLE_128B) and Z' (the
// subcarrier's z, expanded once) as the B operand.
//
// 3xTF32 (fp32-level accuracy): Hb = the raw fp32 tile read as tf32 (the tensor core
// uses its top 19 bits), Hs = H - trunc_tf32(H) (one elementwise pass), Zb / Zs the
// rounded split of Z'.  Per K step of 8 reals two UMMAs:
//     D[:, 0:64] += Hb [Zb ; Zs]^T   (N = 64: the Zb and Zs products side by side)
//     D[:, 0:32] += Hs Zb^T          (N = 32)
// and x = D[:, 0:32] + D[:, 32:64] in the epilogue.
//
// Persistent, warp-specialised, one CTA per SM (10 warps):
//   warp 8     TMA producer: 128-antenna blocks of H into a 4-stage ring (Hb).  H is an
//              input of the call, so it is fetched without griddepcontrol.wait
//              (overlapping the solve kernel's tail).
//   warps 4-7  prep: Z' operand once per subcarrier into a double buffer (the z rows are
//              prefetched into registers one subcarrier ahead), residual plane Hs per
//              block into a double buffer of its own.
//   warp 9     UMMA issuer: 16 UMMAs per block into a double-buffered TMEM accumulator.
//   warps 0-3  epilogue: TMEM lane quarter -> x rows (coalesced: one antenna per lane),
//              the subcarrier's power, and its per-subcarrier scalars (fin).
//
// HT = true (the default): the residual plane Hs goes to TMEM instead of a shared-memory buffer.
// The prep warp of lane quarter q reads antenna row 32q + lane of the raw block (16 16-byte loads
// of its own row), forms Hs in registers and stores its 64 reals as 64 TMEM columns of its lane;
// the Hs Zb^T product is then a .ts UMMA with A from TMEM (M = 128 antenna rows, K = 64 reals).
// That removes the shared-memory write of Hs and the UMMA's shared-memory read of it (the
// ablation of DESIGN.md §7 charges 3.8 us of 29.2 to the residual round trip) and frees the two
// 32 KB Hs buffers for two more raw ring stages (6 x 32 KB of H in flight).
#pragma once

// diagnostics only (scripts/gram_diag.sh builds, never the shipped build): 1 = no UMMAs, 2 = no UMMAs
// and no residual math, 3 = 2 and no x stores
#ifndef DP_PC2_DIAG
#define DP_PC2_DIAG 0
#endif
#include "tcgen05.cuh"

namespace dpk {

constexpr int PC2_ROWS = 128;                   // antennas per block (UMMA M)
constexpr int PC2_NS = 4;                       // raw H ring stages
constexpr int PC2_NH = 2;                       // residual (Hs) buffers
constexpr int PC2_BOX = PC2_ROWS * 128;         // one TMA box: 128 rows x 32 fp32 = 16 KB
constexpr int PC2_STAGE = 2 * PC2_BOX;          // Hb: 2 K-halves = 32 KB (Hs buffers: same size)
constexpr int PC2_ZOP = 64 * 64 * 4;            // Z' operand: 64 rows (Zb 0..31, Zs 32..63) x 64 K (x2 buffers)
constexpr int PC2_THREADS = 320;
__host__ __device__ constexpr int pc2_ns(bool ht) { return ht ? PC2_NS + PC2_NH : PC2_NS; }   // raw stages
__host__ __device__ constexpr size_t pc2_smem(bool ht) {
  return (size_t)(PC2_NS + PC2_NH) * PC2_STAGE + 2 * PC2_ZOP + 1024;   // HT: the Hs buffers become raw stages
}
constexpr size_t PC2_SMEM = pc2_smem(false);

// byte offset of 16-byte chunk c (reals 4c..4c+3, c < 16) of row r in a K-major SWIZZLE_128B block
// of PC2_ROWS rows (two 16 KB boxes of 32 reals)
__device__ __forceinline__ uint32_t pc2_chunk(int r, int c) {
  return (uint32_t)((c >> 3) * PC2_BOX + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

template <bool HT>
__global__ void __launch_bounds__(PC2_THREADS, 1) precode_tc2_kernel(const __grid_constant__ CUtensorMap tmH, Args a) {
  pdl_trigger();   // early: the next kernel may launch once every CTA of this grid has started
                   // (it still waits for this grid's completion in griddepcontrol.wait)
  constexpr int NS = pc2_ns(HT);
  extern __shared__ __align__(1024) uint8_t smem_dyn[];
  uint8_t *sm = smem_dyn + ((1024u - (tc::smem_u32(smem_dyn) & 1023u)) & 1023u);
  uint8_t *hsb = sm + (size_t)PC2_NS * PC2_STAGE;   // residual buffers (!HT)
  uint8_t *zop = sm + (size_t)(PC2_NS + PC2_NH) * PC2_STAGE;   // Z' double buffer
  __shared__ __align__(8) uint64_t full[NS], stage_free[NS], hs_full[PC2_NH], hs_free[PC2_NH];
  __shared__ __align__(8) uint64_t acc_full[2], acc_empty[2], zready[2], zfree[2];
  __shared__ uint32_t tmem_base;
  __shared__ float pw_red[4];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nblk = a.Bl / PC2_ROWS;
  const int n_items = a.n_sc;
  constexpr uint32_t TCOLS = HT ? 256 : 128;        // D double buffer (+ HT: Hs double buffer at 128 + 64 b)
  if (warp == 0) {
    tc::tmem_alloc(&tmem_base, TCOLS);
    tc::tmem_relinquish();
  }
  if (tid == 32) {
    for (int i = 0; i < NS; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&stage_free[i], 1);
    }
    for (int i = 0; i < PC2_NH; ++i) {
      tc::mbar_init(&hs_full[i], 128);
      tc::mbar_init(&hs_free[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&acc_full[i], 1);
      tc::mbar_init(&acc_empty[i], 128);
      tc::mbar_init(&zready[i], 128);
      tc::mbar_init(&zfree[i], 1);
    }
    tc::fence_mbar_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tm = tmem_base;

  if (warp == 8) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int s = 0, ph = 0, g = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        for (int blk = 0; blk < nblk; ++blk, ++g) {
          if (g >= NS) tc::mbar_wait(&stage_free[s], ph ^ 1);
          uint8_t *st = sm + (size_t)s * PC2_STAGE;
          const int row0 = item * a.Bl + blk * PC2_ROWS;
          tc::mbar_arrive_expect_tx(&full[s], 2 * PC2_BOX);
          tc::tma_load_2d(st, &tmH, 0, row0, &full[s]);
          tc::tma_load_2d(st + PC2_BOX, &tmH, 32, row0, &full[s]);
          if (++s == NS) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ UMMA issuer
    if (lane == 0) {
      constexpr uint32_t ID64 = tc::idesc_tf32(128, 64), ID32 = tc::idesc_tf32(128, 32);
      int s = 0, ph = 0, g = 0;
      for (int item = blockIdx.x, n = 0; item < n_items; item += gridDim.x, ++n) {
        const uint32_t zo = tc::smem_u32(zop + (size_t)(n & 1) * PC2_ZOP);
        tc::mbar_wait(&zready[n & 1], (n >> 1) & 1);
        tc::fence_after_sync();
        for (int blk = 0; blk < nblk; ++blk, ++g) {
          const int b = g & 1;
          if (g >= 2) tc::mbar_wait(&acc_empty[b], ((g >> 1) - 1) & 1);
          tc::mbar_wait(&full[s], ph);
          tc::mbar_wait(&hs_full[b], (g >> 1) & 1);   // Hs buffer g % 2 (PC2_NH = 2)
          tc::fence_after_sync();
          const uint32_t hb = tc::smem_u32(sm + (size_t)s * PC2_STAGE);
          const uint32_t hs = tc::smem_u32(hsb + (size_t)b * PC2_STAGE);
          const uint32_t d = tm + 64 * b;
#pragma unroll
          for (int t = 0; t < 8; ++t) {               // K = 64 reals in 8 steps of 8
            const uint32_t koff = (uint32_t)(t >> 2) * PC2_BOX + (uint32_t)(t & 3) * 32;
            const uint64_t zd = tc::smem_desc(zo + t * 2 * 64 * 16, 64 * 16, 128);
            if (DP_PC2_DIAG < 1) {
              tc::mma_tf32(d, tc::smem_desc_sw128(hb + koff, 1024), zd, ID64, t > 0 ? 1u : 0u);
              if (HT) tc::mma_tf32_ts(d, tm + 128 + 64 * b + 8 * t, zd, ID32, 1u);   // Hs from TMEM
              else tc::mma_tf32(d, tc::smem_desc_sw128(hs + koff, 1024), zd, ID32, 1u);
            }
          }
          tc::mma_commit(&stage_free[s]);
          tc::mma_commit(&hs_free[b]);
          tc::mma_commit(&acc_full[b]);
          if (++s == NS) { s = 0; ph ^= 1; }
        }
        tc::mma_commit(&zfree[n & 1]);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ prep (warps 4-7)
    const int ptid = tid - 128;
    int s = 0, ph = 0, g = 0;
    // z rows of the next subcarrier are prefetched into registers (thread element e = ptid + 128 i:
    // Z' row r = e / 32, u = e % 32, symbol k = r % 16; rows r and r + 16 read the same z)
    pdl_wait();                                       // z is the solve kernel's output
    float2 zv[8];
    auto load_z = [&](int item) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int e = ptid + 128 * i, k = (e >> 5) & 15, u = e & 31;
        zv[i] = (item < n_items && k < a.K) ? __ldg(a.zin + ((size_t)item * a.K + k) * 32 + u) : make_float2(0.f, 0.f);
      }
    };
    load_z(blockIdx.x);
    for (int item = blockIdx.x, n = 0; item < n_items; item += gridDim.x, ++n) {
      {  // Z' = [Zb ; Zs]: rows 0..15 Re-rows k, 16..31 Im-rows k (big), rows +32 small
        const int zb = n & 1;
        uint8_t *zo = zop + (size_t)zb * PC2_ZOP;
        if (n >= 2) tc::mbar_wait(&zfree[zb], ((n >> 1) - 1) & 1);   // UMMAs of subcarrier n-2 done with it
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int e = ptid + 128 * i, r = e >> 5, u = e & 31;
          const float2 v = zv[i];
          const float c0 = (r < 16) ? v.x : v.y, c1 = (r < 16) ? v.y : -v.x;
          const uint32_t b0 = tc::to_tf32(c0), b1 = tc::to_tf32(c1);
          const uint32_t s0 = tc::to_tf32(c0 - __uint_as_float(b0)), s1 = tc::to_tf32(c1 - __uint_as_float(b1));
          *reinterpret_cast<uint2 *>(zo + tc::kmaj_off(64, r, 2 * u)) = make_uint2(b0, b1);
          *reinterpret_cast<uint2 *>(zo + tc::kmaj_off(64, 32 + r, 2 * u)) = make_uint2(s0, s1);
        }
        tc::fence_proxy_async();
        mbar_arrive(&zready[zb]);
        load_z(item + gridDim.x);
      }
      for (int blk = 0; blk < nblk; ++blk, ++g) {
        const int hbuf = g & 1;
        tc::mbar_wait(&full[s], ph);
        if (g >= PC2_NH) tc::mbar_wait(&hs_free[hbuf], ((g >> 1) - 1) & 1);
        uint8_t *st = sm + (size_t)s * PC2_STAGE;
        if constexpr (HT) {
          // this lane's antenna row r of the block: Hs = H - trunc_tf32(H) -> TMEM lane r, columns = reals
          const int r = ptid;                                  // warp 4 + q holds rows 32 q .. (its lane quarter)
          float h[64];
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const float4 v = *reinterpret_cast<const float4 *>(st + pc2_chunk(r, c));
            h[4 * c] = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
            h[4 * c + 1] = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
            h[4 * c + 2] = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
            h[4 * c + 3] = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
          }
          const uint32_t th = tm + 128 + 64 * hbuf + ((uint32_t)(32 * (warp - 4)) << 16);
#pragma unroll
          for (int cb = 0; cb < 4; ++cb) tc::tmem_st16(th + 16 * cb, *reinterpret_cast<float(*)[16]>(h + 16 * cb));
          tc::tmem_wait_st();
          tc::fence_before_sync();
        } else {
          const uint4 *src = reinterpret_cast<const uint4 *>(st);
          uint4 *dst = reinterpret_cast<uint4 *>(hsb + (size_t)hbuf * PC2_STAGE);
          constexpr int NV = DP_PC2_DIAG >= 2 ? 0 : 2 * PC2_BOX / 16 / 128;      // 16 vectors per thread
          uint4 v[NV > 0 ? NV : 1];
#pragma unroll
          for (int i = 0; i < NV; ++i) v[i] = src[ptid + 128 * i];
#pragma unroll
          for (int i = 0; i < NV; ++i) {                  // Hs = H - trunc_tf32(H), same swizzled positions
            float4 f;
            f.x = __uint_as_float(v[i].x) - __uint_as_float(v[i].x & 0xFFFFE000u);
            f.y = __uint_as_float(v[i].y) - __uint_as_float(v[i].y & 0xFFFFE000u);
            f.z = __uint_as_float(v[i].z) - __uint_as_float(v[i].z & 0xFFFFE000u);
            f.w = __uint_as_float(v[i].w) - __uint_as_float(v[i].w & 0xFFFFE000u);
            dst[ptid + 128 * i] = *reinterpret_cast<uint4 *>(&f);
          }
          tc::fence_proxy_async();
        }
        mbar_arrive(&hs_full[hbuf]);
        if (++s == NS) { s = 0; ph ^= 1; }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 0-3)
    // M = 128: D row r (antenna r of the block) is TMEM lane r; columns 0..15 Re(k),
    // 16..31 Im(k) of the big products (+ Hs Zb), 32..63 the Zs products.
    pdl_wait();                                       // beta (solve kernel) is read below
    int g = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      float pw = 0.f;
      for (int blk = 0; blk < nblk; ++blk, ++g) {
        const int b = g & 1;
        tc::mbar_wait(&acc_full[b], (g >> 1) & 1);
        tc::fence_after_sync();
        float v[4][16];
        const uint32_t ta = tm + ((uint32_t)(32 * warp) << 16) + 64 * b;
#pragma unroll
        for (int c = 0; c < 4; ++c) tc::tmem_ld16_nowait(ta + 16 * c, v[c]);
        tc::tmem_wait_ld();
        tc::fence_before_sync();
        mbar_arrive(&acc_empty[b]);
        float2 *x = a.x + (size_t)item * a.K * a.Bl + blk * PC2_ROWS + 32 * warp + lane;
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (k < a.K && DP_PC2_DIAG < 3) {
            const float re = v[0][k] + v[2][k], im = v[1][k] + v[3][k];
            x[(size_t)k * a.Bl] = make_float2(re, im);
            pw = fmaf(re, re, fmaf(im, im, pw));
          }
      }
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) pw += __shfl_xor_sync(0xffffffffu, pw, m);
      if (lane == 0) pw_red[warp] = pw;
      named_sync(1, 128);
      if (tid == 0) {
        a.fin[2 * item] = a.fin_inv_beta ? __fdividef(1.f, __ldcg(a.beta + item)) : 0.f;
        a.fin[2 * item + 1] = (pw_red[0] + pw_red[1]) + (pw_red[2] + pw_red[3]);
      }
      named_sync(1, 128);
    }
  }
  pdl_trigger();
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tm, TCOLS);
}

}  // namespace dpk
