// gram_tc.cuh — tensor-core (tcgen05 / TMEM / TMA) batched Gram for U = 32 (sm_100a).
//
// Work item = (subcarrier, group): G = sum_{b in group} h_b h_b^H; PD groups
// are all local antennas, FD groups are clusters.  With X = [Re H | Im H] (nb x 64,
// real) and P = X^T X (64 x 64):
//     Re G = P[0:32, 0:32] + P[32:64, 32:64],   Im G = P[32:64, 0:32] - P[0:32, 32:64].
// 3xTF32 keeps fp32-level accuracy: X = Xb + Xs with Xb = tf32(X), Xs = tf32(X - Xb),
//     P ~= Xb^T Xb + Xs^T Xb + (Xs^T Xb)^T.
// One kind::tf32 UMMA per 8 antennas computes both products: M = 128 with
// A = [Xb^T ; Xs^T] (rows 0..63 big, 64..127 small), N = 64 with B = Xb^T, the first
// 64 rows of the same shared-memory operand.
//
// Warp-specialised persistent pipeline (6 warps, 2 CTAs per SM):
//   warp 4  TMA: streams 32-antenna chunks of H (8 KB, contiguous) with cp.async.bulk
//           into an NR-stage raw ring (mbarrier transaction counts);
//   warps 0-3 split: convert raw chunks into tf32 big/small planes of the operand
//           (interleaved K-major layout, tcgen05.cuh) in an NS-stage ring; at each
//           item boundary they also run the previous item's epilogue (TMEM ->
//           registers -> shared staging -> packed Hermitian G in HBM);
//   warp 5  UMMA: one elected thread issues 4 UMMAs per chunk into a TMEM accumulator
//           (double-buffered, 2 x 64 columns) and commits stages / accumulators.
// All hand-offs are full/empty mbarrier pairs; no block-wide barrier in the loop.
#pragma once
#include "tcgen05.cuh"

namespace dpk {

constexpr int TCG_TK = 32;                          // antennas per chunk
constexpr int TCG_NR = 4;                           // raw (TMA) ring stages
constexpr int TCG_NS = 2;                           // operand ring stages
constexpr int TCG_RAW = TCG_TK * 32 * 8;            // raw chunk bytes: 8 KB
constexpr int TCG_OPR = 128 * TCG_TK * 4;           // operand stage: 128 rows x 32 K tf32 = 16 KB
constexpr int TCG_LD = 68;                          // staging row stride (floats; 16-byte rows)
constexpr int TCG_THREADS = 192;
constexpr size_t TCG_SMEM = (size_t)TCG_NR * TCG_RAW + (size_t)TCG_NS * TCG_OPR + 128 * TCG_LD * 4 + 1024;

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t *mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(mbar)) : "memory");
}

__global__ void __launch_bounds__(TCG_THREADS, 1) gram_tc_kernel(Args a) {
  pdl_wait();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *raw = smem_raw;
  uint8_t *opr = raw + (size_t)TCG_NR * TCG_RAW;
  float *stg = reinterpret_cast<float *>(opr + (size_t)TCG_NS * TCG_OPR);
  __shared__ __align__(8) uint64_t raw_full[TCG_NR], raw_empty[TCG_NR];
  __shared__ __align__(8) uint64_t opr_full[TCG_NS], opr_empty[TCG_NS];
  __shared__ __align__(8) uint64_t acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_items = a.n_sc * a.nchunks;          // (subcarrier, group)
  const int nck = a.S / TCG_TK;                    // chunks per item
  const int my_items = (n_items - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const int total = my_items * nck;                // this CTA's chunks, g -> (item g / nck, chunk g % nck)
  if (warp == 0) {
    tc::tmem_alloc(&tmem_base, 128);
    tc::tmem_relinquish();
  }
  if (tid == 32) {
    for (int i = 0; i < TCG_NR; ++i) { tc::mbar_init(&raw_full[i], 1); tc::mbar_init(&raw_empty[i], 128); }
    for (int i = 0; i < TCG_NS; ++i) { tc::mbar_init(&opr_full[i], 128); tc::mbar_init(&opr_empty[i], 1); }
    for (int i = 0; i < 2; ++i) { tc::mbar_init(&acc_full[i], 1); tc::mbar_init(&acc_empty[i], 128); }
    tc::fence_mbar_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tm = tmem_base;

  if (warp == 4) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int rs = 0, rph = 0, item = blockIdx.x, c = 0;
      for (int g = 0; g < total; ++g) {
        if (g >= TCG_NR) tc::mbar_wait_sleep(&raw_empty[rs], rph ^ 1);
        const float2 *src = a.H + ((size_t)item * a.S + (size_t)c * TCG_TK) * 32;
        tc::mbar_arrive_expect_tx(&raw_full[rs], TCG_RAW);
        tc::bulk_g2s(raw + (size_t)rs * TCG_RAW, src, TCG_RAW, &raw_full[rs]);
        if (++rs == TCG_NR) { rs = 0; rph ^= 1; }
        if (++c == nck) { c = 0; item += gridDim.x; }
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ UMMA issuer
    if (lane == 0) {
      constexpr uint32_t IDESC = tc::idesc_tf32(128, 64);
      const uint32_t opr_u32 = tc::smem_u32(opr);
      int it = 0, c = 0, os = 0, oph = 0;
      for (int g = 0; g < total; ++g) {
        const int b = it & 1;
        if (c == 0 && it >= 2) tc::mbar_wait_sleep(&acc_empty[b], ((it >> 1) - 1) & 1);
        tc::mbar_wait_sleep(&opr_full[os], oph);
        tc::fence_after_sync();
        const uint32_t acc = tm + (uint32_t)b * 64;
        const uint32_t ab = opr_u32 + (uint32_t)os * TCG_OPR;
#pragma unroll
        for (int t = 0; t < TCG_TK / 8; ++t) {
          const uint64_t d = tc::smem_desc(ab + t * 2 * 128 * 16, 128 * 16, 128);   // A = [Xb^T;Xs^T], B = Xb^T
          tc::mma_tf32(acc, d, d, IDESC, (c > 0 || t > 0) ? 1u : 0u);
        }
        tc::mma_commit(&opr_empty[os]);
        if (c == nck - 1) tc::mma_commit(&acc_full[b]);
        if (++os == TCG_NS) { os = 0; oph ^= 1; }
        if (++c == nck) { c = 0; ++it; }
      }
    }
  } else {
    // ------------------------------------------------------------ split + epilogue (warps 0-3)
    // mapping: row u = lane, antenna quads k0 = 4 (warp + 4 i), i = 0, 1: reads are
    // consecutive per warp, each plane store is one 16-byte vector (4 antennas of row u)
    int it = 0, c = 0, rs = 0, rph = 0, os = 0, oph = 0;
    for (int g = 0; g <= total; ++g) {
      if (g < total) {
        tc::mbar_wait(&raw_full[rs], rph);
        if (g >= TCG_NS) tc::mbar_wait(&opr_empty[os], oph ^ 1);
        const float2 *src = reinterpret_cast<const float2 *>(raw + (size_t)rs * TCG_RAW);
        uint8_t *ob = opr + (size_t)os * TCG_OPR;
        float2 h[2][4];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int q = 0; q < 4; ++q) h[i][q] = src[(4 * (warp + 4 * i) + q) * 32 + lane];
        mbar_arrive(&raw_empty[rs]);                     // raw stage consumed (values in registers)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          uint32_t rb[4], ib[4], rsm[4], ism[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            rb[q] = tc::to_tf32(h[i][q].x);
            ib[q] = tc::to_tf32(h[i][q].y);
            rsm[q] = tc::to_tf32(h[i][q].x - __uint_as_float(rb[q]));
            ism[q] = tc::to_tf32(h[i][q].y - __uint_as_float(ib[q]));
          }
          const int k0 = 4 * (warp + 4 * i);
          *reinterpret_cast<uint4 *>(ob + tc::kmaj_off(128, lane, k0)) = make_uint4(rb[0], rb[1], rb[2], rb[3]);
          *reinterpret_cast<uint4 *>(ob + tc::kmaj_off(128, 32 + lane, k0)) = make_uint4(ib[0], ib[1], ib[2], ib[3]);
          *reinterpret_cast<uint4 *>(ob + tc::kmaj_off(128, 64 + lane, k0)) =
              make_uint4(rsm[0], rsm[1], rsm[2], rsm[3]);
          *reinterpret_cast<uint4 *>(ob + tc::kmaj_off(128, 96 + lane, k0)) =
              make_uint4(ism[0], ism[1], ism[2], ism[3]);
        }
        tc::fence_proxy_async();
        mbar_arrive(&opr_full[os]);
        if (++rs == TCG_NR) { rs = 0; rph ^= 1; }
        if (++os == TCG_NS) { os = 0; oph ^= 1; }
      }
      // epilogue of item it-1 (its UMMAs were issued while this item was being split)
      if ((g == total || c == 0) && it > 0) {
        const int pit = it - 1, b = pit & 1;
        tc::mbar_wait(&acc_full[b], (pit >> 1) & 1);
        tc::fence_after_sync();
        // TMEM lane r = D row r: r < 64 -> (Xb^T Xb)[r], r >= 64 -> (Xs^T Xb)[r - 64]
        const uint32_t acc = tm + (uint32_t)b * 64 + ((uint32_t)(32 * warp) << 16);
        float d[64];
#pragma unroll
        for (int cb = 0; cb < 4; ++cb) {
          float v[16];
          tc::tmem_ld16(acc + 16 * cb, v);
#pragma unroll
          for (int j = 0; j < 16; ++j) d[16 * cb + j] = v[j];
        }
        tc::fence_before_sync();
        mbar_arrive(&acc_empty[b]);                      // accumulator free for item pit + 2
        named_sync(1, 128);                              // previous epilogue done with staging
        float4 *row = reinterpret_cast<float4 *>(stg + tid * TCG_LD);
#pragma unroll
        for (int j = 0; j < 16; ++j) row[j] = make_float4(d[4 * j], d[4 * j + 1], d[4 * j + 2], d[4 * j + 3]);
        named_sync(1, 128);
        // P = D1 + D2 + D2^T ; D1 = stg rows 0..63, D2 = stg rows 64..127
        auto P = [&](int r, int s) {
          return stg[r * TCG_LD + s] + stg[(64 + r) * TCG_LD + s] + stg[(64 + s) * TCG_LD + r];
        };
        float2 *out = a.Gout + (size_t)(blockIdx.x + pit * gridDim.x) * npacked(32);
        for (int e = tid; e < 32 * 32; e += 128) {
          const int u = e >> 5, v = e & 31;
          if (u <= v) {
            const float gr = P(u, v) + P(32 + u, 32 + v);
            const float gi = P(32 + u, v) - P(u, 32 + v);
            out[pidx(32, u, v)] = make_float2(gr, gi);
          }
        }
      }
      if (++c == nck) { c = 0; ++it; }
    }
  }
  pdl_trigger();
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tm, 128);
}

}  // namespace dpk
