// fd_tc.cuh — FD-WF fused kernel for U = 32, S = B_c = 32 with the cluster Gram on
// the tensor cores (tcgen05 / TMEM / TMA, sm_100a) and the rest on the packed FP32
// pipe.  Same per-problem math and output as fd_fused_kernel (kernels.cuh):
//     G_c = H_c H_c^H  ->  A = G_c + kappa_c I  ->  -A^{-1}, beta_c (Lemma 1,
//     Sec. III-C)  ->  z = A^{-1} s / beta_c  ->  x_c = H_c^H z,  power partial.
//
// Gram on the tensor core.  With X = the fp32 tile viewed as 32 antenna rows x 64
// reals (j = 2u + {0: re, 1: im}),  P = X^T X  (64 x 64) and
//     Re G[u][v] = P[2u][2v] + P[2u+1][2v+1],   Im G[u][v] = P[2u+1][2v] - P[2u][2v+1].
// The TMA tile (two boxes of 32 reals x 32 rows, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B:
// 32-byte chunk c of 128-byte row r stored at c ^ (r % 4)) is directly an MN-major
// UMMA operand for both A = X^T and B = X (K = antennas) -- MN-major tf32 operands
// must use this SWIZZLE_128B_BASE32B layout (descriptor type 1; LBO = 4096 between
// the two 32-real atoms, SBO = 512 between 4-row K groups; verified by
// scripts/tc_probe.py).  The raw fp32 tile is the "big" tf32 operand (the tensor
// core reads the top 19 bits); one elementwise pass makes the residual
// Xs = X - trunc_tf32(X) in the same layout.  3xTF32:  P = Xb^T Xb + Xs^T Xb + Xb^T Xs,
// 12 UMMAs (M = N = 64, K = 8) accumulated in TMEM: an M = 64 accumulator uses lanes
// 0-15 of each 32-lane quarter, so problems 2g and 2g+1 share columns 64g.. (lane
// offset 0 / 16) and one 32x32b TMEM load feeds all 32 threads in the epilogue.
//
// CTA = 4 warps, one (subcarrier, cluster) problem each (12 warps per SM at 168
// registers: the SIMT solver needs them, so there is no separate producer warp).
//   thread 0:      TMA the 4 tiles; after its own residual, wait for the others' and
//                  issue 4 x 12 UMMAs; commit -> mma_done.
//   warps 0-3:     residual of their own tile -> plane_ready; then (all four, TMEM lane
//                  quarters) read P rows 16w..16w+15 of every problem, pair rows 2l and
//                  2l+1 across lanes (shfl_xor 1) and write G column l to the owning
//                  warp's staging; dealloc TMEM; then the SIMT solver of fd_fused_kernel
//                  (sweep, whitening) and the precode from the swizzled tile.
// smem: [4 tiles x 8 KB][4 regions x 9 KB][4 slots of 2 x 32 complex]; a region holds the residual
// plane, then the G staging (32 columns x 34 complex), then s and zT.
#pragma once
#include "tcgen05.cuh"

namespace dpk {

// many-waiter completions (every warp of the CTA waits): parked try_wait (DP_FD_SPIN: plain polling)
#ifndef DP_FD_ABL
#define DP_FD_ABL 0   // diagnostics builds only: 1 no sweep, 2 no SIMT precode, 4 no Gram UMMAs (timing ablation)
#endif
#ifdef DP_FD_SPIN
#define WAITF tc::mbar_wait
#else
#define WAITF tc::mbar_wait_park
#endif

constexpr int FDT_TILE = 8192;                 // 32 rows x 64 fp32, two SW128 boxes of 4 KB
constexpr int FDT_REG = 9216;                  // per-warp region (1024-aligned)
constexpr int FDT_GLD = 34;                    // G staging column stride (complex), 272 B
constexpr int FDT_THREADS = 128;
#ifdef DP_FD_SWEEP2D
constexpr int FDT_SLOT = 1280;                // per problem: 4 pivot-row buffers of 36 complex + 32 row scales (sweep_2d)
#else
constexpr int FDT_SLOT = 512;                 // per problem: 2 pivot-row buffers of 32 complex (sweep_sg2)
#endif
constexpr size_t FDT_SMEM = 4 * FDT_TILE + 4 * FDT_REG + 4 * FDT_SLOT + 1024;

// UMMA shared-memory descriptor of an MN-major SWIZZLE_128B_BASE32B operand: 128-byte
// rows along MN (32 tf32), 4-row K groups SBO bytes apart, MN atoms LBO bytes apart.
__device__ __forceinline__ uint64_t smem_desc_mn_sw128b32(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;
  return d;
}
// kind::tf32, f32 accumulate, A and B MN-major
__host__ __device__ constexpr uint32_t idesc_tf32_mn(int M, int N) {
  return tc::idesc_tf32(M, N) | (1u << 15) | (1u << 16);
}

// 16-byte chunk c' (complex 2c', 2c'+1) of tile row r in the TMA SW128_ATOM_32B layout
__device__ __forceinline__ float4 ld_chunk_sw128(const uint8_t *tile, int r, int cp) {
  return *reinterpret_cast<const float4 *>(tile + ((cp >> 3) << 12) + (r << 7) + ((((cp & 7) >> 1) ^ (r & 3)) << 5) +
                                           ((cp & 1) << 4));
}

// z rows of the FD kernel: the symbols-innermost whitening of kernels.cuh (whiten_Tg)
constexpr int FDT_SP = WT_SP;
template <int KC>
__device__ __forceinline__ void whiten_T(const float2 (&d)[32], float ib, const float2 *sT, float2 *zT, int K, int l) {
  whiten_Tg<32, KC>(d, ib, sT, zT, K, l);
}

// x[k][r] = sum_u conj(H[r][u]) z[k][u] for the lane's row r = l (S = U = 32)
template <int KC>
__device__ __forceinline__ float precode_sw128(const uint8_t *tile, const float2 *zT, int K, float2 *__restrict__ x,
                                               size_t xstride, int l, int zs_ = 0) {
  constexpr int KCP = ZL<KC>::KCP;
  const int zs = zs_ ? zs_ : ZL<KC>::zs(K);
  float pw = 0.f;
  for (int k0 = 0, q = 0; k0 < K; k0 += KC, ++q) {
    float2 acc[KC];
#pragma unroll
    for (int j = 0; j < KC; ++j) acc[j] = make_float2(0.f, 0.f);
    const float2 *zq = zT + q * KCP;
#pragma unroll 4
    for (int c = 0; c < 16; ++c) {
      const float4 h = ld_chunk_sw128(tile, l, c);
      const float2 h0 = lo2(h), h1 = hi2(h);
      const float2 *z0 = zq + (2 * c) * zs, *z1 = z0 + zs;
#pragma unroll
      for (int j = 0; j < KC; j += 2) {
        if (j + 1 < KC) {
          const float4 za = *reinterpret_cast<const float4 *>(z0 + j);
          const float4 zb = *reinterpret_cast<const float4 *>(z1 + j);
          cfma_cj(acc[j], h0, lo2(za));
          cfma_cj(acc[j + 1], h0, hi2(za));
          cfma_cj(acc[j], h1, lo2(zb));
          cfma_cj(acc[j + 1], h1, hi2(zb));
        } else {
          cfma_cj(acc[j], h0, z0[j]);
          cfma_cj(acc[j], h1, z1[j]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < KC; ++j)
      if (k0 + j < K) {
        x[(size_t)(k0 + j) * xstride + l] = acc[j];
        pw += cabs2(acc[j]);
      }
  }
  return pw;
}

// x[k][r] = sum_u conj(H[r][u]) z[k][u] with the symbols split in two halves (WTC path): lane l
// computes antennas r0 = l & 15 and r1 = r0 + 16 for the symbols kg KH .. kg KH + KH-1 (kg = l >> 4,
// KH = ceil(KC / 2)), reading z from zT[u][8 kg + m] (the layout fd_tc's tensor-core whitening
// writes).  Per pair of users: 2 tile loads (rows r0, r1) + 8 z loads for 4 KH complex MACs, against
// 1 + 2 KH loads for 2 KH MACs with one row per lane (precode_sw128): a third fewer shared-memory
// loads, the same FFMA2 count.  Rows r0 and r0 + 16 keep the swizzled tile reads at 4 bank positions.
template <int KC>
__device__ __forceinline__ float precode_sw128_h(const uint8_t *tile, const float2 *zT, int K, float2 *__restrict__ x,
                                                 size_t xstride, int l) {
  constexpr int KH = (KC + 1) / 2;
  const int r0 = l & 15, r1 = r0 + 16, kg = l >> 4;
  float2 a0[KH], a1[KH];
#pragma unroll
  for (int m = 0; m < KH; ++m) a0[m] = a1[m] = make_float2(0.f, 0.f);
  const float2 *zq = zT + 8 * kg;
#pragma unroll 2
  for (int c = 0; c < 16; ++c) {
    const float4 h0 = ld_chunk_sw128(tile, r0, c), h1 = ld_chunk_sw128(tile, r1, c);
    const float2 *za = zq + (2 * c) * FDT_SP, *zb = za + FDT_SP;   // users 2c, 2c+1
#pragma unroll
    for (int m = 0; m < KH; m += 2) {
      if (m + 1 < KH) {
        const float4 va = *reinterpret_cast<const float4 *>(za + m);
        const float4 vb = *reinterpret_cast<const float4 *>(zb + m);
        cfma_cj(a0[m], lo2(h0), lo2(va));
        cfma_cj(a0[m + 1], lo2(h0), hi2(va));
        cfma_cj(a1[m], lo2(h1), lo2(va));
        cfma_cj(a1[m + 1], lo2(h1), hi2(va));
        cfma_cj(a0[m], hi2(h0), lo2(vb));
        cfma_cj(a0[m + 1], hi2(h0), hi2(vb));
        cfma_cj(a1[m], hi2(h1), lo2(vb));
        cfma_cj(a1[m + 1], hi2(h1), hi2(vb));
      } else {
        const float2 va = za[m], vb = zb[m];
        cfma_cj(a0[m], lo2(h0), va);
        cfma_cj(a1[m], lo2(h1), va);
        cfma_cj(a0[m], hi2(h0), vb);
        cfma_cj(a1[m], hi2(h1), vb);
      }
    }
  }
  float pw = 0.f;
#pragma unroll
  for (int m = 0; m < KH; ++m) {
    const int k = kg * KH + m;
    if (k < K) {
      x[(size_t)k * xstride + r0] = a0[m];
      x[(size_t)k * xstride + r1] = a1[m];
      pw += cabs2(a0[m]) + cabs2(a1[m]);
    }
  }
  return pw;
}

// 2-D register-blocked Hermitian sweep for U = 32, one warp per problem (the Gauss-Jordan sweep of
// sweep_sg2 on the Jacobi-equilibrated A, P:285-286 / Lemma 1).  Lane (r, c) = (lane >> 3, lane & 7)
// owns the 8 x 4 block rows 8r .. 8r+7, columns 4c .. 4c+3 of A.  Per pivot k a lane needs only the
// pivot-row entries of its 8 rows (the pivot column, by Hermitian symmetry) and of its 4 columns:
// 6 16-byte loads (12 shared-memory wavefronts) instead of the 16 broadcast loads (32 wavefronts)
// of the column-per-lane sweep, for the same 64 FFMA2.
//   Update (i, j != k):  a_ij -= conj(R_i) sig_j,  sig_j = R_j / d  (sig_k = 1 - 1/d: column k
//   becomes a_ik / d),  R = pivot row k, d = a_kk.  Row k (a_kj -> a_kj / d) takes the same update
//   with R_k replaced by d - 1 (a_kj - (d - 1) a_kj / d = a_kj / d); the pivot entry is set to -1/d.
// The next pivot row is updated first (look-ahead) and published by its 8 owner lanes into one of
// four rotating row buffers (one __syncwarp per pivot).  Row-buffer position of entry j: j + 2 (j >> 4)
// (a 16-byte gap after 16 entries keeps the column-part loads of the 8 column groups conflict-free).
// In: g = G staging of the problem (column j at g + j * FDT_GLD, complex), A = G + kappa I.
// Out: g columns = -A^{-1} (zeroed when not HPD); returns beta (Lemma 1, Eq. 6).
__device__ __forceinline__ int rbpos(int j) { return j + 2 * (j >> 4); }
__device__ __forceinline__ float sweep_2d(float2 *g, uint8_t *sl, int lane, float kappa, float coef, bool &ok) {
  const int r = lane >> 3, c = lane & 7;
  float2 *buf = reinterpret_cast<float2 *>(sl);               // [4][36]
  float *rs = reinterpret_cast<float *>(sl + 4 * 36 * 8);     // [32] row / column scales
  const float dl = g[lane * FDT_GLD + lane].x + kappa;        // own diagonal (lane = column index)
  const bool gd = (dl > 0.f) && (dl < INFINITY);
  rs[lane] = gd ? rsqrtf(dl) : 1.f;
  float2 w[8][4];
#pragma unroll
  for (int jj = 0; jj < 4; ++jj) {
    const float2 *col = g + (4 * c + jj) * FDT_GLD + 8 * r;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const float4 v = *reinterpret_cast<const float4 *>(col + 2 * m);
      w[2 * m][jj] = lo2(v);
      w[2 * m + 1][jj] = hi2(v);
    }
  }
  const bool hasdiag = (c >> 1) == r;                          // block holds (4c + jj, 4c + jj)
#pragma unroll
  for (int jj = 0; jj < 4; ++jj) {
    if (hasdiag && !(c & 1)) w[jj][jj] = make_float2(w[jj][jj].x + kappa, 0.f);
    if (hasdiag && (c & 1)) w[4 + jj][jj] = make_float2(w[4 + jj][jj].x + kappa, 0.f);
  }
  __syncwarp();
  float rr[8], rc[4];
  {
    const float4 a0 = *reinterpret_cast<const float4 *>(rs + 8 * r), a1 = *reinterpret_cast<const float4 *>(rs + 8 * r + 4);
    const float4 b0 = *reinterpret_cast<const float4 *>(rs + 4 * c);
    rr[0] = a0.x; rr[1] = a0.y; rr[2] = a0.z; rr[3] = a0.w; rr[4] = a1.x; rr[5] = a1.y; rr[6] = a1.z; rr[7] = a1.w;
    rc[0] = b0.x; rc[1] = b0.y; rc[2] = b0.z; rc[3] = b0.w;
  }
#pragma unroll
  for (int ii = 0; ii < 8; ++ii)
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) w[ii][jj] = cscale(w[ii][jj], rr[ii] * rc[jj]);
  const int cpos = 4 * c + 2 * (c >> 2), rpos = 8 * r + 2 * (r >> 1);
  if (r == 0) {                                               // row 0 opens the sweep
    *reinterpret_cast<float4 *>(buf + cpos) = make_float4(w[0][0].x, w[0][0].y, w[0][1].x, w[0][1].y);
    *reinterpret_cast<float4 *>(buf + cpos + 2) = make_float4(w[0][2].x, w[0][2].y, w[0][3].x, w[0][3].y);
  }
  __syncwarp();
  float pmin = buf[0].x, pmax = pmin;
  float id = rcp_approx(pmin);
#pragma unroll 1
  for (int kk = 0; kk < 32; kk += 8) {
    const bool pr = (r == (kk >> 3));                          // this block's pivot rows are my rows
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int k = kk + j;
      const float2 *cur = buf + 36 * (j & 3);
      float2 *nxt = buf + 36 * ((j + 1) & 3);
      const float4 c01 = *reinterpret_cast<const float4 *>(cur + cpos);
      const float4 c23 = *reinterpret_cast<const float4 *>(cur + cpos + 2);
      float2 R[8];
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const float4 v = *reinterpret_cast<const float4 *>(cur + rpos + 2 * m);
        R[2 * m] = lo2(v);
        R[2 * m + 1] = hi2(v);
      }
      float2 sg[4] = {cscale(lo2(c01), id), cscale(hi2(c01), id), cscale(lo2(c23), id), cscale(hi2(c23), id)};
      const bool pc = (c == (k >> 2));                         // my columns hold column k (jj = k & 3)
      if (pc) sg[j & 3] = make_float2(1.f - id, 0.f);
      if (pr) R[j].x -= 1.f;                                   // row k: d -> d - 1
      const int jn = (j + 1) & 7;
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) cfms_cj(w[jn][jj], R[jn], sg[jj]);   // row k+1 first
      const bool pn = (j < 7) ? pr : (r == (kk >> 3) + 1);     // my rows hold row k+1
      if (pn && k + 1 < 32) {
        *reinterpret_cast<float4 *>(nxt + cpos) = make_float4(w[jn][0].x, w[jn][0].y, w[jn][1].x, w[jn][1].y);
        *reinterpret_cast<float4 *>(nxt + cpos + 2) = make_float4(w[jn][2].x, w[jn][2].y, w[jn][3].x, w[jn][3].y);
      }
      __syncwarp();
      float idn = 1.f;
      if (k + 1 < 32) {
        const float dn = nxt[rbpos(k + 1)].x;                 // a_{k+1,k+1}
        pmin = fminf(pmin, dn);
        pmax = fmaxf(pmax, dn);
        idn = rcp_approx(dn);
      }
#pragma unroll
      for (int ii = 0; ii < 8; ++ii)
        if (ii != jn)
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) cfms_cj(w[ii][jj], R[ii], sg[jj]);
      if (pr && pc) w[j][j & 3] = make_float2(-id, 0.f);      // the pivot entry
      id = idn;
    }
  }
  // undo the equilibration: A^{-1} = D^{-1/2} A'^{-1} D^{-1/2}; Lemma 1 traces
  float tr = 0.f, f = 0.f;
#pragma unroll
  for (int ii = 0; ii < 8; ++ii)
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      w[ii][jj] = cscale(w[ii][jj], rr[ii] * rc[jj]);
      f += cabs2(w[ii][jj]);
    }
#pragma unroll
  for (int jj = 0; jj < 4; ++jj) {
    if (hasdiag && !(c & 1)) tr -= w[jj][jj].x;
    if (hasdiag && (c & 1)) tr -= w[4 + jj][jj].x;
  }
  tr = sg_sum<32>(tr);
  f = sg_sum<32>(f);
  // Lemma 1, Eq. (6):  beta^2 = Es/rho^2 (tr A^{-1} - kappa ||A^{-1}||_F^2)
  const float rad = coef * (tr - kappa * f);
  const bool all_gd = __all_sync(0xffffffffu, gd);
  ok = all_gd && (pmin > 0.f) && (pmax < INFINITY) && (rad > 0.f) && (rad < INFINITY);
#pragma unroll
  for (int jj = 0; jj < 4; ++jj) {
    float2 *col = g + (4 * c + jj) * FDT_GLD + 8 * r;
#pragma unroll
    for (int m = 0; m < 4; ++m)
      *reinterpret_cast<float4 *>(col + 2 * m) =
          ok ? make_float4(w[2 * m][jj].x, w[2 * m][jj].y, w[2 * m + 1][jj].x, w[2 * m + 1][jj].y) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  return ok ? sqrtf(rad) : 1.f;
}

// Per-subcarrier scalars folded into the FD kernel (replaces fd_finish_kernel):
// fin[sc] = {sum_c 1/beta_c, sum_c power_c} over the rank's Cl clusters, ascending c
// (the order of finish_sc, so the result is bit-identical).  a.fold = CTAs per
// subcarrier: 1 -> the CTA's 4 problems hold 4/Cl whole subcarriers; 2, 4, 8 -> a
// thread-block cluster of a.fold CTAs (launched with that cluster shape) holds one
// subcarrier: ranks 1.. push their 8 partials into rank 0's shared memory with
// st.async (completion counted in bytes on rank 0's mbarrier) and exit; only rank 0
// waits.  The mbarrier is initialised before a cluster barrier at kernel start.
struct __align__(16) FoldSmem {
  float rb[8][4], rp[8][4];  // rank 0: partials pushed by ranks 1..7 (16-byte rows: st.async.v4)
  float fb[4], fp[4];        // this CTA's per-problem 1/beta_c and power
  uint64_t bar;
};
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t map_rank(const void *p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(tc::smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_v4(uint32_t raddr, float4 v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(raddr),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(rbar)
               : "memory");
}
// The cluster barrier that orders rank 0's mbarrier init before the other ranks' st.async is
// split: arrive (release) at kernel start, wait (acquire) only just before the push at the
// end, by which time every CTA of the cluster has long arrived — no stall at kernel start.
__device__ __forceinline__ void fd_fold_init(const Args &a, FoldSmem &f) {
  if (a.fold > 1) {
    if (threadIdx.x == 0 && cluster_rank() == 0) {
      tc::mbar_init(&f.bar, 1);
      tc::fence_mbar_init();
      tc::mbar_arrive_expect_tx(&f.bar, 32u * (a.fold - 1));
    }
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");   // init already fenced (fence.mbarrier_init)
  }
}
__device__ __forceinline__ void fd_fold_finish(const Args &a, FoldSmem &f, int p0, int warp, int lane, float ib, float pw,
                                               bool writer = true) {
  if (lane == 0 && writer) { f.fb[warp] = ib; f.fp[warp] = pw; }   // warp = the problem's slot 0..3
  __syncthreads();
  const int nprob = a.n_sc * a.nchunks;
  if (a.fold == 1) {
    const int per = 4 / a.nchunks;                             // subcarriers in this CTA
    if (threadIdx.x < per) {
      const int q0 = threadIdx.x * a.nchunks, sc = (p0 + q0) / a.nchunks;
      if (p0 + q0 < nprob) {
        float b = 0.f, w = 0.f;
        for (int c = 0; c < a.nchunks; ++c) { b += f.fb[q0 + c]; w += f.fp[q0 + c]; }
        a.fin[2 * sc] = a.fin_inv_beta ? b : 0.f;
        a.fin[2 * sc + 1] = w;
      }
    }
    return;
  }
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");   // pairs with fd_fold_init
  if (threadIdx.x != 0) return;
  const uint32_t rank = cluster_rank();
  if (rank != 0) {                                             // push to rank 0 and leave
    st_async_v4(map_rank(&f.rb[rank][0], 0), make_float4(f.fb[0], f.fb[1], f.fb[2], f.fb[3]), map_rank(&f.bar, 0));
    st_async_v4(map_rank(&f.rp[rank][0], 0), make_float4(f.fp[0], f.fp[1], f.fp[2], f.fp[3]), map_rank(&f.bar, 0));
    return;
  }
  tc::mbar_wait(&f.bar, 0);
  float b = 0.f, w = 0.f;
  for (int c = 0; c < 4; ++c) { b += f.fb[c]; w += f.fp[c]; }
  for (int r = 1; r < a.fold; ++r)
    for (int c = 0; c < 4; ++c) { b += f.rb[r][c]; w += f.rp[r][c]; }
  const int sc = p0 / a.nchunks;
  a.fin[2 * sc] = a.fin_inv_beta ? b : 0.f;
  a.fin[2 * sc + 1] = w;
}

// WTC: whitening on the tensor cores (see below); false: SIMT whitening (whiten_T)
template <int KC, bool WTC>
__global__ void __launch_bounds__(FDT_THREADS, 3) fd_tc_kernel(const __grid_constant__ CUtensorMap tmH, Args a) {
  pdl_trigger();   // early: the next kernel may launch once every CTA of this grid has started
                   // (it still waits for this grid's completion in griddepcontrol.wait)
  constexpr int U = 32;
  extern __shared__ __align__(1024) uint8_t smem_dyn[];
  // align by an offset (not integer casts) so the compiler keeps the shared state space: LDS, not LD
  uint8_t *sm = smem_dyn + ((1024u - (tc::smem_u32(smem_dyn) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t tile_full[4], plane_ready[4], mma_done, wz_done[2];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(16) FoldSmem fold;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nprob = a.n_sc * a.nchunks;
  const int p0 = blockIdx.x * 4;
  fd_fold_init(a, fold);
  const int np = min(4, nprob - p0);
  auto tile = [&](int p) { return sm + (size_t)p * FDT_TILE; };
  auto region = [&](int p) { return sm + 4 * FDT_TILE + (size_t)p * FDT_REG; };
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) { tc::mbar_init(&tile_full[i], 1); tc::mbar_init(&plane_ready[i], 1); }
    tc::mbar_init(&mma_done, 1);
    tc::mbar_init(&wz_done[0], 1);
    tc::mbar_init(&wz_done[1], 1);
    tc::fence_mbar_init();
    // H is an input of the call (no predecessor kernel writes it): its tiles are fetched
    // before griddepcontrol.wait, overlapping the previous kernel's tail
    for (int p = 0; p < np; ++p) {   // cluster (sc, cl) = rows sc Bl + 32 cl (Bl > 32 nchunks: unequal runs)
      const int pp = p0 + p, row = (pp / a.nchunks) * a.Bl + (pp % a.nchunks) * 32;
      tc::mbar_arrive_expect_tx(&tile_full[p], FDT_TILE);
      tc::tma_load_2d(tile(p), &tmH, 0, row, &tile_full[p]);
      tc::tma_load_2d(tile(p) + 4096, &tmH, 32, row, &tile_full[p]);
    }
    // and the tiles of the CTA that will most likely reuse this SM slot go to L2
    const int pn = p0 + 4 * a.pf_dist;
    if (a.pf_dist > 0 && pn < nprob) {
      const int n = min(4, nprob - pn);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.H + (size_t)pn * 32 * U),
                   "r"((uint32_t)n * FDT_TILE)
                   : "memory");
    }
  }
  if (warp == 0) {
    tc::tmem_alloc(&tmem_base, 128);
    tc::tmem_relinquish();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tm = tmem_base;
  // Programmatic dependent launch: nothing before the x stores reads or writes an output of a
  // preceding kernel (H and s are inputs of the call; the Gram, sweep and whitening live in this
  // CTA's shared memory and TMEM), so griddepcontrol.wait sits just before them -- CTAs that start
  // on SMs the preceding kernel has already left run their problems up to the precode meanwhile.

  // ---------------------------------------------------------------- solver warps 0-3
  const int p = warp;
  const bool active = p < np;
  const uint8_t *tl = tile(p);
  uint8_t *rg = region(p);
  if (active) {
    WAITF(&tile_full[p], 0);
    const uint4 *src = reinterpret_cast<const uint4 *>(tl);
    float4 *dst = reinterpret_cast<float4 *>(rg);
    uint4 v16[FDT_TILE / 16 / 32];
#pragma unroll
    for (int j = 0; j < FDT_TILE / 16 / 32; ++j) v16[j] = src[lane + 32 * j];
#pragma unroll
    for (int j = 0; j < FDT_TILE / 16 / 32; ++j) {         // residual Xs = X - trunc_tf32(X)
      const uint4 v = v16[j];
      dst[lane + 32 * j] = make_float4(__uint_as_float(v.x) - __uint_as_float(v.x & 0xFFFFE000u),
                           __uint_as_float(v.y) - __uint_as_float(v.y & 0xFFFFE000u),
                           __uint_as_float(v.z) - __uint_as_float(v.z & 0xFFFFE000u),
                           __uint_as_float(v.w) - __uint_as_float(v.w & 0xFFFFE000u));
    }
    tc::fence_proxy_async();
    __syncwarp();
    if (lane == 0) mbar_arrive(&plane_ready[p]);
  }
  if (tid == 0) {                                             // UMMA issue (elected thread of warp 0)
    constexpr uint32_t IDESC = idesc_tf32_mn(64, 64);
    for (int q = 0; q < np; ++q) {
      tc::mbar_wait(&plane_ready[q], 0);
      tc::fence_after_sync();
      const uint32_t xb = tc::smem_u32(tile(q)), xs = tc::smem_u32(region(q));
      const uint32_t d = tm + 64 * (q >> 1) + ((uint32_t)(16 * (q & 1)) << 16);   // M = 64 D: lanes 16 (q&1) + 0..15
#pragma unroll
      for (int t = 0; t < 4; ++t) {                            // antennas 8t .. 8t+7
        const uint64_t b = smem_desc_mn_sw128b32(xb + 1024 * t, 4096, 512);
        const uint64_t s = smem_desc_mn_sw128b32(xs + 1024 * t, 4096, 512);
        if (DP_FD_ABL & 4) continue;
        tc::mma_tf32(d, b, b, IDESC, t > 0 ? 1u : 0u);         // Xb^T Xb
        tc::mma_tf32(d, s, b, IDESC, 1u);                      // Xs^T Xb
        tc::mma_tf32(d, b, s, IDESC, 1u);                      // Xb^T Xs
      }
    }
    tc::mma_commit(&mma_done);
  }
  __syncwarp();
  WAITF(&mma_done, 0);
  tc::fence_after_sync();
  // ---- epilogue: TMEM lane 32 warp + i holds P row r = 16 warp + (i & 15) of problem
  // 2 g + (i >> 4) in columns 64 g .. 64 g + 63 (two M = 64 accumulators share columns)
  {
    const bool odd = lane & 1;
    const int l = (16 * warp + (lane & 15)) >> 1;             // G column produced by this lane pair
#pragma unroll 1
    for (int g = 0; 2 * g < np; ++g) {
      const int q = 2 * g + (lane >> 4);
      float2 *gst = reinterpret_cast<float2 *>(region(q < np ? q : 0));
      const uint32_t ta = tm + 64 * g + ((uint32_t)(32 * warp) << 16);
      float v[4][16];
#pragma unroll
      for (int c = 0; c < 4; ++c) tc::tmem_ld16_nowait(ta + 16 * c, v[c]);
      tc::tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const float *v0 = v[c], *v2 = v[c + 2];   // columns 16c.. (even lanes' half), 16(c+2).. (odd lanes')
        float A[16], B[16];                                   // rows 2l and 2l+1 of the half this lane owns
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float r = __shfl_xor_sync(0xffffffffu, odd ? v0[j] : v2[j], 1);
          A[j] = odd ? r : v0[j];
          B[j] = odd ? v2[j] : r;
        }
        if (q < np) {
          const int u0 = 8 * (c + (odd ? 2 : 0));
          float4 *o = reinterpret_cast<float4 *>(gst + l * FDT_GLD + u0);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            o[j] = make_float4(A[4 * j] + B[4 * j + 1], A[4 * j + 1] - B[4 * j],
                               A[4 * j + 2] + B[4 * j + 3], A[4 * j + 3] - B[4 * j + 2]);
        }
      }
    }
  }
  tc::fence_before_sync();
  named_sync(1, 128);                                         // G staging complete, TMEM reads done
  if (!WTC && warp == 0) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tm, 128);
  }
  const int pr = p0 + p;
  float fold_b = 0.f, fold_p = 0.f;                           // this problem's 1/beta_c and power (fold)
  if (a.Gout) pdl_wait();
  if (active && a.Gout) {                                     // dp_debug_gram: packed G_c of the FD path
    const float2 *g = reinterpret_cast<const float2 *>(rg) + lane * FDT_GLD;
    for (int u = 0; u <= lane; ++u) a.Gout[(size_t)pr * npacked(32) + pidx(32, u, lane)] = g[u];
  }
  if (a.Gout) {                                               // (debug launches never fold)
    if (WTC) {
      tc::fence_after_sync();
      if (warp == 0) tc::tmem_dealloc(tm, 128);
    }
    return;
  }
  // ---------------------------------------------------------------- SIMT solver
  const int sc = (active ? pr : p0) / a.nchunks, cl = pr % a.nchunks;
  const int l = lane;
  uint8_t *slot8 = sm + 4 * FDT_TILE + 4 * FDT_REG + (size_t)p * FDT_SLOT;
  float2 *slot = reinterpret_cast<float2 *>(slot8);
  float2 col[U];
#pragma unroll
  for (int u = 0; u < U; ++u) col[u] = make_float2(0.f, 0.f);
  bool ok = false;
  float beta = 1.f;
  // region: [ss (K x U), later zT (U x FDT_SP)] [sT (U x FDT_SP) | WTC: pieces of the s operand]
  float2 *ss = reinterpret_cast<float2 *>(rg), *zT = ss, *sT = ss + U * FDT_SP;
  auto piece = [&](int q) { return region(q >> 2) + 4608 + 1024 * (q & 3); };   // S' piece q = plane * 8 + t
  if constexpr (WTC) {
    // column-per-lane sweep (sweep_sg2); DP_FD_SWEEP2D (diagnostics builds): the 2-D blocked sweep in
    // place on the G staging (-A^{-1} columns written back), then column l to lane l for the A' rows
    float2 *gs = reinterpret_cast<float2 *>(rg);
    if (DP_FD_ABL & 1) ok = true;
    else if (active) {
#ifndef DP_FD_SWEEP2D
      float2 *g = gs + l * FDT_GLD;
      const float dl = g[l].x + a.kappa;
      g[l] = make_float2(dl, 0.f);
#pragma unroll
      for (int u = 0; u < U; u += 2) {
        const float4 v = *reinterpret_cast<const float4 *>(g + u);
        col[u] = lo2(v);
        col[u + 1] = hi2(v);
      }
      __syncwarp();
      // s of this subcarrier -> warp 0's region (free until zT): read by the S' build after the sweep
      if (a.s_wait) pdl_wait();                               // s from the broadcast: its kernel complete
      if (warp == 0) sg_copy_async<U>(reinterpret_cast<float2 *>(rg), a.s + (size_t)sc * a.K * U, a.K * U, l);
      beta = sweep_sg2<U>(col, slot, l, dl, a.kappa, a.coef, ok);
#else
      beta = sweep_2d(gs, slot8, l, a.kappa, a.coef, ok);
      __syncwarp();
      const float2 *g = gs + l * FDT_GLD;
#pragma unroll
      for (int u = 0; u < U; u += 2) {
        const float4 v = *reinterpret_cast<const float4 *>(g + u);
        col[u] = lo2(v);
        col[u + 1] = hi2(v);
      }
#endif
    }
    // ---- Whitening on the tensor cores:  Z = A^{-1} S / beta for the CTA's 4 problems at
    // once (they share s: same subcarrier).  Real form with j = 2v + {0: re, 1: im}:
    //   A'[32p + u][j]  = (A_p^{-1}[u][v] / beta_p) (re, im)         M = 128 (4 x 32 rows)
    //   S'[n][j]: n = k < 16: (Re s_k[v], -Im s_k[v]); n = 16 + k: (Im s_k[v], Re s_k[v])   N = 32
    //   D[32p + u][k] = Re z_k[u], D[32p + u][16 + k] = Im z_k[u]     (K = 64)
    // A' is written by each warp into its own TMEM lane quarter (A operand from TMEM),
    // S' (K-major interleaved, N = 32) in 16 pieces of 1 KB (one per K step and plane)
    // in the regions' second halves.  3xTF32: A'b S'b + A'b S's, then A's S'b after A's
    // replaces A'b in TMEM (TMEM holds 128 columns: A' 64, D 32).
#ifndef DP_FD_SWEEP2D
    cp_async_wait_all();                                      // warp 0: the staged s
#endif
    named_sync(1, 128);                                       // every warp has read its G staging
#ifndef DP_FD_SWEEP2D
    const float2 *s_st = reinterpret_cast<const float2 *>(region(0));
#endif
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = tid + 128 * i, n = e >> 5, v = e & 31, k = n & 15;
      float2 w = make_float2(0.f, 0.f);
      if (k < a.K) {
#ifndef DP_FD_SWEEP2D
        const float2 sv = s_st[k * U + v];
#else
        const float2 sv = __ldg(a.s + ((size_t)sc * a.K + k) * U + v);
#endif
        w = n < 16 ? make_float2(sv.x, -sv.y) : make_float2(sv.y, sv.x);
      }
      const int j = 2 * v, t = j >> 3;
      const uint32_t off = ((j & 7) >> 2) * 512 + (n >> 3) * 128 + (n & 7) * 16 + (j & 3) * 4;
      *reinterpret_cast<float2 *>(piece(t) + off) = w;
      const float2 r = make_float2(w.x - __uint_as_float(__float_as_uint(w.x) & 0xFFFFE000u),
                                   w.y - __uint_as_float(__float_as_uint(w.y) & 0xFFFFE000u));
      *reinterpret_cast<float2 *>(piece(8 + t) + off) = r;
    }
    tc::fence_proxy_async();
  } else {
    float dl = 1.f;
    if (active) {
      float2 *g = reinterpret_cast<float2 *>(rg) + l * FDT_GLD;
      dl = g[l].x + a.kappa;
      g[l] = make_float2(dl, 0.f);                              // A = G_c + kappa_c I (own row only)
#pragma unroll
      for (int u = 0; u < U; u += 2) {
        const float4 v = *reinterpret_cast<const float4 *>(g + u);
        col[u] = lo2(v);
        col[u + 1] = hi2(v);
      }
    }
    __syncwarp();
    if (a.s_wait) pdl_wait();
    sg_copy_async<U>(ss, a.s + (size_t)sc * a.K * U, a.K * U, l);
    if (DP_FD_ABL & 1) ok = true;
    else if (active) beta = sweep_sg2<U>(col, slot, l, dl, a.kappa, a.coef, ok);   // col <- -A^{-1}[:, l]
  }
  const float ib = ok ? -__fdividef(1.f, beta) : 0.f;       // failed problems: x = 0
  if constexpr (WTC) {
    const uint32_t tq = tm + ((uint32_t)(32 * warp) << 16);  // this warp's TMEM lane quarter
    float av[4][16];                                          // A' row l: A^{-1}[l][v]/beta = ib conj(col[v])
#pragma unroll
    for (int v = 0; v < U; ++v) {
      av[v >> 3][(2 * v) & 15] = ib * col[v].x;
      av[v >> 3][(2 * v + 1) & 15] = -ib * col[v].y;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) tc::tmem_st16(tq + 16 * c, av[c]);
    tc::tmem_wait_st();
    tc::fence_before_sync();
    named_sync(1, 128);
    constexpr uint32_t ID = tc::idesc_tf32(128, 32);
    if (tid == 0) {
      tc::fence_after_sync();
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const uint64_t bb = tc::smem_desc(tc::smem_u32(piece(t)), 512, 128);
        const uint64_t bs = tc::smem_desc(tc::smem_u32(piece(8 + t)), 512, 128);
        tc::mma_tf32_ts(tm + 64, tm + 8 * t, bb, ID, t > 0 ? 1u : 0u);   // A'b S'b
        tc::mma_tf32_ts(tm + 64, tm + 8 * t, bs, ID, 1u);                // A'b S's
      }
      tc::mma_commit(&wz_done[0]);
    }
    WAITF(&wz_done[0], 0);
    tc::fence_after_sync();
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int j = 0; j < 16; ++j)
        av[c][j] = av[c][j] - __uint_as_float(__float_as_uint(av[c][j]) & 0xFFFFE000u);   // A's
#pragma unroll
    for (int c = 0; c < 4; ++c) tc::tmem_st16(tq + 16 * c, av[c]);
    tc::tmem_wait_st();
    tc::fence_before_sync();
    named_sync(1, 128);
    if (tid == 0) {
      tc::fence_after_sync();
#pragma unroll
      for (int t = 0; t < 8; ++t)
        tc::mma_tf32_ts(tm + 64, tm + 8 * t, tc::smem_desc(tc::smem_u32(piece(t)), 512, 128), ID, 1u);   // A's S'b
      tc::mma_commit(&wz_done[1]);
    }
    WAITF(&wz_done[1], 0);
    tc::fence_after_sync();
    float zv[2][16];
    tc::tmem_ld16_nowait(tq + 64, zv[0]);
    tc::tmem_ld16_nowait(tq + 80, zv[1]);
    tc::tmem_wait_ld();
    // zT[u][8 kg + m] = z_{kg KH + m}[u] (precode_sw128_h), zero padded
    constexpr int KH = (KC + 1) / 2;
    float4 *zo = reinterpret_cast<float4 *>(zT + l * FDT_SP);
    auto sym = [](int pos) { return pos < 8 ? (pos < KH ? pos : -1) : (pos - 8 < KC - KH ? KH + pos - 8 : -1); };
#pragma unroll
    for (int pos = 0; pos < 16; pos += 2) {
      const int k0 = sym(pos), k1 = sym(pos + 1);
      if (k0 < 0 && k1 < 0) continue;
      zo[pos >> 1] = make_float4(k0 >= 0 ? zv[0][k0 & 15] : 0.f, k0 >= 0 ? zv[1][k0 & 15] : 0.f,
                                 k1 >= 0 ? zv[0][k1 & 15] : 0.f, k1 >= 0 ? zv[1][k1 & 15] : 0.f);
    }
    tc::fence_before_sync();
    named_sync(1, 128);                                       // TMEM reads done
    if (warp == 0) {
      tc::fence_after_sync();
      tc::tmem_dealloc(tm, 128);
    }
  } else {
    cp_async_wait_all();
    __syncwarp();
    if (active) {                                             // sT[v][k] = s_k[v] (lane v), zero padded
      constexpr int KP = (KC + 1) & ~1;
      float4 *row = reinterpret_cast<float4 *>(sT + l * FDT_SP);
#pragma unroll
      for (int j = 0; j < KP; j += 2) {
        const float2 s0 = j < a.K ? ss[j * U + l] : make_float2(0.f, 0.f);
        const float2 s1 = j + 1 < a.K ? ss[(j + 1) * U + l] : make_float2(0.f, 0.f);
        row[j >> 1] = make_float4(s0.x, s0.y, s1.x, s1.y);
      }
      __syncwarp();
      whiten_T<KC>(col, ib, sT, zT, a.K, l);
    }
  }
  __syncwarp();
  pdl_wait();                                                 // the predecessor's outputs (x, beta, ...) complete
  if (active) {
    float2 *xo = a.x + (size_t)sc * a.K * a.Bl + (size_t)cl * a.S;
    float pw = (DP_FD_ABL & 2) ? 0.f
               : WTC ? precode_sw128_h<KC>(tl, zT, a.K, xo, (size_t)a.Bl, l)
                     : precode_sw128<KC>(tl, zT, a.K, xo, (size_t)a.Bl, l, FDT_SP);
    pw = sg_sum<U>(pw);
    if (l == 0) {
      a.beta[pr] = ok ? beta : qnan();
      a.pw[pr] = pw;
      if (!ok) atomicAdd(a.bad, 1);
    }
    fold_b = 1.f / (ok ? beta : qnan());
    fold_p = pw;
  }
  pdl_trigger();
  if (a.fold) fd_fold_finish(a, fold, p0, warp, lane, fold_b, fold_p);
}

}  // namespace dpk
