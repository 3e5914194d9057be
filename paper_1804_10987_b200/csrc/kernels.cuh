// kernels.cuh — sm_100a kernels of the decentralized WF precoders
// (arXiv 1804.10987).  Included once, by dp_api.cu.
//
// Execution model.  All arithmetic is complex fp32 (the paper's
// precision, cuBLAS C* routines).  The unit of work is a SUB-GROUP
// (SG) of U consecutive lanes of a warp (U in {4, 8, 16, 32}; 32/U SGs per
// warp).  Lane l of an SG owns column l of every U x U matrix of its problem,
// kept in registers:
//   gram_sg    G[:, l]  = sum_b h_b conj(h_b[l])                (G_c = H_c H_c^H)
//   solve_sg   right-looking Cholesky A = L L^H
//              forward substitution  W0 = L^{-1}
//              back substitution     A^{-1} = W0^H W0
//              beta from tr A^{-1} = ||W0||_F^2 and ||A^{-1}||_F^2 (Lemma 1, Eq. 6)
//   whiten_sg  z_k[l] = sum_v conj(A^{-1}[v][l]) s_k[v] / beta
//   precode_sg x_k[b] = sum_u conj(H[b][u]) z_k[u]               (x_c = H_c^H z)
// H tiles live in shared memory with a 16-byte-chunk XOR swizzle so that both
// access patterns are conflict-free: row broadcast (Gram) and one row per lane
// (precode).  No atomics on data: every sum has a fixed order, so results are
// bit-reproducible run to run.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace dpk {

// ------------------------------------------------------------------ complex helpers
// acc += a * conj(b)
__device__ __forceinline__ void cfma_bc(float2 &acc, float2 a, float2 b) {
  acc.x = fmaf(a.x, b.x, acc.x); acc.x = fmaf(a.y, b.y, acc.x);
  acc.y = fmaf(a.y, b.x, acc.y); acc.y = fmaf(-a.x, b.y, acc.y);
}
// acc += conj(a) * b
__device__ __forceinline__ void cfma_cj(float2 &acc, float2 a, float2 b) {
  acc.x = fmaf(a.x, b.x, acc.x); acc.x = fmaf(a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y); acc.y = fmaf(-a.y, b.x, acc.y);
}
// acc -= conj(a) * b
__device__ __forceinline__ void cfms_cj(float2 &acc, float2 a, float2 b) {
  acc.x = fmaf(-a.x, b.x, acc.x); acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(-a.x, b.y, acc.y); acc.y = fmaf(a.y, b.x, acc.y);
}
// acc -= a * b
__device__ __forceinline__ void cfms(float2 &acc, float2 a, float2 b) {
  acc.x = fmaf(-a.x, b.x, acc.x); acc.x = fmaf(a.y, b.y, acc.x);
  acc.y = fmaf(-a.x, b.y, acc.y); acc.y = fmaf(-a.y, b.x, acc.y);
}
__device__ __forceinline__ float cabs2(float2 a) { return fmaf(a.x, a.x, a.y * a.y); }
__device__ __forceinline__ float qnan() { return __int_as_float(0x7fc00000); }

// sum over the U lanes of an SG (butterfly; every lane gets the total)
template <int U>
__device__ __forceinline__ float sg_sum(float v) {
#pragma unroll
  for (int m = U / 2; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m, U);
  return v;
}

// ------------------------------------------------------------------ swizzled H tile
// Tile row b holds U complex = U/2 16-byte chunks; chunk c of row b is stored at
// chunk position c ^ swz(b).  For every U, 8 consecutive rows read at one chunk
// index land in 8 distinct 16-byte bank groups (precode: one row per lane), and
// a row is still read as aligned float4 chunks (Gram: row broadcast).
template <int U>
__device__ __forceinline__ int swz(int b) {
  constexpr int CPR = U / 2;                      // chunks per row
  constexpr int RPS = CPR >= 8 ? 1 : 8 / CPR;     // rows per 128-byte bank sweep
  constexpr int NS = CPR >= 8 ? 8 : CPR;          // distinct swizzle values
  return (b / RPS) % NS;
}
template <int U>
__device__ __forceinline__ float4 tile_chunk(const float2 *tile, int b, int c) {
  return *reinterpret_cast<const float4 *>(tile + (size_t)b * U + 2 * (c ^ swz<U>(b)));
}
template <int U>
__device__ __forceinline__ float2 tile_elem(const float2 *tile, int b, int u) {
  return tile[(size_t)b * U + 2 * ((u >> 1) ^ swz<U>(b)) + (u & 1)];
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Cooperative async copy of `rows` contiguous rows of H (global [rows][U]) into
// a swizzled tile, by threads tid, tid + nthreads, ...
template <int U>
__device__ __forceinline__ void load_tile_async(float2 *tile, const float2 *__restrict__ g, int rows,
                                                int tid, int nthreads) {
  constexpr int CPR = U / 2;
  const int nchunks = rows * CPR;
  for (int i = tid; i < nchunks; i += nthreads) {
    const int b = i / CPR, c = i % CPR;
    cp_async16(tile + (size_t)b * U + 2 * (c ^ swz<U>(b)), g + 2 * (size_t)i);
  }
}

// ------------------------------------------------------------------ z layout
// zT[u][k] with symbols grouped in chunks of KC, each chunk starting at an even
// (16-byte aligned) offset: index(u, k) = u*zs + (k/KC)*KCP + k%KC.
template <int KC> struct ZL {
  static constexpr int KCP = (KC + 1) & ~1;
  __host__ __device__ static int nkc(int K) { return (K + KC - 1) / KC; }
  __host__ __device__ static int zs(int K) { return nkc(K) * KCP + 2; }
  __device__ static int idx(int zs_, int u, int k) { return u * zs_ + (k / KC) * KCP + (k % KC); }
};

// ------------------------------------------------------------------ (a) Gram
// Column l of the Gram of rows [0, nrows) of a tile: acc[u] += h_b[u] conj(h_b[l]).
// Rows are absolute tile rows (the swizzle phase depends on the row index).
template <int U>
__device__ __forceinline__ void gram_sg(const float2 *tile, int row0, int nrows, int l, float2 (&acc)[U]) {
#pragma unroll 2
  for (int b = row0; b < row0 + nrows; ++b) {
    const float2 own = tile_elem<U>(tile, b, l);
#pragma unroll
    for (int c = 0; c < U / 2; ++c) {
      const float4 h = tile_chunk<U>(tile, b, c);      // same address for the whole SG: broadcast
      cfma_bc(acc[2 * c], make_float2(h.x, h.y), own);
      cfma_bc(acc[2 * c + 1], make_float2(h.z, h.w), own);
    }
  }
}

// ------------------------------------------------------------------ (b) solve
// Scratch per SG: slot[U] + M[U][MS] (MS = U + 2 keeps rows 16-byte aligned).
template <int U> struct Scr {
  static constexpr int MS = U + 2;
  static constexpr int SIZE = U + U * MS;   // complex elements
};

// In: a[] = column l of A = G + kappa I (full Hermitian column, lane l of the SG).
// Out: d[] = column l of A^{-1}; returns beta (Lemma 1).  ok = false if a Cholesky
// pivot is not a finite positive number or beta's radicand is not.
template <int U>
__device__ __forceinline__ float solve_sg(float2 (&a)[U], float2 (&d)[U], float2 *scr, int l,
                                          float kappa, float coef, bool &ok) {
  float2 *slot = scr;
  float2 *M = scr + U;
  constexpr int MS = Scr<U>::MS;
  ok = true;
  // ---- Cholesky, right-looking.  Lane l holds column l of the trailing matrix
  // including its upper part, so lane i's a[k] = A^(k)[k][i] = conj(A^(k)[i][k]):
  // publishing a[k] through `slot` broadcasts the pivot column.
#pragma unroll
  for (int k = 0; k < U; ++k) {
    slot[l] = a[k];
    __syncwarp();
    float dk = slot[k].x;                        // A^(k)[k][k]
    const bool good = (dk > 0.f) && (dk < INFINITY);
    ok = ok && good;
    dk = good ? dk : 1.f;
    // (constant trip counts with compile-time guards so that nvcc unrolls fully
    // and a[] stays in registers)
    if (l > k) {
      const float il2 = __fdividef(1.f, dk);
      const float2 m = make_float2(a[k].x * il2, a[k].y * il2);  // conj(L[l][k]) / L[k][k]
#pragma unroll
      for (int i = 0; i < U; ++i)
        if (i > k) cfms_cj(a[i], slot[i], m);                      // a[i] -= L[i][k] conj(L[l][k])
    } else if (l == k) {
      const float il = rsqrtf(dk);
#pragma unroll
      for (int i = 0; i < U; ++i)
        if (i > k) { a[i].x *= il; a[i].y *= il; }                 // L[i][k]
      a[k] = make_float2(dk * il, 0.f);                            // L[k][k] = sqrt(dk)
    }
    __syncwarp();
  }
#pragma unroll
  for (int i = 0; i < U; ++i) M[l * MS + i] = a[i];                   // M[k][i] = L[i][k], i >= k
  __syncwarp();
  // ---- forward substitution L X = I; lane l holds column l of X = L^{-1}
  float2 x[U];
#pragma unroll
  for (int i = 0; i < U; ++i) x[i] = make_float2(i == l ? 1.f : 0.f, 0.f);
#pragma unroll
  for (int k = 0; k < U; ++k) {
    const float il = __fdividef(1.f, M[k * MS + k].x);
    const float2 xk = make_float2(x[k].x * il, x[k].y * il);
    x[k] = xk;
#pragma unroll
    for (int i = 0; i < U; ++i)
      if (i > k) cfms(x[i], M[k * MS + i], xk);                       // x[i] -= L[i][k] x[k]
  }
  __syncwarp();
  float t = 0.f;                                                      // tr A^{-1} = ||L^{-1}||_F^2
#pragma unroll
  for (int i = 0; i < U; ++i) { t += cabs2(x[i]); M[l * MS + i] = x[i]; }   // M[j][i] = W0[i][j]
  __syncwarp();
  // ---- back substitution A^{-1} = L^{-H} L^{-1}:  d[u] = sum_{m>=u} conj(W0[m][u]) W0[m][l]
  float f = 0.f;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int m = 0; m < U; ++m)
      if (m >= u) cfma_cj(acc, M[u * MS + m], x[m]);
    d[u] = acc;
    f += cabs2(acc);
  }
  t = sg_sum<U>(t);
  f = sg_sum<U>(f);
  // Lemma 1, Eq. (6):  beta^2 = Es/rho^2 (tr A^{-1} - kappa ||A^{-1}||_F^2)
  const float r = coef * (t - kappa * f);
  const bool good = (r > 0.f) && (r < INFINITY);
  ok = ok && good;
  __syncwarp();
  return good ? sqrtf(r) : 1.f;
}

// ------------------------------------------------------------------ whitening
// z_k[l] = ib * sum_v conj(d[v]) s_k[v]  (d = column l of Hermitian A^{-1}, so
// conj(d[v]) = A^{-1}[l][v]).  Written to zT for k in [kbeg, nkc*KC) step kstep,
// zeros for k >= K.
template <int U, int KC>
__device__ __forceinline__ void whiten_sg(const float2 (&d)[U], float ib, const float2 *__restrict__ s,
                                          int K, int kbeg, int kstep, float2 *zT, int l) {
  const int zs = ZL<KC>::zs(K);
  const int kend = ZL<KC>::nkc(K) * KC;
  for (int k = kbeg; k < kend; k += kstep) {
    float2 acc = make_float2(0.f, 0.f);
    if (k < K) {
      const float4 *sk = reinterpret_cast<const float4 *>(s + (size_t)k * U);
#pragma unroll
      for (int c = 0; c < U / 2; ++c) {
        const float4 v = __ldg(sk + c);
        cfma_cj(acc, d[2 * c], make_float2(v.x, v.y));
        cfma_cj(acc, d[2 * c + 1], make_float2(v.z, v.w));
      }
      acc.x *= ib; acc.y *= ib;
    }
    zT[ZL<KC>::idx(zs, l, k)] = acc;
  }
}

// ------------------------------------------------------------------ (c) precode
// x[k][b] = sum_u conj(H[b][u]) z[k][u] for rows b = l, l+U, ... < nrows of a tile.
// Writes x[k * xstride + b]; returns the lane's sum of |x|^2.
// Rows are absolute tile rows row0 + r; x is indexed by r.
template <int U, int KC>
__device__ __forceinline__ float precode_sg(const float2 *tile, int row0, int nrows, const float2 *zT, int K,
                                            float2 *__restrict__ x, size_t xstride, int l) {
  constexpr int KCP = ZL<KC>::KCP;
  const int zs = ZL<KC>::zs(K);
  float pw = 0.f;
  for (int b = l; b < nrows; b += U) {
    for (int k0 = 0, q = 0; k0 < K; k0 += KC, ++q) {
      float2 acc[KC];
#pragma unroll
      for (int j = 0; j < KC; ++j) acc[j] = make_float2(0.f, 0.f);
#pragma unroll 4
      for (int c = 0; c < U / 2; ++c) {
        const float4 h = tile_chunk<U>(tile, row0 + b, c);
        const float2 h0 = make_float2(h.x, h.y), h1 = make_float2(h.z, h.w);
        const float2 *z0 = zT + (2 * c) * zs + q * KCP;   // z[.][2c], broadcast within the SG
        const float2 *z1 = z0 + zs;                        // z[.][2c+1]
#pragma unroll
        for (int j = 0; j < KC; j += 2) {
          if (j + 1 < KC) {
            const float4 za = *reinterpret_cast<const float4 *>(z0 + j);
            const float4 zb = *reinterpret_cast<const float4 *>(z1 + j);
            cfma_cj(acc[j], h0, make_float2(za.x, za.y));
            cfma_cj(acc[j + 1], h0, make_float2(za.z, za.w));
            cfma_cj(acc[j], h1, make_float2(zb.x, zb.y));
            cfma_cj(acc[j + 1], h1, make_float2(zb.z, zb.w));
          } else {
            cfma_cj(acc[j], h0, z0[j]);
            cfma_cj(acc[j], h1, z1[j]);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < KC; ++j) {
        if (k0 + j < K) {
          x[(size_t)(k0 + j) * xstride + b] = acc[j];
          pw += cabs2(acc[j]);
        }
      }
    }
  }
  return pw;
}

// ------------------------------------------------------------------ kernel arguments
struct Args {
  const float2 *H;      // H_local [n_sc][Bl][U]
  const float2 *s;      // s [n_sc][K][U]
  float2 *x;            // x_local [n_sc][K][Bl]
  const float2 *G;      // packed Gram input  [n_sc][groups][U(U+1)/2]  (solve kernels)
  float2 *Gout;         // packed Gram output [n_sc][groups][U(U+1)/2]  (gram kernel)
  const float2 *zin;    // z input  [n_sc][zgroups][K][U]                (precode kernel)
  float2 *zout;         // z output [n_sc][groups][K][U]                 (solve kernel)
  float *beta;          // per-problem beta (NaN when not HPD)
  float *pw;            // per (subcarrier, chunk) power partials [n_sc][nchunks]
  int *bad;             // count of non-HPD problems
  int n_sc, Bl, K, S;   // S = rows per chunk
  int nchunks;          // chunks per subcarrier = Bl / S
  int groups;           // problems per subcarrier of the solve kernel
  int zgroups;          // z groups per subcarrier in precode (1 = shared by all chunks)
  int chunks_per_zgroup;
  float kappa, coef;    // regulariser and Es / rho_x^2
};

__host__ __device__ constexpr int npacked(int U) { return U * (U + 1) / 2; }
__device__ __forceinline__ int pidx(int U, int u, int v) {   // u <= v, row-major upper triangle
  return u * U - (u * (u - 1)) / 2 + (v - u);
}
// column l of G + kappa I from packed upper-triangle storage
template <int U>
__device__ __forceinline__ void load_packed_col(const float2 *Gp, int l, float kappa, float2 (&acc)[U]) {
#pragma unroll
  for (int u = 0; u < U; ++u) {
    float2 g;
    if (u <= l) g = Gp[pidx(U, u, l)];
    else { g = Gp[pidx(U, l, u)]; g.y = -g.y; }
    if (u == l) { g.x += kappa; g.y = 0.f; }
    acc[u] = g;
  }
}

// ================================================================== FD fused kernel
// One SG per (subcarrier, cluster) problem, NSG = (blockDim/32)*(32/U) problems per
// CTA with consecutive problem ids (= consecutive antenna rows of H_local).  Single
// pass over H: cp.async tile -> Gram -> +kappa_c -> Cholesky -> L^{-1} -> A^{-1}
// -> beta_c -> z = A^{-1} s / beta_c -> x_c = H_c^H z -> power partial.
// smem per SG: tile S*U + scratch max(Scr::SIZE, U*zs).
template <int U, int KC>
__global__ void __launch_bounds__(256) fd_fused_kernel(Args a) {
  constexpr int PPW = 32 / U;
  extern __shared__ __align__(16) float2 smem[];
  const int nw = blockDim.x >> 5;
  const int NSG = nw * PPW;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sg = warp * PPW + lane / U, l = lane % U;
  const int nprob = a.n_sc * a.nchunks;
  const int p0 = blockIdx.x * NSG;
  const int np = min(NSG, nprob - p0);
  const int zs = ZL<KC>::zs(a.K);
  const int scr_sz = max(Scr<U>::SIZE, U * zs);
  const int tile_sz = a.S * U;
  float2 *tile = smem + (size_t)sg * (tile_sz + scr_sz);
  float2 *scr = tile + tile_sz;
  {
    const float2 *g = a.H + (size_t)p0 * tile_sz;
    for (int q = 0; q < np; ++q)
      load_tile_async<U>(smem + (size_t)q * (tile_sz + scr_sz), g + (size_t)q * tile_sz, a.S, threadIdx.x,
                         blockDim.x);
    cp_async_wait_all();
    __syncthreads();
  }
  // Inactive SGs (tail CTA) run the warp-synchronous code on a clamped problem
  // and write nothing.
  const bool active = sg < np;
  const int p = active ? p0 + sg : p0;
  if (!active) tile = smem;   // valid, loaded data
  const int sc = p / a.nchunks, cl = p % a.nchunks;
  float2 acc[U];
#pragma unroll
  for (int i = 0; i < U; ++i) acc[i] = make_float2(0.f, 0.f);
  gram_sg<U>(tile, 0, a.S, l, acc);
#pragma unroll
  for (int i = 0; i < U; ++i)
    if (i == l) { acc[i].x += a.kappa; acc[i].y = 0.f; }
  float2 d[U];
  bool ok;
  const float beta = solve_sg<U>(acc, d, scr, l, a.kappa, a.coef, ok);
  const float ib = ok ? __fdividef(1.f, beta) : 0.f;   // failed problems output x = 0
  whiten_sg<U, KC>(d, ib, a.s + (size_t)sc * a.K * U, a.K, 0, 1, scr, l);
  __syncwarp();
  float pw = 0.f;
  if (active)
    pw = precode_sg<U, KC>(tile, 0, a.S, scr, a.K, a.x + (size_t)sc * a.K * a.Bl + (size_t)cl * a.S,
                           (size_t)a.Bl, l);
  pw = sg_sum<U>(pw);
  if (active && l == 0) {
    a.beta[p] = ok ? beta : qnan();
    a.pw[p] = pw;
    if (!ok) atomicAdd(a.bad, 1);
  }
}

// ================================================================== per-subcarrier CTA kernels
// One CTA per subcarrier; SG g handles chunk g (rows [g*S, (g+1)*S) of H_local[sc]).
// MODE_GRAM:          tile -> Gram per chunk -> (per chunk | adder tree) -> packed G out
// MODE_PD_FUSED:      tile -> Gram -> adder tree -> warp 0: solve + whiten -> precode
// MODE_SOLVE_PRECODE: packed G in -> warp 0: solve + whiten ; tile -> precode
// MODE_PRECODE:       z in (per z group) ; tile -> precode
// smem: [tile Bl*U][tree (nw/2)*U*MS][scr PPW*Scr::SIZE][zT zgroups*U*zs]
enum { MODE_GRAM = 0, MODE_PD_FUSED = 1, MODE_SOLVE_PRECODE = 2, MODE_PRECODE = 3 };

template <int U, int KC, int MODE, bool PER_CHUNK>
__global__ void __launch_bounds__(256) sc_kernel(Args a) {
  constexpr int PPW = 32 / U;
  constexpr int MS = Scr<U>::MS;
  extern __shared__ __align__(16) float2 smem[];
  const int nw = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sg = warp * PPW + lane / U, l = lane % U;
  const int sc = blockIdx.x;
  const int zs = ZL<KC>::zs(a.K);
  const int zg = (MODE == MODE_PRECODE) ? a.zgroups : 1;
  float2 *tile = smem;
  float2 *tree = tile + (size_t)a.Bl * U;
  float2 *scr = tree + (size_t)(nw / 2) * U * MS;
  float2 *zT = scr + (size_t)PPW * Scr<U>::SIZE;
  load_tile_async<U>(tile, a.H + (size_t)sc * a.Bl * U, a.Bl, threadIdx.x, blockDim.x);
  if (MODE == MODE_PRECODE) {
    const float2 *src = a.zin + (size_t)sc * zg * a.K * U;     // z[sc][g][k][u] -> zT[g]
    const int kend = ZL<KC>::nkc(a.K) * KC;
    for (int i = threadIdx.x; i < zg * U * kend; i += blockDim.x) {
      const int g = i / (U * kend), r = i % (U * kend), u = r / kend, k = r % kend;
      zT[(size_t)g * U * zs + ZL<KC>::idx(zs, u, k)] =
          (k < a.K) ? src[((size_t)g * a.K + k) * U + u] : make_float2(0.f, 0.f);
    }
  }
  cp_async_wait_all();
  __syncthreads();

  if (MODE == MODE_GRAM || MODE == MODE_PD_FUSED) {
    float2 acc[U];
#pragma unroll
    for (int i = 0; i < U; ++i) acc[i] = make_float2(0.f, 0.f);
    if (sg < a.nchunks) gram_sg<U>(tile, sg * a.S, a.S, l, acc);
    if (MODE == MODE_GRAM && PER_CHUNK) {
      if (sg < a.nchunks) {
        float2 *out = a.Gout + ((size_t)sc * a.nchunks + sg) * npacked(U);
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (u <= l) out[pidx(U, u, l)] = acc[u];
      }
      return;
    }
    // feedforward adder tree G = sum_c G_c: over the SGs of a warp, then
    // across warps, in a fixed order
#pragma unroll
    for (int m = U; m < 32; m <<= 1)
#pragma unroll
      for (int i = 0; i < U; ++i) {
        acc[i].x += __shfl_xor_sync(0xffffffffu, acc[i].x, m);
        acc[i].y += __shfl_xor_sync(0xffffffffu, acc[i].y, m);
      }
    for (int half = nw / 2; half >= 1; half >>= 1) {
      if (warp >= half && warp < 2 * half && lane < U) {
        float2 *buf = tree + (size_t)(warp - half) * U * MS;
#pragma unroll
        for (int i = 0; i < U; ++i) buf[i * MS + l] = acc[i];
      }
      __syncthreads();
      if (warp < half && lane < U) {
        const float2 *buf = tree + (size_t)warp * U * MS;
#pragma unroll
        for (int i = 0; i < U; ++i) { acc[i].x += buf[i * MS + l].x; acc[i].y += buf[i * MS + l].y; }
      }
      __syncthreads();
    }
    if (MODE == MODE_GRAM) {
      if (warp == 0 && lane < U) {
        float2 *out = a.Gout + (size_t)sc * npacked(U);
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (u <= l) out[pidx(U, u, l)] = acc[u];
      }
      return;
    }
    if (warp == 0) {
      // all SGs of warp 0 hold G (lane l of each SG: column l); SG 0 is
      // authoritative, the others redo the solve to share the whitening
      // SGs > 0 of warp 0 hold only warp 0's partial sum: take SG 0's column l
#pragma unroll
      for (int i = 0; i < U; ++i) {
        acc[i].x = __shfl_sync(0xffffffffu, acc[i].x, l);
        acc[i].y = __shfl_sync(0xffffffffu, acc[i].y, l);
      }
#pragma unroll
      for (int i = 0; i < U; ++i)
        if (i == l) { acc[i].x += a.kappa; acc[i].y = 0.f; }
      float2 d[U];
      bool ok;
      const float beta = solve_sg<U>(acc, d, scr + (size_t)(lane / U) * Scr<U>::SIZE, l, a.kappa, a.coef, ok);
      const float ib = ok ? __fdividef(1.f, beta) : 0.f;
      whiten_sg<U, KC>(d, ib, a.s + (size_t)sc * a.K * U, a.K, lane / U, PPW, zT, l);
      if (lane == 0) {
        a.beta[sc] = ok ? beta : qnan();
        if (!ok) atomicAdd(a.bad, 1);
      }
    }
    __syncthreads();
  }
  if (MODE == MODE_SOLVE_PRECODE) {
    if (warp == 0) {
      float2 acc[U];
      load_packed_col<U>(a.G + (size_t)sc * npacked(U), l, a.kappa, acc);
      float2 d[U];
      bool ok;
      const float beta = solve_sg<U>(acc, d, scr + (size_t)(lane / U) * Scr<U>::SIZE, l, a.kappa, a.coef, ok);
      const float ib = ok ? __fdividef(1.f, beta) : 0.f;
      whiten_sg<U, KC>(d, ib, a.s + (size_t)sc * a.K * U, a.K, lane / U, PPW, zT, l);
      if (lane == 0) {
        a.beta[sc] = ok ? beta : qnan();
        if (!ok) atomicAdd(a.bad, 1);
      }
    }
    __syncthreads();
  }
  // precode: SG g -> chunk g
  float pw = 0.f;
  if (sg < a.nchunks) {
    const int g = (MODE == MODE_PRECODE && zg > 1) ? sg / a.chunks_per_zgroup : 0;
    pw = precode_sg<U, KC>(tile, sg * a.S, a.S, zT + (size_t)g * U * zs, a.K,
                           a.x + (size_t)sc * a.K * a.Bl + (size_t)sg * a.S, (size_t)a.Bl, l);
  }
  pw = sg_sum<U>(pw);
  if (sg < a.nchunks && l == 0) a.pw[(size_t)sc * a.nchunks + sg] = pw;
}

// ================================================================== (b) standalone solve kernel
// One SG per (subcarrier, group) problem: packed G -> beta, z = A^{-1} s / beta.
// 4 warps per CTA.
template <int U>
__global__ void __launch_bounds__(128) solve_kernel(Args a) {
  constexpr int PPW = 32 / U;
  extern __shared__ __align__(16) float2 smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sg = warp * PPW + lane / U, l = lane % U;
  const int nprob = a.n_sc * a.groups;
  const int pr = blockIdx.x * (4 * PPW) + sg;
  const bool active = pr < nprob;
  const int p = active ? pr : nprob - 1;
  const int sc = p / a.groups;
  float2 *scr = smem + (size_t)sg * Scr<U>::SIZE;
  float2 acc[U];
  load_packed_col<U>(a.G + (size_t)p * npacked(U), l, a.kappa, acc);
  float2 d[U];
  bool ok;
  const float beta = solve_sg<U>(acc, d, scr, l, a.kappa, a.coef, ok);
  const float ib = ok ? __fdividef(1.f, beta) : 0.f;
  if (!active) return;
  const float2 *s = a.s + (size_t)sc * a.K * U;
  for (int k = 0; k < a.K; ++k) {
    float2 z = make_float2(0.f, 0.f);
#pragma unroll
    for (int v = 0; v < U; ++v) cfma_cj(z, d[v], __ldg(s + (size_t)k * U + v));
    a.zout[((size_t)p * a.K + k) * U + l] = make_float2(z.x * ib, z.y * ib);
  }
  if (l == 0) {
    a.beta[p] = ok ? beta : qnan();
    if (!ok) atomicAdd(a.bad, 1);
  }
}

// ================================================================== scalar finish
// Per subcarrier, fixed order over local parts: fin[sc] = {sum_c 1/beta_c (FD) or
// 1/beta (PD), sum of power partials}.
__global__ void finish_kernel(const float *beta, int nbeta, const float *pw, int npw, int n_sc, int fd,
                              float *fin) {
  const int sc = blockIdx.x * blockDim.x + threadIdx.x;
  if (sc >= n_sc) return;
  float ib = 0.f, p = 0.f;
  if (fd) {
    for (int c = 0; c < nbeta; ++c) ib += 1.f / beta[(size_t)sc * nbeta + c];
  } else {
    ib = 1.f / beta[sc];
  }
  for (int c = 0; c < npw; ++c) p += pw[(size_t)sc * npw + c];
  fin[2 * sc] = ib;
  fin[2 * sc + 1] = p;
}

// which: 1 -> rx = 1 / fin[.][0] ; 2 -> power = fin[.][1]
__global__ void read_scalars_kernel(const float *fin, int n_sc, int which, float *dst) {
  const int sc = blockIdx.x * blockDim.x + threadIdx.x;
  if (sc >= n_sc) return;
  dst[sc] = (which == 1) ? 1.f / fin[2 * sc] : fin[2 * sc + 1];
}

}  // namespace dpk
