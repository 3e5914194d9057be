// kernels.cuh — sm_100a kernels of the decentralized WF precoders
// (arXiv 1804.10987).  Included once, by dp_api.cu.
//
// Execution model.  All arithmetic is complex fp32 (the paper's
// precision, cuBLAS C* routines).  The unit of work is a SUB-GROUP
// (SG) of U consecutive lanes of a warp (U in {4, 8, 16, 32}; 32/U SGs per
// warp).  Lane l of an SG owns column l of the U x U matrices of its problem:
//   gram_sg    G = sum_b h_b h_b^H over a tile's rows, Hermitian-reduced
//              (G_c = H_c H_c^H)
//   solve_sg   A = G + kappa I = L D L^H (Cholesky in root-free LDL^H form,
//              P:285), W0 = L^{-1} (forward substitution), A^{-1} =
//              W0^H D^{-1} W0 (back substitution), and beta from
//              tr A^{-1} and ||A^{-1}||_F^2 (Lemma 1, Eq. 6)
//   whiten_sg  z_k = A^{-1} s_k / beta
//   precode_sg x_k[b] = sum_u conj(H[b][u]) z_k[u]              (x_c = H_c^H z)
// H tiles live in shared memory with a 16-byte-chunk XOR swizzle (period 8
// rows) so that both access patterns are conflict-free: row broadcast (Gram)
// and one row per lane (precode).  No atomics on data: every sum has a fixed
// order, so results are bit-reproducible run to run.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

namespace dpk {

// ------------------------------------------------------------------ complex helpers
// Complex multiply-accumulates run on the packed FP32 pipe (fma.rn.f32x2 -> FFMA2,
// sm_100a): one complex MAC = 2 FFMA2,  acc += P * y.x + Q * y.y  with P, Q derived
// from one operand.  ptxas folds the swaps / partial negations of P, Q and the
// broadcast of y.x, y.y into FFMA2 operand modifiers (.LO_HI, .NP, .F32), so no extra
// instructions are issued; the FMA pipe does the same work in half the issue slots.
__device__ __forceinline__ unsigned long long pk2(float2 a) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
  return r;
}
// d += a * b (element-wise, packed)
__device__ __forceinline__ void fma2(float2 &d, float2 a, float2 b) {
  unsigned long long D = pk2(d);
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(D) : "l"(pk2(a)), "l"(pk2(b)));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(D));
}
__device__ __forceinline__ void cmac2(float2 &acc, float2 P, float2 Q, float2 y) {
  fma2(acc, P, make_float2(y.x, y.x));
  fma2(acc, Q, make_float2(y.y, y.y));
}
// acc += a * conj(b)
__device__ __forceinline__ void cfma_bc(float2 &acc, float2 a, float2 b) {
  cmac2(acc, make_float2(b.x, -b.y), make_float2(b.y, b.x), a);
}
// acc += conj(a) * b
__device__ __forceinline__ void cfma_cj(float2 &acc, float2 a, float2 b) {
  cmac2(acc, make_float2(a.x, -a.y), make_float2(a.y, a.x), b);
}
// acc -= conj(a) * b
__device__ __forceinline__ void cfms_cj(float2 &acc, float2 a, float2 b) {
  cmac2(acc, make_float2(-b.x, -b.y), make_float2(-b.y, b.x), a);
}
// acc -= a * b
__device__ __forceinline__ void cfms(float2 &acc, float2 a, float2 b) {
  cmac2(acc, make_float2(-a.x, -a.y), make_float2(a.y, -a.x), b);
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
__device__ __forceinline__ float cabs2(float2 a) { return fmaf(a.x, a.x, a.y * a.y); }
__device__ __forceinline__ float qnan() { return __int_as_float(0x7fc00000); }
__device__ __forceinline__ float2 lo2(float4 v) { return make_float2(v.x, v.y); }
__device__ __forceinline__ float2 hi2(float4 v) { return make_float2(v.z, v.w); }

// sum over the U lanes of an SG (butterfly; every lane gets the total)
template <int U>
__device__ __forceinline__ float sg_sum(float v) {
#pragma unroll
  for (int m = U / 2; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m, U);
  return v;
}

// ------------------------------------------------------------------ swizzled H tile
// Tile row b holds U complex = U/2 16-byte chunks; chunk c of row b is stored at
// chunk position c ^ swz(b).  swz has period 8 in b for every U; 8 consecutive
// rows read at one chunk index land in 8 distinct 16-byte bank groups.
template <int U>
__host__ __device__ constexpr int swz(int b) {
  return (b / ((U / 2) >= 8 ? 1 : 8 / (U / 2))) % ((U / 2) >= 8 ? 8 : (U / 2));
}
template <int U>
__device__ __forceinline__ float4 ld_chunk(const float2 *row, int c, int sw) {
  return *reinterpret_cast<const float4 *>(row + 2 * (c ^ sw));
}
template <int U>
__device__ __forceinline__ float2 ld_elem(const float2 *row, int u, int sw) {
  return row[2 * ((u >> 1) ^ sw) + (u & 1)];
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

// Async copy of n complex (n even, 16-byte aligned) by the U lanes of an SG.
template <int U>
__device__ __forceinline__ void sg_copy_async(float2 *dst, const float2 *__restrict__ src, int n, int l) {
  for (int i = l; i < n / 2; i += U) cp_async16(dst + 2 * i, src + 2 * i);
}

// row stride (complex) of the transposed s and of z in the symbols-innermost whitening
// (whiten_Tg): 144-byte rows, 16-byte aligned, spread over the banks
constexpr int WT_SP = 18;

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
// Hermitian-reduced assignment of G entries to the U lanes of an SG:
//   top[r], r < U/2:  G[r][l]                        (rows 0..U/2-1, every column)
//   br[r],  r < U/4:  G[U/2 + (U/4)h + r][U/2 + l']   (bottom-right block, split in two
//                      row halves h = l / (U/2); column l' = l % (U/2))
// 3U/4 entries per lane instead of U, every load a broadcast (two addresses per
// warp for the bottom-right rows).  The lower-left block is (top-right)^H.
template <int U> struct GAcc {
  float2 top[U / 2];
  float2 br[U / 4];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < U / 2; ++i) top[i] = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < U / 4; ++i) br[i] = make_float2(0.f, 0.f);
  }
};

template <int U>
__device__ __forceinline__ void gram_row(const float2 *row, int sw, int l, GAcc<U> &g) {
  constexpr int H2 = U / 2, Q = U / 4;
  const int h = l / H2, lc = H2 + (l % H2);
  const float2 own = ld_elem<U>(row, l, sw);        // h_b[l]
  const float2 own2 = ld_elem<U>(row, lc, sw);      // h_b[U/2 + l']
#pragma unroll
  for (int c = 0; c < H2 / 2; ++c) {                // rows 0..U/2-1: broadcast
    const float4 v = ld_chunk<U>(row, c, sw);
    cfma_bc(g.top[2 * c], lo2(v), own);
    cfma_bc(g.top[2 * c + 1], hi2(v), own);
  }
  if constexpr (Q >= 2) {
#pragma unroll
    for (int c = 0; c < Q / 2; ++c) {               // rows U/2 + Q h + .. : two addresses per warp
      const float4 v = ld_chunk<U>(row, H2 / 2 + h * (Q / 2) + c, sw);
      cfma_bc(g.br[2 * c], lo2(v), own2);
      cfma_bc(g.br[2 * c + 1], hi2(v), own2);
    }
  } else {                                          // U = 4: one bottom-right row per lane
    cfma_bc(g.br[0], ld_elem<U>(row, H2 + h, sw), own2);
  }
}

// Gram over tile rows [row0, row0 + nrows); with row0 % 8 == 0 the swizzle of
// each 8-row group is a compile-time constant.
template <int U>
__device__ __forceinline__ void gram_sg(const float2 *tile, int row0, int nrows, int l, GAcc<U> &g) {
  int b = row0;
  const int end = row0 + nrows;
  if ((row0 & 7) == 0)
  for (; b + 8 <= end; b += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) gram_row<U>(tile + (size_t)(b + j) * U, swz<U>(j), l, g);
  }
  for (; b < end; ++b) gram_row<U>(tile + (size_t)b * U, swz<U>(b), l, g);
}

// Scatter a lane's entries into M[u][v] (row stride MS) and read back column l
// of the full Hermitian G + kappa I.
template <int U, int MS>
__device__ __forceinline__ void gram_to_column(const GAcc<U> &g, float2 *M, int l, float kappa,
                                               float2 (&a)[U]) {
  constexpr int H2 = U / 2, Q = U / 4;
  const int h = l / H2, lc = H2 + (l % H2);
#pragma unroll
  for (int r = 0; r < H2; ++r) M[r * MS + l] = g.top[r];
#pragma unroll
  for (int r = 0; r < Q; ++r) M[(H2 + Q * h + r) * MS + lc] = g.br[r];
  __syncwarp();
#pragma unroll
  for (int u = 0; u < U; ++u) {
    float2 v;
    if (u < H2 || l >= H2) v = M[u * MS + l];
    else v = cconj(M[l * MS + u]);                  // lower-left block = (top-right)^H
    if (u == l) { v.x += kappa; v.y = 0.f; }
    a[u] = v;
  }
  __syncwarp();
}

// Column l of G + kappa I straight from the Hermitian-reduced registers; only the
// lower-left block (= (top-right)^H) crosses lanes through shared memory:
//   u <  U/2           own top[u]
//   u >= U/2, l >= U/2 bottom-right: rows U/2 .. U/2+U/4-1 from lane l - U/2 (shuffle),
//                      the rest own br[]
//   u >= U/2, l <  U/2 conj(top[l] of lane u), transposed through T[U/2][U/2 + 2]
template <int U>
__host__ __device__ constexpr int tsz(int) { return (U / 2) * (U / 2 + 2); }
template <int U>
__device__ __forceinline__ void gacc_to_column(const GAcc<U> &g, float2 *T, int l, float kappa,
                                               float2 (&a)[U]) {
  constexpr int H2 = U / 2, Q = U / 4, TS = H2 + 2;
  const bool hi = l >= H2;
  if (hi) {
#pragma unroll
    for (int r = 0; r < H2; r += 2)
      *reinterpret_cast<float4 *>(T + (l - H2) * TS + r) =
          make_float4(g.top[r].x, g.top[r].y, g.top[r + 1].x, g.top[r + 1].y);
  }
  float2 nb[Q];
#pragma unroll
  for (int r = 0; r < Q; ++r) {
    nb[r].x = __shfl_xor_sync(0xffffffffu, g.br[r].x, H2, U);
    nb[r].y = __shfl_xor_sync(0xffffffffu, g.br[r].y, H2, U);
  }
  __syncwarp();
  const int lc = l % H2;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    float2 v;
    if (u < H2) {
      v = g.top[u];
    } else {
      const int j = u - H2;
      const float2 t = T[j * TS + lc];
      v = hi ? ((j < Q) ? nb[j] : g.br[j - Q]) : cconj(t);
    }
    if (u == l) { v.x += kappa; v.y = 0.f; }
    a[u] = v;
  }
  __syncwarp();
}

// Upper-triangle packed index (u <= v, row-major).
__host__ __device__ constexpr int npacked(int U) { return U * (U + 1) / 2; }
__device__ __forceinline__ int pidx(int U, int u, int v) { return u * U - (u * (u - 1)) / 2 + (v - u); }

// Write a lane's entries with u <= v to packed storage.
template <int U>
__device__ __forceinline__ void gram_store_packed(const GAcc<U> &g, float2 *out, int l) {
  constexpr int H2 = U / 2, Q = U / 4;
  const int h = l / H2, lc = H2 + (l % H2);
#pragma unroll
  for (int r = 0; r < H2; ++r)
    if (r <= l) out[pidx(U, r, l)] = g.top[r];
#pragma unroll
  for (int r = 0; r < Q; ++r) {
    const int u = H2 + Q * h + r;
    if (u <= lc) out[pidx(U, u, lc)] = g.br[r];
  }
}

// Column l of G + kappa I from packed upper-triangle storage.
template <int U>
__device__ __forceinline__ void load_packed_col(const float2 *Gp, int l, float kappa, float2 (&a)[U]) {
#pragma unroll
  for (int u = 0; u < U; ++u) {
    float2 g;
    if (u <= l) g = Gp[pidx(U, u, l)];
    else g = cconj(Gp[pidx(U, l, u)]);
    if (u == l) { g.x += kappa; g.y = 0.f; }
    a[u] = g;
  }
}

// ------------------------------------------------------------------ (b) solve
// Scratch per SG: slot[U] + M[U][MS] (MS = U + 2 keeps rows 16-byte aligned).
template <int U> struct Scr {
  static constexpr int MS = U + 2;
  static constexpr int SIZE = U + U * MS;   // complex elements
};
// FD fused scratch per SG: [slot 2U][T region]; the T region first holds the
// lower-left Gram block transpose (U/2 x (U/2 + 2)), then s (K x U, staged during
// the sweep) followed by zT.  (Reading s through L1 instead cost 8%: long-scoreboard
// stalls in the whitening loop.)
template <int U, int KC>
__host__ __device__ inline int fd_scr_size(int K) {
  const int m1 = (U / 2) * (U / 2 + 2);
  const int m2 = K <= 16 ? (K * U > U * WT_SP ? K * U : U * WT_SP) + U * WT_SP   // ss|zT, sT (whiten_Tg)
                         : K * U + U * ZL<KC>::zs(K);
  return 2 * U + (m1 > m2 ? m1 : m2);
}
// solve kernel scratch per SG: [slot 2U][packed G][s K x U][zT U x zs]
template <int U, int KC>
__host__ __device__ inline int solve_scr_size(int K) {
  if (K <= 16)                                            // ss | zT, sT (whiten_Tg)
    return 2 * U + U * (U + 1) / 2 + (K * U > U * WT_SP ? K * U : U * WT_SP) + U * WT_SP;
  return 2 * U + U * (U + 1) / 2 + K * U + U * ZL<KC>::zs(K);
}

// In: a[] = column l of A = G + kappa I (full Hermitian column).
// Out: d[] = column l of A^{-1}; returns beta (Lemma 1).  ok = false if a pivot
// of A is not a finite positive number (A not HPD) or beta's radicand is not.
// A = L D L^H with unit lower L: the root-free form of the Cholesky factor
// L_chol = L D^{1/2}.  The pivot column broadcast uses Hermitian symmetry.
template <int U>
__device__ __forceinline__ float solve_sg(float2 (&a)[U], float2 (&d)[U], float2 *scr, int l,
                                          float kappa, float coef, bool &ok) {
  float2 *slot = scr;
  float2 *M = scr + U;
  constexpr int MS = Scr<U>::MS;
  ok = true;
  // ---- LDL^H, right-looking.  Lane l holds column l of the trailing matrix incl.
  // its upper part, so lane i's a[k] = A^(k)[k][i] = conj(A^(k)[i][k]).
#pragma unroll
  for (int k = 0; k < U; ++k) {
    slot[l] = a[k];
    __syncwarp();
    float dk = slot[k].x;                                   // pivot d_k = A^(k)[k][k]
    const bool good = (dk > 0.f) && (dk < INFINITY);
    ok = ok && good;
    dk = good ? dk : 1.f;
    if (l > k) {
      const float2 m = cscale(a[k], __fdividef(1.f, dk));   // A^(k)[k][l] / d_k
#pragma unroll
      for (int i = 0; i < U; ++i)
        if (i > k) cfms_cj(a[i], slot[i], m);               // a[i] -= A[i][k] A[k][l] / d_k
    }
    if (l == k) a[k] = make_float2(dk, 0.f);
    __syncwarp();
  }
  // M[k][i] = A^(k)[i][k] = d_k L[i][k] (i > k);  M[k][k] = d_k
#pragma unroll
  for (int i = 0; i < U; ++i) M[l * MS + i] = a[i];
  __syncwarp();
  // ---- forward substitution L X = I (unit diagonal); lane l holds column l of W0 = L^{-1}
  float2 x[U];
#pragma unroll
  for (int i = 0; i < U; ++i) x[i] = make_float2(i == l ? 1.f : 0.f, 0.f);
  float t = 0.f;                                            // tr A^{-1} = sum_m |W0[m][l]|^2 / d_m
#pragma unroll
  for (int k = 0; k < U; ++k) {
    const float idk = __fdividef(1.f, M[k * MS + k].x);
    const float2 sk = cscale(x[k], idk);                    // W0[k][l] / d_k
    t = fmaf(sk.x, x[k].x, fmaf(sk.y, x[k].y, t));
    if (l == k) slot[k] = make_float2(idk, 0.f);
#pragma unroll
    for (int i = 0; i < U; ++i)
      if (i > k) cfms(x[i], M[k * MS + i], sk);             // x[i] -= L[i][k] x[k]
  }
  __syncwarp();
  // M[j][m] = W0[m][j] (lane j writes its column as row j), then x[m] <- W0[m][l] / d_m
#pragma unroll
  for (int i = 0; i < U; ++i) M[l * MS + i] = x[i];
  __syncwarp();
#pragma unroll
  for (int m = 0; m < U; ++m) x[m] = cscale(x[m], slot[m].x);
  // ---- A^{-1} = W0^H D^{-1} W0:  d[u] = sum_{m >= u} conj(W0[m][u]) W0[m][l] / d_m
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

// In-place symmetric (Hermitian) Gauss-Jordan sweep: pivot k performs the k-th
// step of the root-free Cholesky (LDL^H) elimination of the trailing block and,
// in the same pass, the k-th forward/back substitution step on the block already
// eliminated, so after U pivots w holds column l of -A^{-1} (Goodnight's sweep).
// Every lane updates every row at every pivot (no triangular lockstep waste), and
// the pivot row is broadcast through `slot` using Hermitian symmetry: lane i
// publishes its row-k entry a_ki = conj(a_ik).  The runtime pivot loop keeps the
// code small (instruction-cache resident): R pivots are unrolled per iteration and
// the register column is rotated by R rows at the end of it, so the pivot row is
// always a compile-time register.
// One-pivot look-ahead: at pivot k each lane first updates row k+1, publishes it
// (the next pivot row) into the other half of the double-buffered slot and issues
// the load + reciprocal of the next pivot, then updates the remaining rows; the
// broadcast / reciprocal latency of pivot k+1 hides behind pivot k's FMAs.
// In: w[] = column l of A = G + kappa I.  Out: w[] = column l of -A^{-1}; returns
// beta (Lemma 1, Eq. 6); ok = false if a pivot is not finite and positive (A not
// HPD) or beta's radicand is not.  slot: 2U complex.
template <int U>
__device__ __forceinline__ float sweep_sg(float2 (&w)[U], float2 *slot, int l, float kappa, float coef,
                                          bool &ok, int nvalid = U) {
  constexpr int R = U >= 4 ? 4 : U;
  ok = true;
  // ---- Jacobi equilibration A' = D^{-1/2} A D^{-1/2} (unit diagonal, pivots in (0, 1])
  float dl = 0.f;
#pragma unroll
  for (int p = 0; p < U; ++p)
    if (p == l) dl = w[p].x;
  ok = (dl > 0.f) && (dl < INFINITY);
  const float rl = ok ? rsqrtf(dl) : 1.f;
  slot[l] = make_float2(rl, 0.f);
  __syncwarp();
#pragma unroll
  for (int p = 0; p < U; p += 2) {
    const float4 r2 = *reinterpret_cast<const float4 *>(slot + p);
    w[p] = cscale(w[p], r2.x * rl);
    w[p + 1] = cscale(w[p + 1], r2.z * rl);
  }
  __syncwarp();
  // ---- sweep.  Buffer k & 1 holds pivot k's row at rotated positions (l - kk) & (U-1).
  slot[l] = w[0];
  __syncwarp();
  float id;
  {
    float d0 = slot[0].x;
    const bool g0 = (d0 > 0.f) && (d0 < INFINITY);
    ok = ok && g0;
    id = __fdividef(1.f, g0 ? d0 : 1.f);
  }
#pragma unroll 1
  for (int kk = 0; kk < U; kk += R) {
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int k = kk + j;                       // pivot (register position j holds row k)
      const float2 *cur = slot + (j & 1) * U;     // R even: the parity of k is the parity of j
      float2 *nxt = slot + ((j + 1) & 1) * U;
      const bool piv = (l == k);
      // Non-pivot lanes: a_pl -= a_pk a_kl / d.  The pivot lane's own column holds
      // a_pk, the Hermitian mirror of the broadcast conj(a_kp), so sigma = 1 - 1/d
      // turns it into a_pk / d (equal up to the rounding asymmetry of the mirrors,
      // which the unit-diagonal scaling keeps at the level of the pivots' rounding).
      const float2 sig = piv ? make_float2(1.f - id, 0.f) : cscale(w[j], id);
      const int jn = (j + 1 < U) ? j + 1 : 0;       // register position of row k+1 (U = R: wraps, unused)
      // 1. row k+1 first, published as the next pivot row
      float idn = 1.f;
      bool gn = true;
      if (j + 1 < U) {
        cfms_cj(w[jn], cur[jn], sig);
        const int shift = (j == R - 1) ? R : 0;   // next pivot opens a new block: its base is kk + R
        nxt[(l - kk - shift) & (U - 1)] = w[jn];
        __syncwarp();
        float dn = nxt[(j == R - 1) ? 0 : jn].x;  // a_{k+1,k+1}
        gn = (dn > 0.f) && (dn < INFINITY);
        idn = __fdividef(1.f, gn ? dn : 1.f);
      }
      // 2. the other rows
#pragma unroll
      for (int p = 0; p < U; p += 2) {
        const float4 sv = *reinterpret_cast<const float4 *>(cur + p);
        const bool done0 = (p == j) || (j + 1 < U && p == jn), done1 = (p + 1 == j) || (j + 1 < U && p + 1 == jn);
        if (!done0) cfms_cj(w[p], lo2(sv), sig);
        if (!done1) cfms_cj(w[p + 1], hi2(sv), sig);
      }
      w[j] = piv ? make_float2(-id, 0.f) : cscale(w[j], id);
      if (k + 1 < U) ok = ok && gn;
      id = idn;
      __syncwarp();                               // cur is rewritten as the slot of pivot k+2
    }
    float2 t[R];                                  // rotate rows up by R
#pragma unroll
    for (int q = 0; q < R; ++q) t[q] = w[q];
#pragma unroll
    for (int p = 0; p + R < U; ++p) w[p] = w[p + R];
#pragma unroll
    for (int q = 0; q < R; ++q) w[U - R + q] = t[q];
  }
  // ---- undo the equilibration: A^{-1} = D^{-1/2} A'^{-1} D^{-1/2}
  slot[l] = make_float2(rl, 0.f);
  __syncwarp();
  float tr = 0.f, f = 0.f;
#pragma unroll
  for (int p = 0; p < U; p += 2) {
    const float4 r2 = *reinterpret_cast<const float4 *>(slot + p);
    w[p] = cscale(w[p], r2.x * rl);
    w[p + 1] = cscale(w[p + 1], r2.z * rl);
    f += cabs2(w[p]) + cabs2(w[p + 1]);
    if (p == l) tr = -w[p].x;                     // diagonal of A^{-1}
    if (p + 1 == l) tr = -w[p + 1].x;
  }
  __syncwarp();
  if (l >= nvalid) tr = f = 0.f;                  // padding lanes (fd_small.cuh): decoupled unit block
  tr = sg_sum<U>(tr);
  f = sg_sum<U>(f);
  // Lemma 1, Eq. (6):  beta^2 = Es/rho^2 (tr A^{-1} - kappa ||A^{-1}||_F^2)
  const float r = coef * (tr - kappa * f);
  const bool good = (r > 0.f) && (r < INFINITY);
  ok = ok && good;
  return good ? sqrtf(r) : 1.f;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// sweep_sg with a leaner pivot step (used by fd_tc): the caller passes its diagonal
// entry dl = A[l][l]; reciprocals are rcp.approx.ftz (no denormal fix-up: equilibrated
// pivots lie in (0, 1]); the per-pivot validity test is replaced by running min / max
// of the pivots, checked once at the end (a NaN anywhere reaches tr A^{-1} and fails
// the radicand test).  Same arithmetic on every matrix entry as sweep_sg.
template <int U>
__device__ __forceinline__ float sweep_sg2(float2 (&w)[U], float2 *slot, int l, float dl, float kappa, float coef,
                                           bool &ok) {
  constexpr int R = U >= 4 ? 4 : U;
  const bool gd = (dl > 0.f) && (dl < INFINITY);
  const float rl = gd ? rsqrtf(dl) : 1.f;
  slot[l] = make_float2(rl, 0.f);
  __syncwarp();
#pragma unroll
  for (int p = 0; p < U; p += 2) {
    const float4 r2 = *reinterpret_cast<const float4 *>(slot + p);
    w[p] = cscale(w[p], r2.x * rl);
    w[p + 1] = cscale(w[p + 1], r2.z * rl);
  }
  __syncwarp();
  slot[l] = w[0];
  __syncwarp();
  float pmin = slot[0].x, pmax = pmin;
  float id = rcp_approx(pmin);
#pragma unroll 1
  for (int kk = 0; kk < U; kk += R) {
    const int rot = (l - kk) & (U - 1), rotn = (l - kk - R) & (U - 1);
    const bool last_blk = kk + R >= U;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int k = kk + j;
      const float2 *cur = slot + (j & 1) * U;
      float2 *nxt = slot + ((j + 1) & 1) * U;
      const bool piv = (l == k);
      const float2 sig = piv ? make_float2(1.f - id, 0.f) : cscale(w[j], id);
      const int jn = (j + 1 < U) ? j + 1 : 0;
      float idn = 1.f;
      if (j + 1 < U) {
        cfms_cj(w[jn], cur[jn], sig);
        nxt[(j == R - 1) ? rotn : rot] = w[jn];
        __syncwarp();
        float dn = nxt[(j == R - 1) ? 0 : jn].x;
        if (j == R - 1) dn = last_blk ? 1.f : dn;   // no pivot after the last one
        pmin = fminf(pmin, dn);
        pmax = fmaxf(pmax, dn);
        idn = rcp_approx(dn);
      }
#pragma unroll
      for (int p = 0; p < U; p += 2) {
        const float4 sv = *reinterpret_cast<const float4 *>(cur + p);
        const bool done0 = (p == j) || (j + 1 < U && p == jn), done1 = (p + 1 == j) || (j + 1 < U && p + 1 == jn);
        if (!done0) cfms_cj(w[p], lo2(sv), sig);
        if (!done1) cfms_cj(w[p + 1], hi2(sv), sig);
      }
      w[j] = piv ? make_float2(-id, 0.f) : cscale(w[j], id);
      id = idn;
      __syncwarp();
    }
    float2 t[R];
#pragma unroll
    for (int q = 0; q < R; ++q) t[q] = w[q];
#pragma unroll
    for (int p = 0; p + R < U; ++p) w[p] = w[p + R];
#pragma unroll
    for (int q = 0; q < R; ++q) w[U - R + q] = t[q];
  }
  slot[l] = make_float2(rl, 0.f);
  __syncwarp();
  float tr = 0.f, f = 0.f;
#pragma unroll
  for (int p = 0; p < U; p += 2) {
    const float4 r2 = *reinterpret_cast<const float4 *>(slot + p);
    w[p] = cscale(w[p], r2.x * rl);
    w[p + 1] = cscale(w[p + 1], r2.z * rl);
    f += cabs2(w[p]) + cabs2(w[p + 1]);
    if (p == l) tr = -w[p].x;
    if (p + 1 == l) tr = -w[p + 1].x;
  }
  __syncwarp();
  tr = sg_sum<U>(tr);
  f = sg_sum<U>(f);
  // Lemma 1, Eq. (6):  beta^2 = Es/rho^2 (tr A^{-1} - kappa ||A^{-1}||_F^2)
  const float r = coef * (tr - kappa * f);
  const bool all_gd = sg_sum<U>(gd ? 0.f : 1.f) == 0.f;   // every diagonal of this problem valid
  ok = all_gd && (pmin > 0.f) && (pmax < INFINITY) && (r > 0.f) && (r < INFINITY);
  if (!ok) {                                              // non-HPD: no NaN/Inf may reach the outputs
#pragma unroll
    for (int p = 0; p < U; ++p) w[p] = make_float2(0.f, 0.f);
  }
  return ok ? sqrtf(r) : 1.f;
}

// ------------------------------------------------------------------ whitening
// z_k[l] = ib * sum_v conj(d[v]) s_k[v]  (d = column l of Hermitian A^{-1}, so
// conj(d[v]) = A^{-1}[l][v]).  Written to zT for k in [kbeg, nkc*KC) step kstep,
// zeros for k >= K.  Two symbols per iteration for independent FMA chains.
template <int U, int KC, bool GS = false>
__device__ __forceinline__ void whiten_sg(const float2 (&d)[U], float ib, const float2 *s,
                                          int K, int kbeg, int kstep, float2 *zT, int l) {
  const int zs = ZL<KC>::zs(K);
  const int kend = ZL<KC>::nkc(K) * KC;
  for (int k = kbeg; k < kend; k += 2 * kstep) {
    const int k2 = k + kstep;
    float2 a0 = make_float2(0.f, 0.f), a1 = a0, b0 = a0, b1 = a0;
    const float4 *s0 = reinterpret_cast<const float4 *>(s + (size_t)min(k, K - 1) * U);
    const float4 *s1 = reinterpret_cast<const float4 *>(s + (size_t)min(k2, K - 1) * U);
#pragma unroll
    for (int c = 0; c < U / 2; ++c) {
      const float4 v = GS ? __ldg(s0 + c) : s0[c];   // GS: s read through L1 (global)
      const float4 w = GS ? __ldg(s1 + c) : s1[c];
      cfma_cj(a0, d[2 * c], lo2(v));
      cfma_cj(a1, d[2 * c + 1], hi2(v));
      cfma_cj(b0, d[2 * c], lo2(w));
      cfma_cj(b1, d[2 * c + 1], hi2(w));
    }
    const float ia = k < K ? ib : 0.f, ibb = k2 < K ? ib : 0.f;
    zT[ZL<KC>::idx(zs, l, k)] = make_float2((a0.x + a1.x) * ia, (a0.y + a1.y) * ia);
    if (k2 < kend) zT[ZL<KC>::idx(zs, l, k2)] = make_float2((b0.x + b1.x) * ibb, (b0.y + b1.y) * ibb);
  }
}

// Whitening with the symbols innermost (K <= 16, one chunk of KC) for an SG of U lanes:
//   z_k[l] = ib * sum_v conj(d[v]) s_k[v],  d = column l of -A^{-1} (Hermitian), ib = -1/beta,
// for all k at once: per v one conj(d[v]) multiplier feeds KC independent accumulators (no long
// dependent FMA chains); s read from a transposed copy sT[v][k] (row stride WT_SP complex,
// broadcast loads within the SG); z written as zT[u][k] (row stride WT_SP).
template <int U, int KC>
__device__ __forceinline__ void whiten_Tg(const float2 (&d)[U], float ib, const float2 *sT, float2 *zT, int K, int l) {
  constexpr int KP = (KC + 1) & ~1;
  float2 acc[KP];
#pragma unroll
  for (int j = 0; j < KP; ++j) acc[j] = make_float2(0.f, 0.f);
#pragma unroll
  for (int v = 0; v < U; ++v) {
    const float4 *row = reinterpret_cast<const float4 *>(sT + v * WT_SP);
#pragma unroll
    for (int j = 0; j < KP; j += 2) {
      const float4 sv = row[j >> 1];
      cfma_cj(acc[j], d[v], lo2(sv));
      cfma_cj(acc[j + 1], d[v], hi2(sv));
    }
  }
  float4 *zo = reinterpret_cast<float4 *>(zT + l * WT_SP);
#pragma unroll
  for (int j = 0; j < KP; j += 2) {
    const float a0 = j < K ? ib : 0.f, a1 = j + 1 < K ? ib : 0.f;
    zo[j >> 1] = make_float4(acc[j].x * a0, acc[j].y * a0, acc[j + 1].x * a1, acc[j + 1].y * a1);
  }
}
// sT[l][k] = s_k[l] (lane l of the SG writes its row; zero padded to KP) from ss [K][U]
template <int U, int KC>
__device__ __forceinline__ void transpose_s(const float2 *ss, float2 *sT, int K, int l) {
  constexpr int KP = (KC + 1) & ~1;
  float4 *row = reinterpret_cast<float4 *>(sT + l * WT_SP);
#pragma unroll
  for (int j = 0; j < KP; j += 2) {
    const float2 s0 = j < K ? ss[j * U + l] : make_float2(0.f, 0.f);
    const float2 s1 = j + 1 < K ? ss[(j + 1) * U + l] : make_float2(0.f, 0.f);
    row[j >> 1] = make_float4(s0.x, s0.y, s1.x, s1.y);
  }
}

// ------------------------------------------------------------------ (c) precode
// x[k][r] = sum_u conj(H[row0 + r][u]) z[k][u] for r = l, l+U, ... < nrows.
// Writes x[k * xstride + r]; returns the lane's sum of |x|^2.
template <int U, int KC>
__device__ __forceinline__ float precode_sg(const float2 *tile, int row0, int nrows, const float2 *zT, int K,
                                            float2 *__restrict__ x, size_t xstride, int l, int zs_ = 0,
                                            int rfirst = -1, int rstep = U) {
  constexpr int KCP = ZL<KC>::KCP;
  const int zs = zs_ ? zs_ : ZL<KC>::zs(K);
  float pw = 0.f;
  for (int r = rfirst < 0 ? l : rfirst; r < nrows; r += rstep) {
    const int b = row0 + r;
    const float2 *row = tile + (size_t)b * U;
    const int sw = swz<U>(b);
    for (int k0 = 0, q = 0; k0 < K; k0 += KC, ++q) {
      float2 acc[KC];
#pragma unroll
      for (int j = 0; j < KC; ++j) acc[j] = make_float2(0.f, 0.f);
      const float2 *zq = zT + q * KCP;
#pragma unroll 4
      for (int c = 0; c < U / 2; ++c) {
        const float4 h = ld_chunk<U>(row, c, sw);
        const float2 h0 = lo2(h), h1 = hi2(h);
        const float2 *z0 = zq + (2 * c) * zs;              // z[.][2c], broadcast within the SG
        const float2 *z1 = z0 + zs;                        // z[.][2c+1]
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
      for (int j = 0; j < KC; ++j) {
        if (k0 + j < K) {
          x[(size_t)(k0 + j) * xstride + r] = acc[j];
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
  const float2 *G;      // packed Gram input  [n_sc][groups][U(U+1)/2]  (solve kernel)
  float2 *Gout;         // packed Gram output [n_sc][groups][U(U+1)/2]  (gram kernel)
  const float2 *zin;    // z input  [n_sc][zgroups][K][U]                (precode kernel)
  float2 *zout;         // z output [n_sc][groups][K][U]                 (solve kernel)
  float2 *Wout;         // prepare: W = A^{-1}/beta packed [n_sc][groups][U(U+1)/2] (solve kernel; no z)
  float *beta;          // per-problem beta (NaN when not HPD)
  float *pw;            // per (subcarrier, chunk) power partials [n_sc][nchunks]
  int *bad;             // count of non-HPD problems
  int n_sc, Bl, K, S;   // S = rows per chunk
  int nchunks;          // chunks per subcarrier = Bl / S
  int groups;           // problems per subcarrier of the solve kernel
  int zgroups;          // z groups per subcarrier in precode (1 = shared by all chunks)
  int chunks_per_zgroup;
  float kappa, coef;    // regulariser and Es / rho_x^2
  float *fin;           // [n_sc][2]: {sum 1/beta (PD: 1/beta, FD: over local clusters), sum power}
  int nbeta;            // beta entries per subcarrier: PD 1, FD clusters per rank
  int fin_inv_beta;     // 1: fin[.][0] = sum 1/beta ; 0: fin[.][0] = 0 (PD ranks != 0)
  int pf_dist;          // fd_tc: L2-prefetch the tiles of CTA blockIdx.x + pf_dist (0: off)
  int fold;             // fd_tc: per-subcarrier scalars in-kernel (CTAs per subcarrier; 0 = finish kernel)
  int hrow_off;         // host only: H rows before a.H in its allocation (unequal-cluster runs; TMA extent)
  int rep;              // fd_fused: sub-groups per problem (1, 2, 4, 8; 0 = 1), see fd_fused_kernel
  int s_wait;           // single-pass FD kernels: s was written by a collective / kernel earlier on the
                        // stream (the s broadcast), so griddepcontrol.wait before reading it
  double kappa64, coef64;   // DP_FLAG_FP64 kernels (f64.cuh): kappa and coef unrounded
};

// Programmatic dependent launch: wait for the predecessor grid's completion (and
// memory flush) before touching its outputs; let the successor start launching.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// named barrier over n threads; plain mbarrier arrive (tensor-core kernels' hand-offs)
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t *mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(mbar)) : "memory");
}

// Per-subcarrier scalars in a fixed order over the local parts (read through L2:
// other CTAs wrote them).
__device__ __forceinline__ void finish_sc(const Args &a, int sc) {
  float ib = 0.f, p = 0.f;
  for (int c = 0; c < a.nbeta; ++c) ib += 1.f / __ldcg(a.beta + (size_t)sc * a.nbeta + c);
  for (int c = 0; c < a.nchunks; ++c) p += __ldcg(a.pw + (size_t)sc * a.nchunks + c);
  a.fin[2 * sc] = a.fin_inv_beta ? ib : 0.f;
  a.fin[2 * sc + 1] = p;
}

// ================================================================== FD fused kernel
// One SG per (subcarrier, cluster) problem, NSG = (blockDim/32)*(32/U) problems per
// CTA with consecutive problem ids (= consecutive antenna rows of H_local).  Single
// pass over H: cp.async tile -> Gram -> +kappa_c -> LDL^H -> L^{-1} -> A^{-1}
// -> beta_c -> z = A^{-1} s / beta_c -> x_c = H_c^H z -> power partial.
// smem per SG: tile S*U + scratch U + max(U/2 (U/2 + 2), K*U + U*zs).
template <int U, int KC>
__global__ void __launch_bounds__(128, U == 16 ? 4 : 3) fd_fused_kernel(Args a) {
  pdl_trigger();   // early: the next kernel may launch once every CTA of this grid has started
                   // (it still waits for this grid's completion in griddepcontrol.wait; this kernel's
                   // own wait sits before its first output write, see below)
  constexpr int PPW = 32 / U;
  extern __shared__ __align__(16) float2 smem[];
  const int nw = blockDim.x >> 5;
  const int NSG = nw * PPW;
  // R = a.rep sub-groups (replicas) per problem, consecutive lane groups of one warp: the antenna
  // rows of the Gram and of the precode are split over them (their Gram partials summed by a
  // butterfly, identical in every replica), the U x U sweep and the whitening run in every replica
  // (same operands, same results); replica 0 writes the scalars.  R > 1 gives the small problems
  // (U <= 16, few rows per lane) R times the lanes: shorter dependent chains and more warps.
  const int R = a.rep > 1 ? a.rep : 1;
  const int NPB = NSG / R;                                // problems per CTA
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sg = warp * PPW + lane / U, l = lane % U;
  const int q = sg / R, rj = sg % R;                      // problem within the CTA, replica
  const int nprob = a.n_sc * a.nchunks;
  const int p0 = blockIdx.x * NPB;
  const int np = min(NPB, nprob - p0);
  const int scr_sz = fd_scr_size<U, KC>(a.K);
  const int tile_sz = a.S * U;
  const int pstride = tile_sz + R * scr_sz;               // per problem: [tile][R scratch]
  float2 *tile = smem + (size_t)q * pstride;
  float2 *scr = tile + tile_sz + (size_t)rj * scr_sz;
  {
    if (a.Bl == a.nchunks * a.S) {   // clusters contiguous in H: problem p at p S rows
      const float2 *g = a.H + (size_t)p0 * tile_sz;
      for (int qq = 0; qq < np; ++qq)
        load_tile_async<U>(smem + (size_t)qq * pstride, g + (size_t)qq * tile_sz, a.S, threadIdx.x, blockDim.x);
    } else {                         // a run of unequal clusters: cluster (sc, cl) at rows sc Bl + cl S
      for (int qq = 0; qq < np; ++qq) {
        const int pq = p0 + qq;
        const float2 *g = a.H + ((size_t)(pq / a.nchunks) * a.Bl + (size_t)(pq % a.nchunks) * a.S) * U;
        load_tile_async<U>(smem + (size_t)qq * pstride, g, a.S, threadIdx.x, blockDim.x);
      }
    }
    cp_async_wait_all();
    __syncthreads();
  }
  // Inactive SGs (tail CTA) run the warp-synchronous code on problem 0's data and write nothing.
  const bool active = q < np;
  const int p = active ? p0 + q : p0;
  if (!active) tile = smem;
  const int sc = p / a.nchunks, cl = p % a.nchunks;
  float2 *slot = scr, *T = scr + 2 * U, *ss = scr + 2 * U, *zT = ss + a.K * U;
  float2 col[U];
  {
    GAcc<U> g;
    g.zero();
    const int rows = a.S / R;                             // host: S % R == 0
    gram_sg<U>(tile, rj * rows, rows, l, g);
    for (int m = U; m < R * U; m <<= 1) {                 // sum the replicas' partials (butterfly)
#pragma unroll
      for (int i = 0; i < U / 2; ++i) {
        g.top[i].x += __shfl_xor_sync(0xffffffffu, g.top[i].x, m);
        g.top[i].y += __shfl_xor_sync(0xffffffffu, g.top[i].y, m);
      }
#pragma unroll
      for (int i = 0; i < U / 4; ++i) {
        g.br[i].x += __shfl_xor_sync(0xffffffffu, g.br[i].x, m);
        g.br[i].y += __shfl_xor_sync(0xffffffffu, g.br[i].y, m);
      }
    }
    gacc_to_column<U>(g, T, l, a.kappa, col);
  }
  // stage s_k of this subcarrier into the (now free) T region while the sweep runs
  if (a.s_wait) pdl_wait();
  sg_copy_async<U>(ss, a.s + (size_t)sc * a.K * U, a.K * U, l);
  bool ok;
  float dl = 0.f;                                         // this lane's diagonal entry A[l][l]
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (u == l) dl = col[u].x;
  const float beta = sweep_sg2<U>(col, slot, l, dl, a.kappa, a.coef, ok);   // col <- -A^{-1}[:, l]
  const float ib = ok ? -__fdividef(1.f, beta) : 0.f;   // sign folds -A^{-1}; failed problems: x = 0
  cp_async_wait_all();
  __syncwarp();
  int zs = 0;                                             // zT row stride for the precode
  if (a.K <= 16) {                                        // symbols innermost over a transposed s
    float2 *sT = ss + (a.K * U > U * WT_SP ? a.K * U : U * WT_SP);
    transpose_s<U, KC>(ss, sT, a.K, l);
    __syncwarp();
    zT = ss;                                              // ss is dead after the transpose
    whiten_Tg<U, KC>(col, ib, sT, zT, a.K, l);
    zs = WT_SP;
  } else {
    whiten_sg<U, KC>(col, ib, ss, a.K, 0, 1, zT, l);
  }
  __syncwarp();
  pdl_wait();   // H, s are inputs of the call; nothing above touches a predecessor's outputs
  float pw = 0.f;
  if (active)
    pw = precode_sg<U, KC>(tile, 0, a.S, zT, a.K, a.x + (size_t)sc * a.K * a.Bl + (size_t)cl * a.S,
                           (size_t)a.Bl, l, zs, rj * U + l, R * U);
  pw = sg_sum<U>(pw);
  for (int m = U; m < R * U; m <<= 1) pw += __shfl_xor_sync(0xffffffffu, pw, m);
  if (active && l == 0 && rj == 0) {
    a.beta[p] = ok ? beta : qnan();
    a.pw[p] = pw;
    if (!ok) atomicAdd(a.bad, 1);
  }
  if (a.fold) {
    // the CTA's NPB problems are whole subcarriers (NPB % nchunks == 0): per-subcarrier scalars
    // here, in the order of finish_sc (ascending cluster), instead of fd_finish_kernel
    __shared__ float fb[32], fp[32];
    if (l == 0 && rj == 0) { fb[q] = 1.f / (ok ? beta : qnan()); fp[q] = pw; }
    __syncthreads();
    const int per = NPB / a.nchunks;
    if ((int)threadIdx.x < per) {
      const int q0 = threadIdx.x * a.nchunks;
      if (p0 + q0 < nprob) {
        const int sc0 = (p0 + q0) / a.nchunks;
        float b = 0.f, w = 0.f;
        for (int c = 0; c < a.nchunks; ++c) { b += fb[q0 + c]; w += fp[q0 + c]; }
        a.fin[2 * sc0] = a.fin_inv_beta ? b : 0.f;
        a.fin[2 * sc0 + 1] = w;
      }
    }
  }
  pdl_trigger();
}

// ================================================================== (a) Gram kernel
// One CTA per subcarrier; SG g computes the Gram of chunk g (rows [g*S, (g+1)*S)
// of H_local[sc]).  PER_CHUNK: packed Gram per chunk.  Otherwise the feedforward
// adder tree G = sum_c G_c: over the SGs of a warp (butterfly), then across
// warps through shared memory, in a fixed order; packed G out.
// smem: [tile Bl*U][tree (nw/2) * 32 * (3U/4) complex]
template <int U, bool PER_CHUNK>
__global__ void __launch_bounds__(256) gram_kernel(Args a) {
  pdl_trigger();   // early: the next kernel may launch once every CTA of this grid has started
                   // (it still waits for this grid's completion in griddepcontrol.wait)
  pdl_wait();
  constexpr int PPW = 32 / U;
  constexpr int NE = U / 2 + U / 4;
  extern __shared__ __align__(16) float2 smem[];
  const int nw = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sg = warp * PPW + lane / U, l = lane % U;
  const int sc = blockIdx.x;
  float2 *tile = smem;
  float2 *tree = tile + (size_t)a.Bl * U;
  load_tile_async<U>(tile, a.H + (size_t)sc * a.Bl * U, a.Bl, threadIdx.x, blockDim.x);
  cp_async_wait_all();
  __syncthreads();
  GAcc<U> g;
  g.zero();
  if (sg < a.nchunks) gram_sg<U>(tile, sg * a.S, a.S, l, g);
  if constexpr (PER_CHUNK) {
    if (sg < a.nchunks) gram_store_packed<U>(g, a.Gout + ((size_t)sc * a.nchunks + sg) * npacked(U), l);
  } else {
#pragma unroll
    for (int m = U; m < 32; m <<= 1) {
#pragma unroll
      for (int i = 0; i < U / 2; ++i) {
        g.top[i].x += __shfl_xor_sync(0xffffffffu, g.top[i].x, m);
        g.top[i].y += __shfl_xor_sync(0xffffffffu, g.top[i].y, m);
      }
#pragma unroll
      for (int i = 0; i < U / 4; ++i) {
        g.br[i].x += __shfl_xor_sync(0xffffffffu, g.br[i].x, m);
        g.br[i].y += __shfl_xor_sync(0xffffffffu, g.br[i].y, m);
      }
    }
    for (int half = nw / 2; half >= 1; half >>= 1) {
      if (warp >= half && warp < 2 * half) {
        float2 *buf = tree + ((size_t)(warp - half) * 32 + lane) * NE;
#pragma unroll
        for (int i = 0; i < U / 2; ++i) buf[i] = g.top[i];
#pragma unroll
        for (int i = 0; i < U / 4; ++i) buf[U / 2 + i] = g.br[i];
      }
      __syncthreads();
      if (warp < half) {
        const float2 *buf = tree + ((size_t)warp * 32 + lane) * NE;
#pragma unroll
        for (int i = 0; i < U / 2; ++i) { g.top[i].x += buf[i].x; g.top[i].y += buf[i].y; }
#pragma unroll
        for (int i = 0; i < U / 4; ++i) { g.br[i].x += buf[U / 2 + i].x; g.br[i].y += buf[U / 2 + i].y; }
      }
      __syncthreads();
    }
    if (warp == 0 && lane < U) gram_store_packed<U>(g, a.Gout + (size_t)sc * npacked(U), l);
  }
}

// ================================================================== (b) solve kernel
// One SG per (subcarrier, group) problem: packed G -> +kappa -> LDL^H -> A^{-1}
// -> beta -> z = A^{-1} s / beta (written as z[p][k][u]).  4 warps per CTA.
template <int U, int KC>
__global__ void __launch_bounds__(128) solve_kernel(Args a) {
  pdl_trigger();   // early: the next kernel may launch once every CTA of this grid has started
                   // (it still waits for this grid's completion in griddepcontrol.wait)
  pdl_wait();
  constexpr int PPW = 32 / U;
  extern __shared__ __align__(16) float2 smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sg = warp * PPW + lane / U, l = lane % U;
  const int nprob = a.n_sc * a.groups;
  const int pr = blockIdx.x * ((int)(blockDim.x >> 5) * PPW) + sg;   // 1-4 warps per CTA
  const bool active = pr < nprob;
  const int p = active ? pr : nprob - 1;
  const int sc = p / a.groups;
  const int zs = ZL<KC>::zs(a.K);
  constexpr int NP = npacked(U);
  float2 *slot = smem + (size_t)sg * solve_scr_size<U, KC>(a.K);
  float2 *Gs = slot + 2 * U, *ss = Gs + NP, *zT = ss + a.K * U;
  sg_copy_async<U>(Gs, a.G + (size_t)p * NP, NP, l);
  if (!a.Wout) sg_copy_async<U>(ss, a.s + (size_t)sc * a.K * U, a.K * U, l);   // prepare: no symbols
  cp_async_wait_all();
  __syncwarp();
  float2 col[U];
  load_packed_col<U>(Gs, l, a.kappa, col);
  bool ok = true;
  const float dl = Gs[pidx(U, l, l)].x + a.kappa;          // diagonal entry of this lane's column
#ifndef DP_SOLVE_ABL
#define DP_SOLVE_ABL 0   // diagnostics builds only: 1 no sweep, 2 no whitening (timing ablation)
#endif
  const float beta = (DP_SOLVE_ABL & 1) ? 1.f : sweep_sg2<U>(col, slot, l, dl, a.kappa, a.coef, ok);   // col <- -A^{-1}[:, l]
  const float ib = ok ? -__fdividef(1.f, beta) : 0.f;
  if (a.Wout) {                                   // prepare: cache W = A^{-1} / beta (upper, packed)
    if (active) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (u <= l) a.Wout[(size_t)p * NP + pidx(U, u, l)] = cscale(col[u], ib);
      if (l == 0) {
        a.beta[p] = ok ? beta : qnan();
        if (!ok) atomicAdd(a.bad, 1);
      }
    }
    pdl_trigger();
    return;
  }
  __syncwarp();
  if (a.K <= 16) {                                        // symbols innermost over a transposed s
    float2 *sT = ss + (a.K * U > U * WT_SP ? a.K * U : U * WT_SP);
    transpose_s<U, KC>(ss, sT, a.K, l);
    __syncwarp();
    zT = ss;
    if (!(DP_SOLVE_ABL & 2)) whiten_Tg<U, KC>(col, ib, sT, zT, a.K, l);
  } else {
    whiten_sg<U, KC>(col, ib, ss, a.K, 0, 1, zT, l);
  }
  __syncwarp();
  if (!active) return;
  float2 *zo = a.zout + (size_t)p * a.K * U;
  for (int k = 0; k < a.K; ++k) zo[(size_t)k * U + l] = zT[a.K <= 16 ? l * WT_SP + k : ZL<KC>::idx(zs, l, k)];
  if (l == 0) {
    a.beta[p] = ok ? beta : qnan();
    if (!ok) atomicAdd(a.bad, 1);
  }
  pdl_trigger();
}

// ================================================================== apply: whitening from cached W
// One SG per (subcarrier, group) problem: z_k = W s_k with the W = A^{-1}/beta cached by
// a prepare call (packed Hermitian), for the a.K symbols of this apply call (P:286-289:
// the whitening matrix is computed once per channel and applied to every symbol).
template <int U, int KC>
__global__ void __launch_bounds__(128) whiten_kernel(Args a) {
  pdl_trigger();   // early: the next kernel may launch once every CTA of this grid has started
                   // (it still waits for this grid's completion in griddepcontrol.wait)
  pdl_wait();
  constexpr int PPW = 32 / U;
  constexpr int NP = npacked(U);
  extern __shared__ __align__(16) float2 smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sg = warp * PPW + lane / U, l = lane % U;
  const int nprob = a.n_sc * a.groups;
  const int pr = blockIdx.x * ((int)(blockDim.x >> 5) * PPW) + sg;
  const bool active = pr < nprob;
  const int p = active ? pr : nprob - 1;
  const int sc = p / a.groups;
  const int zs = ZL<KC>::zs(a.K);
  float2 *Ws = smem + (size_t)sg * (NP + a.K * U + U * zs);
  float2 *ss = Ws + NP, *zT = ss + a.K * U;
  sg_copy_async<U>(Ws, a.G + (size_t)p * NP, NP, l);
  sg_copy_async<U>(ss, a.s + (size_t)sc * a.K * U, a.K * U, l);
  cp_async_wait_all();
  __syncwarp();
  float2 col[U];
  load_packed_col<U>(Ws, l, 0.f, col);            // column l of W (Hermitian; real diagonal)
  whiten_sg<U, KC>(col, 1.f, ss, a.K, 0, 1, zT, l);
  __syncwarp();
  if (!active) return;
  float2 *zo = a.zout + (size_t)p * a.K * U;
  for (int k = 0; k < a.K; ++k) zo[(size_t)k * U + l] = zT[ZL<KC>::idx(zs, l, k)];
  pdl_trigger();
}

// ================================================================== (c) precode kernel
// One CTA per subcarrier; SG g precodes chunk g with the z of its z group:
// x_c = H_c^H z plus the power partial of the chunk.
// smem: [tile Bl*U][zT zgroups*U*zs]
template <int U, int KC>
__global__ void __launch_bounds__(256) precode_kernel(Args a) {
  pdl_trigger();   // early: the next kernel may launch once every CTA of this grid has started
                   // (it still waits for this grid's completion in griddepcontrol.wait)
  pdl_wait();
  constexpr int PPW = 32 / U;
  extern __shared__ __align__(16) float2 smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sg = warp * PPW + lane / U, l = lane % U;
  const int sc = blockIdx.x;
  const int zs = ZL<KC>::zs(a.K);
  const int zg = a.zgroups;
  float2 *tile = smem;
  float2 *zT = tile + (size_t)a.Bl * U;
  load_tile_async<U>(tile, a.H + (size_t)sc * a.Bl * U, a.Bl, threadIdx.x, blockDim.x);
  {
    const float2 *src = a.zin + (size_t)sc * zg * a.K * U;     // z[sc][g][k][u] -> zT[g]
    const int kend = ZL<KC>::nkc(a.K) * KC;
    for (int i = threadIdx.x; i < zg * U * kend; i += blockDim.x) {
      const int g = i / (U * kend), r = i % (U * kend), k = r / U, u = r % U;
      zT[(size_t)g * U * zs + ZL<KC>::idx(zs, u, k)] =
          (k < a.K) ? src[((size_t)g * a.K + k) * U + u] : make_float2(0.f, 0.f);
    }
  }
  cp_async_wait_all();
  __syncthreads();
  float pw = 0.f;
  if (sg < a.nchunks) {
    const int g = (zg > 1) ? sg / a.chunks_per_zgroup : 0;
    pw = precode_sg<U, KC>(tile, sg * a.S, a.S, zT + (size_t)g * U * zs, a.K,
                           a.x + (size_t)sc * a.K * a.Bl + (size_t)sg * a.S, (size_t)a.Bl, l);
  }
  pw = sg_sum<U>(pw);
  if (sg < a.nchunks && l == 0) a.pw[(size_t)sc * a.nchunks + sg] = pw;
  __syncthreads();
  if (threadIdx.x == 0) finish_sc(a, sc);
  pdl_trigger();
}

// ================================================================== MRT baseline (Fig. 2)
// Fully-distributed MRT: per (subcarrier, cluster) problem one warp,
// Q_c = H_c^H (matched filter), beta_c = sqrt(Es ||H_c||_F^2 / rho_c^2) (Eq. 5 on the
// cluster, coef = Es / rho_c^2), x_c = H_c^H s / beta_c and the power partial.
template <int U>
__global__ void __launch_bounds__(128) mrt_kernel(Args a) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ __align__(16) float2 smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nprob = a.n_sc * a.nchunks;
  const int p = blockIdx.x * 4 + warp;
  if (p >= nprob) return;
  const int sc = p / a.nchunks, cl = p % a.nchunks;
  const float2 *Hc = a.H + ((size_t)sc * a.Bl + (size_t)cl * a.S) * U;
  float2 *ss = smem + (size_t)warp * a.K * U;
  for (int i = lane; i < a.K * U; i += 32) ss[i] = a.s[(size_t)sc * a.K * U + i];
  float fro = 0.f;
  for (int i = lane; i < a.S * U; i += 32) fro += cabs2(Hc[i]);
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) fro += __shfl_xor_sync(0xffffffffu, fro, m);
  const float beta = sqrtf(a.coef * fro);
  const bool ok = beta > 0.f && beta < INFINITY;
  const float ib = ok ? 1.f / beta : 0.f;
  __syncwarp();
  float pw = 0.f;
  for (int b = lane; b < a.S; b += 32) {
    float2 h[U];
#pragma unroll
    for (int u = 0; u < U; ++u) h[u] = Hc[(size_t)b * U + u];
    for (int k = 0; k < a.K; ++k) {
      float2 acc = make_float2(0.f, 0.f);
#pragma unroll
      for (int u = 0; u < U; ++u) cfma_cj(acc, h[u], ss[k * U + u]);      // conj(H[b][u]) s_k[u]
      acc = cscale(acc, ib);
      a.x[((size_t)sc * a.K + k) * a.Bl + (size_t)cl * a.S + b] = acc;
      pw += cabs2(acc);
    }
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) pw += __shfl_xor_sync(0xffffffffu, pw, m);
  // receive scale (reading R24): the cluster's array gain g_c = ||H_c||_F^2 / U (H_c H_c^H ~ g_c I)
  // enters the joint UE scaling, rx = 1 / sum_c (g_c / beta_c); the finish kernel sums 1/beta[],
  // so the effective per-cluster scale beta_c / g_c is stored
  if (lane == 0) {
    a.beta[p] = ok ? beta * (float)U / fro : qnan();
    a.pw[p] = pw;
    if (!ok) atomicAdd(a.bad, 1);
  }
}

// ================================================================== FD scalar finish
// Per subcarrier, fixed order over the local clusters: fin[sc] = {sum_c 1/beta_c,
// sum_c power_c}.  (A separate grid: folding it into the fused kernel needs a
// release fence per cluster, which waits for that warp's x stores and cost ~10%.)
// G = a power of two >= the rank's clusters lanes per subcarrier (a.rep reused as G, set by the
// launcher): lane c loads cluster c's beta and power partial (coalesced, one load per lane instead of a
// dependent load per term), lane 0 of the group sums them in ascending cluster order through
// shuffles -- the order of finish_sc, so the scalars are bit-identical to it and to the in-kernel folds.
static __global__ void __launch_bounds__(128) fd_finish_kernel(Args a) {
  pdl_trigger();   // early: the next kernel may launch once every CTA of this grid has started
                   // (it still waits for this grid's completion in griddepcontrol.wait)
  pdl_wait();
  if (a.rep == 0) {                                        // > 32 partials: one thread per subcarrier
    const int sc = blockIdx.x * blockDim.x + threadIdx.x;
    if (sc < a.n_sc) finish_sc(a, sc);
    return;
  }
  const int G = a.rep, t = blockIdx.x * blockDim.x + threadIdx.x;
  const int sc = t / G, c = t % G, lane = threadIdx.x & 31, base = lane - c;
  const bool in = sc < a.n_sc;
  const float vb = (in && c < a.nbeta) ? 1.f / __ldcg(a.beta + (size_t)sc * a.nbeta + c) : 0.f;
  const float vp = (in && c < a.nchunks) ? __ldcg(a.pw + (size_t)sc * a.nchunks + c) : 0.f;
  float ib = 0.f, p = 0.f;
  for (int j = 0; j < a.nbeta; ++j) ib += __shfl_sync(0xffffffffu, vb, base + j);
  for (int j = 0; j < a.nchunks; ++j) p += __shfl_sync(0xffffffffu, vp, base + j);
  if (in && c == 0) {
    a.fin[2 * sc] = a.fin_inv_beta ? ib : 0.f;
    a.fin[2 * sc + 1] = p;
  }
}

// ================================================================== FD finish, unequal clusters
// Clusters of unequal size / power / tau (Eq. 9) run as maximal runs of equal
// parameters, one FD launch per run; run r wrote beta and power partials of its len[r]
// clusters to vb / vp + n_sc cl0[r] in [sc][len[r]] layout.  Per subcarrier: beta_c ->
// a.beta[sc][Cl], fin = {sum_c 1/beta_c, sum_c power_c}.
constexpr int VAR_MAX_RUNS = 64;
struct VarRuns {
  int n, Cl;
  const float *vb, *vp;
  int cl0[VAR_MAX_RUNS], len[VAR_MAX_RUNS];
};
static __global__ void __launch_bounds__(128) fd_var_finish_kernel(Args a, VarRuns r) {
  pdl_trigger();
  pdl_wait();
  // one warp per subcarrier, lane = cluster (strided); butterfly sums in a fixed order
  const int sc = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (sc >= a.n_sc) return;
  float ib = 0.f, p = 0.f;
  for (int c = lane; c < r.Cl; c += 32) {
    int i = 0;
    while (i + 1 < r.n && r.cl0[i + 1] <= c) ++i;       // run of cluster c
    const size_t o = (size_t)a.n_sc * r.cl0[i] + (size_t)sc * r.len[i] + (c - r.cl0[i]);
    const float b = __ldcg(r.vb + o);
    a.beta[(size_t)sc * r.Cl + c] = b;
    ib += 1.f / b;
    p += __ldcg(r.vp + o);
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    ib += __shfl_xor_sync(0xffffffffu, ib, m);
    p += __shfl_xor_sync(0xffffffffu, p, m);
  }
  if (lane == 0) {
    a.fin[2 * sc] = ib;
    a.fin[2 * sc + 1] = p;
  }
}

// which: 1 -> rx = 1 / fin[.][0] ; 2 -> power = fin[.][1]
static __global__ void read_scalars_kernel(const float *fin, int n_sc, int which, float *dst) {
  const int sc = blockIdx.x * blockDim.x + threadIdx.x;
  if (sc >= n_sc) return;
  dst[sc] = (which == 1) ? 1.f / fin[2 * sc] : fin[2 * sc + 1];
}

}  // namespace dpk
