// f64.cuh — the DP_FLAG_FP64 kernels: the same per-problem steps as the fp32 path with every
// accumulation in fp64 (inputs H, s and outputs x stay complex64).
//
// Why (SURVEY §7 hard part 1): x = H_c^H (H_c H_c^H + kappa I)^{-1} s is dominated by
// the smallest singular directions of H_c; its relative error is ~ eps * cond(A).  A square
// Rayleigh cluster (B_c = U) at 40 dB (kappa_c ~ 3e-3) or in the ZF limit (N0 = 0) has
// cond(A) of 1e4 .. 1e9, so fp32 (eps 6e-8) misses the 1e-4 bar there; fp64 (eps 1.1e-16) does not.
// B200 executes fp64 FMAs at half the fp32 rate (DFMA), so this is an option, not the default.
//
// Steps (each lane l of a sub-group (SG) of U lanes owns column l of its problem's U x U matrices):
//   gram64      G[u][l] = sum_b H[b][u] conj(H[b][l])            (G_c = H_c H_c^H; products of
//                                                                 fp32 inputs are exact in fp64)
//   sweep64     -A^{-1} by the equilibrated Hermitian Gauss-Jordan sweep of A = G + kappa I (pivot k:
//               M[i][j] -= M[i][k] M[k][j] / M[k][k], column / row k scaled by 1 / M[k][k], diagonal
//               -1 / M[k][k]: the Cholesky-type elimination fused with its substitutions);
//               beta = sqrt(Es / rho_x^2 (tr A^{-1} - kappa ||A^{-1}||_F^2))  (Lemma 1, Eq. 6)
//   whiten64    z_k = A^{-1} s_k / beta
//   precode64   x_k[b] = sum_u conj(H[b][u]) z_k[u]               (x_c = H_c^H z)
// Non-HPD problems (a pivot not finite and positive, or a non-positive beta radicand) are flagged
// and zeroed exactly as on the fp32 path.
#pragma once

namespace dpk {

__device__ __forceinline__ double2 d2(float2 v) { return make_double2((double)v.x, (double)v.y); }
// acc += a * conj(b)
__device__ __forceinline__ void dfma_bc(double2 &acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, fma(a.y, b.y, acc.x));
  acc.y = fma(a.y, b.x, fma(-a.x, b.y, acc.y));
}
// acc += conj(a) * b
__device__ __forceinline__ void dfma_cj(double2 &acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, fma(a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(-a.y, b.x, acc.y));
}
// acc -= conj(a) * b
__device__ __forceinline__ void dfms_cj(double2 &acc, double2 a, double2 b) {
  acc.x = fma(-a.x, b.x, fma(-a.y, b.y, acc.x));
  acc.y = fma(-a.x, b.y, fma(a.y, b.x, acc.y));
}
__device__ __forceinline__ double dabs2(double2 a) { return fma(a.x, a.x, a.y * a.y); }

template <int U>
__device__ __forceinline__ double sg_sum64(double v) {
#pragma unroll
  for (int m = U / 2; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m, U);
  return v;
}

// G[u][l] over tile rows [0, rows) of a swizzled tile (load_tile_async<U>)
template <int U>
__device__ __forceinline__ void gram64(const float2 *tile, int rows, int l, double2 (&g)[U]) {
#pragma unroll
  for (int u = 0; u < U; ++u) g[u] = make_double2(0.0, 0.0);
  for (int b = 0; b < rows; ++b) {
    const float2 *row = tile + (size_t)b * U;
    const int sw = swz<U>(b);
    const double2 own = d2(ld_elem<U>(row, l, sw));
#pragma unroll
    for (int c = 0; c < U / 2; ++c) {
      const float4 v = ld_chunk<U>(row, c, sw);
      dfma_bc(g[2 * c], d2(lo2(v)), own);
      dfma_bc(g[2 * c + 1], d2(hi2(v)), own);
    }
  }
}

// In: w = column l of A (Hermitian, real diagonal).  Out: w = column l of -A^{-1}; returns beta.
// slot: U double2 of SG scratch.
template <int U>
__device__ __forceinline__ double sweep64(double2 (&w)[U], double2 *slot, int l, double kappa, double coef,
                                          bool &ok) {
  double dl = 0.0;
#pragma unroll
  for (int p = 0; p < U; ++p)
    if (p == l) dl = w[p].x;
  const bool gd = (dl > 0.0) && (dl < INFINITY);
  const double rl = gd ? 1.0 / sqrt(dl) : 1.0;
  slot[l] = make_double2(rl, 0.0);
  __syncwarp();
#pragma unroll
  for (int p = 0; p < U; ++p) {                       // Jacobi equilibration (unit diagonal)
    const double r = slot[p].x * rl;
    w[p] = make_double2(w[p].x * r, w[p].y * r);
  }
  __syncwarp();
  double pmin = INFINITY, pmax = 0.0;
#pragma unroll
  for (int k = 0; k < U; ++k) {
    slot[l] = w[k];                                   // row k: M[k][l]
    __syncwarp();
    const double d = slot[k].x;                       // pivot M[k][k] (a Schur complement of A)
    pmin = fmin(pmin, d);
    pmax = fmax(pmax, d);
    const double id = 1.0 / d;
    // lanes l != k: M[i][l] -= M[i][k] M[k][l] / d with M[i][k] = conj(M[k][i]) = conj(slot[i]);
    // lane k holds M[i][k] = conj(slot[i]) itself, so m = 1 - 1/d turns the same update into M[i][k] / d
    const double2 m = (l == k) ? make_double2(1.0 - id, 0.0) : make_double2(w[k].x * id, w[k].y * id);
#pragma unroll
    for (int i = 0; i < U; ++i)
      if (i != k) dfms_cj(w[i], slot[i], m);
    w[k] = (l == k) ? make_double2(-id, 0.0) : m;
    __syncwarp();
  }
  slot[l] = make_double2(rl, 0.0);
  __syncwarp();
  double tr = 0.0, f = 0.0;
#pragma unroll
  for (int p = 0; p < U; ++p) {                       // undo the equilibration
    const double r = slot[p].x * rl;
    w[p] = make_double2(w[p].x * r, w[p].y * r);
    f += dabs2(w[p]);
    if (p == l) tr = -w[p].x;
  }
  __syncwarp();
  tr = sg_sum64<U>(tr);
  f = sg_sum64<U>(f);
  // Lemma 1, Eq. (6):  beta^2 = Es/rho_x^2 (tr A^{-1} - kappa ||A^{-1}||_F^2)
  const double r = coef * (tr - kappa * f);
  const bool all_gd = sg_sum64<U>(gd ? 0.0 : 1.0) == 0.0;
  ok = all_gd && (pmin > 0.0) && (pmax < INFINITY) && (r > 0.0) && (r < INFINITY);
  if (!ok) {
#pragma unroll
    for (int p = 0; p < U; ++p) w[p] = make_double2(0.0, 0.0);
  }
  return ok ? sqrt(r) : 1.0;
}

// z[k][l] = ib sum_v conj(w[v]) s[k][v]  (w = column l of -A^{-1}, ib = -1/beta), s [K][U] complex64
template <int U>
__device__ __forceinline__ void whiten64(const double2 (&w)[U], double ib, const float2 *s, int K, double2 *z,
                                         int l) {
  for (int k = 0; k < K; ++k) {
    const float4 *sk = reinterpret_cast<const float4 *>(s + (size_t)k * U);
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int c = 0; c < U / 2; ++c) {
      const float4 v = sk[c];
      dfma_cj(acc, w[2 * c], d2(lo2(v)));
      dfma_cj(acc, w[2 * c + 1], d2(hi2(v)));
    }
    z[(size_t)k * U + l] = make_double2(acc.x * ib, acc.y * ib);
  }
}

// x[k * xstride + b] = sum_u conj(H[b][u]) z[k][u] for rows b = l, l + U, .. < rows of a swizzled tile;
// returns the lane's sum of |x|^2
template <int U>
__device__ __forceinline__ double precode64(const float2 *tile, int rows, const double2 *z, int K,
                                            float2 *__restrict__ x, size_t xstride, int l) {
  double pw = 0.0;
  for (int b = l; b < rows; b += U) {
    const float2 *row = tile + (size_t)b * U;
    const int sw = swz<U>(b);
    float2 h[U];
#pragma unroll
    for (int c = 0; c < U / 2; ++c) {
      const float4 v = ld_chunk<U>(row, c, sw);
      h[2 * c] = lo2(v);
      h[2 * c + 1] = hi2(v);
    }
    for (int k = 0; k < K; ++k) {
      const double2 *zk = z + (size_t)k * U;
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < U; ++u) dfma_cj(acc, d2(h[u]), zk[u]);
      const float2 o = make_float2((float)acc.x, (float)acc.y);
      x[(size_t)k * xstride + b] = o;
      pw += dabs2(d2(o));
    }
  }
  return pw;
}

// per-SG shared memory of fd_f64_kernel (bytes): tile S x U complex64 | s K x U complex64 |
// z K x U complex128 | slot U complex128
__host__ __device__ inline size_t f64_sg_bytes(int S, int U, int K) {
  return (size_t)S * U * 8 + (size_t)K * U * 8 + (size_t)K * U * 16 + (size_t)U * 16;
}

// ================================================================== FD in fp64
// One SG per (subcarrier, cluster) problem (cluster (sc, cl) = rows sc Bl + cl S of H_local),
// NSG = (blockDim / 32) (32 / U) problems per CTA.  beta[p], pw[p] per problem; the per-subcarrier
// scalars follow in fd_finish_kernel.
template <int U>
__global__ void __launch_bounds__(128) fd_f64_kernel(Args a) {
  pdl_trigger();
  pdl_wait();
  constexpr int PPW = 32 / U;
  extern __shared__ __align__(16) uint8_t smem8[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sg = warp * PPW + lane / U, l = lane % U;
  const int NSG = (int)(blockDim.x >> 5) * PPW;
  const int nprob = a.n_sc * a.nchunks;
  const int pr = blockIdx.x * NSG + sg;
  const bool active = pr < nprob;
  const int p = active ? pr : nprob - 1;                 // inactive SGs redo the last problem, write nothing
  const int sc = p / a.nchunks, cl = p % a.nchunks;
  const int S = a.S, K = a.K;
  uint8_t *base = smem8 + (size_t)sg * f64_sg_bytes(S, U, K);
  float2 *tile = reinterpret_cast<float2 *>(base);
  float2 *ss = tile + (size_t)S * U;
  double2 *z = reinterpret_cast<double2 *>(ss + (size_t)K * U);
  double2 *slot = z + (size_t)K * U;
  load_tile_async<U>(tile, a.H + ((size_t)sc * a.Bl + (size_t)cl * S) * U, S, l, U);
  sg_copy_async<U>(ss, a.s + (size_t)sc * K * U, K * U, l);
  cp_async_wait_all();
  __syncwarp();
  double2 w[U];
  gram64<U>(tile, S, l, w);
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (u == l) w[u] = make_double2(w[u].x + (double)a.kappa64, 0.0);   // A = G_c + kappa_c I (Eq. 9)
  bool ok;
  const double beta = sweep64<U>(w, slot, l, a.kappa64, a.coef64, ok);
  const double ib = ok ? -1.0 / beta : 0.0;               // failed problems: x = 0
  whiten64<U>(w, ib, ss, K, z, l);
  __syncwarp();
  double pw = 0.0;
  if (active) pw = precode64<U>(tile, S, z, K, a.x + (size_t)sc * K * a.Bl + (size_t)cl * S, (size_t)a.Bl, l);
  pw = sg_sum64<U>(pw);
  if (active && l == 0) {
    a.beta[p] = ok ? (float)beta : qnan();
    a.pw[p] = (float)pw;
    if (!ok) atomicAdd(a.bad, 1);
  }
  pdl_trigger();
}

// ================================================================== PD in fp64: (a) Gram
// One CTA per subcarrier: packed G64[sc][i] = sum_b H[b][u] conj(H[b][v]) over the rank's Bl rows
// (the first levels of the adder tree G = sum_c G_c), entry i = (u <= v) row-major, each
// thread summing its entries over b in ascending order.
template <int U>
__global__ void __launch_bounds__(128) gram_f64_kernel(Args a, double2 *G64) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ __align__(16) float2 smem[];
  const int sc = blockIdx.x;
  float2 *tile = smem;                                   // [Bl][U], unswizzled
  const float4 *src = reinterpret_cast<const float4 *>(a.H + (size_t)sc * a.Bl * U);
  for (int i = threadIdx.x; i < a.Bl * U / 2; i += blockDim.x) cp_async16(tile + 2 * i, src + i);
  cp_async_wait_all();
  __syncthreads();
  constexpr int NP = npacked(U);
  for (int i = threadIdx.x; i < NP; i += blockDim.x) {
    int u = 0, r = i;
    while (r >= U - u) { r -= U - u; ++u; }
    const int v = u + r;
    double2 acc = make_double2(0.0, 0.0);
    for (int b = 0; b < a.Bl; ++b) dfma_bc(acc, d2(tile[b * U + u]), d2(tile[b * U + v]));
    G64[(size_t)sc * NP + i] = acc;
  }
  pdl_trigger();
}

// ================================================================== PD in fp64: (b) whitening node
// One SG per subcarrier: A = G + kappa I from the packed G64 (summed over all ranks), sweep, beta,
// z64[sc][k][u] = A^{-1} s_k / beta.
template <int U>
__global__ void __launch_bounds__(128) solve_f64_kernel(Args a, const double2 *G64, double2 *z64) {
  pdl_trigger();
  pdl_wait();
  constexpr int PPW = 32 / U, NP = npacked(U);
  extern __shared__ __align__(16) uint8_t smem8[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sg = warp * PPW + lane / U, l = lane % U;
  const int NSG = (int)(blockDim.x >> 5) * PPW;
  const int pr = blockIdx.x * NSG + sg;
  const bool active = pr < a.n_sc;
  const int sc = active ? pr : a.n_sc - 1;
  const int K = a.K;
  float2 *ss = reinterpret_cast<float2 *>(smem8 + (size_t)sg * ((size_t)K * U * 8 + U * 16));
  double2 *slot = reinterpret_cast<double2 *>(ss + (size_t)K * U);
  sg_copy_async<U>(ss, a.s + (size_t)sc * K * U, K * U, l);
  double2 w[U];
  const double2 *g = G64 + (size_t)sc * NP;
#pragma unroll
  for (int u = 0; u < U; ++u) {                           // column l of the Hermitian G + kappa I
    double2 v;
    if (u <= l) v = g[pidx(U, u, l)];
    else { v = g[pidx(U, l, u)]; v.y = -v.y; }
    if (u == l) v = make_double2(v.x + a.kappa64, 0.0);
    w[u] = v;
  }
  cp_async_wait_all();
  __syncwarp();
  bool ok;
  const double beta = sweep64<U>(w, slot, l, a.kappa64, a.coef64, ok);
  const double ib = ok ? -1.0 / beta : 0.0;
  if (active) whiten64<U>(w, ib, ss, K, z64 + (size_t)sc * K * U, l);
  if (active && l == 0) {
    a.beta[sc] = ok ? (float)beta : qnan();
    if (!ok) atomicAdd(a.bad, 1);
  }
  pdl_trigger();
}

// ================================================================== PD in fp64: (c) precode
// One CTA per subcarrier: x[sc][k][b] = sum_u conj(H[b][u]) z64[sc][k][u] for the rank's Bl rows
// (one thread per row), the power of the subcarrier and fin[sc] = {1/beta (rank 0), power}.
template <int U>
__global__ void __launch_bounds__(128) precode_f64_kernel(Args a, const double2 *z64) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ __align__(16) double2 zs[];
  __shared__ double red[4];
  const int sc = blockIdx.x, K = a.K;
  for (int i = threadIdx.x; i < K * U; i += blockDim.x) zs[i] = z64[(size_t)sc * K * U + i];
  __syncthreads();
  double pw = 0.0;
  for (int b = threadIdx.x; b < a.Bl; b += blockDim.x) {
    float2 h[U];
    const float4 *src = reinterpret_cast<const float4 *>(a.H + ((size_t)sc * a.Bl + b) * U);
#pragma unroll
    for (int c = 0; c < U / 2; ++c) {
      const float4 v = __ldg(src + c);
      h[2 * c] = lo2(v);
      h[2 * c + 1] = hi2(v);
    }
    for (int k = 0; k < K; ++k) {
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < U; ++u) dfma_cj(acc, d2(h[u]), zs[k * U + u]);
      const float2 o = make_float2((float)acc.x, (float)acc.y);
      a.x[((size_t)sc * K + k) * a.Bl + b] = o;
      pw += dabs2(d2(o));
    }
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) pw += __shfl_xor_sync(0xffffffffu, pw, m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = pw;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    a.fin[2 * sc] = a.fin_inv_beta ? 1.f / a.beta[sc] : 0.f;
    a.fin[2 * sc + 1] = (float)t;
  }
  pdl_trigger();
}

}  // namespace dpk
