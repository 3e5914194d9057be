// fd_small.cuh — FD-WF for small clusters B_c < U: the first branch of the
// per-cluster precoder,
//     Q_c = (H_c^H H_c + kappa_c I_{B_c})^{-1} H_c^H,     x_c = Q_c s / beta_c,
// with the B_c x B_c regularised Gram instead of the U x U one (same Q_c by the
// push-through identity when kappa_c > 0; "further reduces the computational
// complexity"; and still defined at kappa_c = 0 when H_c has full column rank).
// beta_c^2 = Es/rho_c^2 tr(Q_c^H Q_c) (Eq. 5 for the cluster) = Es/rho_c^2
// (tr W - kappa_c ||W||_F^2) with W = (H_c^H H_c + kappa_c I)^{-1}: the Lemma-1 form in
// the B_c x B_c space, so the same equilibrated Hermitian sweep (sweep_sg) applies.
//
// One sub-group of S lanes (S = 4, 8, 16 or 32, the power of two >= B_c) per (subcarrier,
// cluster) problem; lane a < B_c owns antenna a of the cluster (row a of H_c^T, column a of the
// B_c x B_c matrices):
//   G'[b][a] = sum_u conj(H[b][u]) H[a][u]                       (H_c^H H_c, column a)
//   -W[:, a], beta_c                                             (sweep_sg<S>, Lemma 1 form)
//   t_k[a] = sum_u conj(H[a][u]) s_k[u]                          (H_c^H s_k)
//   x_k[a] = (1/beta_c) sum_b W[a][b] t_k[b]                      (whiten_sg<S> on t)
// Any B_c < U: lanes a >= B_c are padding: their H row is zero and their diagonal is 1, so the
// padded matrix is block diagonal diag(H_c^H H_c + kappa_c I, I) -- the real block's inverse is
// untouched (exactly: the padding block is decoupled), the padding lanes are left out of
// tr W and ||W||_F^2 (sweep_sg's nvalid), and write nothing.
// Not on a BASELINE throughput config (all have B_c >= U): plain SIMT, no tensor cores.
#pragma once

namespace dpk {

// per-SG shared memory (complex): H rows [S][U] + s [K][U] + t [K][S] + zT [S][zs] + slot [2S]
template <int S, int U, int KC>
__host__ __device__ inline int fds_size(int K) {
  return S * U + K * U + K * S + S * ZL<KC>::zs(K) + 2 * S;
}

template <int S, int U, int KC>
__global__ void __launch_bounds__(128) fd_small_kernel(Args a) {
  pdl_trigger();   // early: the next kernel may launch once every CTA of this grid has started
                   // (it still waits for this grid's completion in griddepcontrol.wait; this kernel's
                   // own wait sits before its first output write, see below)
  constexpr int PPW = 32 / S;
  extern __shared__ __align__(16) float2 smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sg = warp * PPW + lane / S, l = lane % S;
  const int NSG = (int)(blockDim.x >> 5) * PPW;
  const int nprob = a.n_sc * a.nchunks;
  const int pr = blockIdx.x * NSG + sg;
  const bool active = pr < nprob;
  const int p = active ? pr : nprob - 1;          // inactive SGs redo the last problem, write nothing
  const int sc = p / a.nchunks, cl = p % a.nchunks;
  const int K = a.K;
  const int Bc = a.S;                             // actual cluster size (<= S; lanes >= Bc pad)
  const bool real = l < Bc;
  float2 *Hs = smem + (size_t)sg * fds_size<S, U, KC>(K);
  float2 *ss = Hs + S * U, *t = ss + K * U, *zT = t + K * S, *slot = zT + S * ZL<KC>::zs(K);
  // own row of H_c and the subcarrier's s
  {
    const float4 *src = reinterpret_cast<const float4 *>(a.H + ((size_t)sc * a.Bl + (size_t)cl * Bc + l) * U);
    float4 *dst = reinterpret_cast<float4 *>(Hs + l * U);
#pragma unroll
    for (int c = 0; c < U / 2; ++c) dst[c] = real ? src[c] : make_float4(0.f, 0.f, 0.f, 0.f);
    if (a.s_wait) pdl_wait();                                 // s from the broadcast: its kernel complete
    for (int i = l; i < K * U / 2; i += S)
      reinterpret_cast<float4 *>(ss)[i] = reinterpret_cast<const float4 *>(a.s + (size_t)sc * K * U)[i];
  }
  __syncwarp();
  const float2 *hl = Hs + l * U;
  // column l of A = H_c^H H_c + kappa_c I (S x S)
  float2 col[S];
#pragma unroll
  for (int b = 0; b < S; ++b) {
    const float2 *hb = Hs + b * U;
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int u = 0; u < U; ++u) cfma_cj(acc, hb[u], hl[u]);   // conj(H[b][u]) H[l][u]
    if (b == l) acc = make_float2(real ? acc.x + a.kappa : 1.f, 0.f);   // padding: unit diagonal
    col[b] = acc;
  }
  // t_k[l] = sum_u conj(H[l][u]) s_k[u]
  for (int k = 0; k < K; ++k) {
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int u = 0; u < U; ++u) cfma_cj(acc, hl[u], ss[k * U + u]);
    t[k * S + l] = acc;
  }
  __syncwarp();
  bool ok;
  const float beta = sweep_sg<S>(col, slot, l, a.kappa, a.coef, ok, Bc);   // col <- -W[:, l]
  const float ib = ok ? -__fdividef(1.f, beta) : 0.f;                    // failed problems: x = 0
  __syncwarp();
  whiten_sg<S, KC>(col, ib, t, K, 0, 1, zT, l);                          // zT[l][k] = x_k[l]
  __syncwarp();
  pdl_wait();   // H, s are inputs of the call; nothing above touches a predecessor's outputs
  float pw = 0.f;
  if (active && real) {
    const int zs = ZL<KC>::zs(K);
    float2 *x = a.x + (size_t)sc * K * a.Bl + (size_t)cl * Bc + l;
    for (int k = 0; k < K; ++k) {
      const float2 v = zT[ZL<KC>::idx(zs, l, k)];
      x[(size_t)k * a.Bl] = v;
      pw += cabs2(v);
    }
  }
  pw = sg_sum<S>(pw);
  if (active && l == 0) {
    a.beta[p] = ok ? beta : qnan();
    a.pw[p] = pw;
    if (!ok) atomicAdd(a.bad, 1);
  }
  pdl_trigger();
}

}  // namespace dpk
