// solve_mw.cuh — regularised U x U solve for U = 32 with the rows of each problem
// split over 4 warps (one CTA per problem).  Same math and outputs as solve_kernel
// (kernels.cuh):  A = G + kappa I (Eq. 5 / Eq. 9),  -A^{-1} by the equilibrated
// Hermitian Gauss-Jordan sweep (the Cholesky-type LDL^H elimination fused with its
// substitutions),  beta by Lemma 1 (Eq. 6),  z_k = A^{-1} s_k / beta
// (P:174-177).
//
// Why split: the PD whitening node has one problem per subcarrier (1200 at cfg4), so
// one warp per problem leaves 2 warps per SM sub-partition and the sweep's serial
// pivot chain (publish row k+1 -> barrier -> reciprocal -> 32-row update) is exposed.
// Here lane l of warp w holds column l, rows 8w .. 8w+7: a pivot costs each warp 8
// row updates (16 FFMA2) instead of 32, four times as many warps are resident, and
// the pivot chain is a block barrier plus one shared-memory round trip.
//
// Pivot k lives in warp k/8, register k%8: the 8 pivots of a row block are unrolled
// (compile-time registers) inside a runtime loop over the 4 blocks, so the code stays
// small.  Look-ahead: during pivot k the owner of row k+1 applies pivot k to that
// row first, publishes it (and the reciprocal of its diagonal) into the other half of
// a double-buffered slot; one __syncthreads per pivot separates the buffers' reads
// and writes.  The owner recomputes the same row again in the common update loop
// (bit-identical operands), which keeps the loop free of warp-dependent skips.
#pragma once

namespace dpk {

constexpr int SMW_R = 8;      // rows per warp
constexpr int SMW_THREADS = 128;

__host__ __device__ inline int smw_smem_elems(int K, int KC) {   // complex elements of dynamic smem
  return npacked(32) + K * 32 + 4 * KC * 32;
}

template <int KC>
__global__ void __launch_bounds__(SMW_THREADS, 9) solve_mw_kernel(Args a) {   // 9 CTAs/SM: 1200 problems in one wave
  constexpr int U = 32, R = SMW_R;
  constexpr int NP = npacked(U);
  extern __shared__ __align__(16) float2 smw[];
  float2 *Gs = smw;                 // packed G of the problem
  float2 *ss = Gs + NP;             // s_k of its subcarrier, [K][U]
  float2 *part = ss + a.K * U;      // whitening partials [4][KC][U]
  __shared__ __align__(16) float2 slot[2][U];
  __shared__ float pinv[2];
  __shared__ float eqs[U];
  __shared__ float red[2][4];
  __shared__ int bad;
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const int p = blockIdx.x;
  const int sc = p / a.groups;
  if (tid == 0) bad = 0;
  pdl_wait();
  for (int i = tid; i < NP / 2; i += SMW_THREADS) cp_async16(Gs + 2 * i, a.G + (size_t)p * NP + 2 * i);
  if (!a.Wout)                                          // prepare calls have no symbols
    for (int i = tid; i < a.K * U / 2; i += SMW_THREADS) cp_async16(ss + 2 * i, a.s + (size_t)sc * a.K * U + 2 * i);
  cp_async_wait_all();
  __syncthreads();

  // column l of A = G + kappa I, rows R w .. R w + R-1 (Hermitian: lower part mirrored)
  float2 c[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int u = R * w + r;
    float2 g = (u <= l) ? Gs[pidx(U, u, l)] : cconj(Gs[pidx(U, l, u)]);
    if (u == l) g = make_float2(g.x + a.kappa, 0.f);
    c[r] = g;
  }
  // Jacobi equilibration A' = D^{-1/2} A D^{-1/2} (unit diagonal)
  if ((l >> 3) == w) {
    float dl = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (R * w + r == l) dl = c[r].x;
    const bool g = (dl > 0.f) && (dl < INFINITY);
    if (!g) bad = 1;
    eqs[l] = g ? rsqrtf(dl) : 1.f;
  }
  __syncthreads();
  const float rl = eqs[l];
#pragma unroll
  for (int r = 0; r < R; ++r) c[r] = cscale(c[r], rl * eqs[R * w + r]);
  // publish pivot row 0 and its reciprocal
  if (w == 0) {
    slot[0][l] = c[0];
    if (l == 0) {
      const float d0 = c[0].x;
      const bool g = (d0 > 0.f) && (d0 < INFINITY);
      if (!g) bad = 1;
      pinv[0] = __fdividef(1.f, g ? d0 : 1.f);
    }
  }
  __syncthreads();

  // ---- sweep: after pivot k, c holds the columns of the partially swept matrix
#pragma unroll 1
  for (int kb = 0; kb < U / R; ++kb) {
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int k = R * kb + j;
      const float2 *cur = slot[j & 1];          // R even: parity of k = parity of j
      float2 *nxt = slot[(j + 1) & 1];
      const float id = pinv[j & 1];
      const float2 akl = cur[l];                 // a_kl (row k of column l)
      const bool piv = (l == k);
      // non-pivot columns: a_il -= a_ik a_kl / a_kk ; pivot column: a_ik -> a_ik / a_kk
      const float2 sig = piv ? make_float2(1.f - id, 0.f) : cscale(akl, id);
      const int jn = (j + 1) % R;                // register of row k+1 in its owner warp
      const int wn = (j + 1 < R) ? kb : kb + 1;  // owner warp of row k+1
      if (k + 1 < U && w == wn) {
        float2 t = c[jn];
        cfms_cj(t, cur[R * w + jn], sig);
        nxt[l] = t;
        if (l == k + 1) {
          const bool g = (t.x > 0.f) && (t.x < INFINITY);
          if (!g) bad = 1;
          pinv[(j + 1) & 1] = __fdividef(1.f, g ? t.x : 1.f);
        }
      }
#pragma unroll
      for (int r = 0; r < R; r += 2) {
        const float4 sv = *reinterpret_cast<const float4 *>(cur + R * w + r);
        cfms_cj(c[r], lo2(sv), sig);
        cfms_cj(c[r + 1], hi2(sv), sig);
      }
      if (w == kb) c[j] = piv ? make_float2(-id, 0.f) : cscale(akl, id);   // row k
      __syncthreads();
    }
  }
  // ---- undo the equilibration: A^{-1} = D^{-1/2} A'^{-1} D^{-1/2};  c = column l of -A^{-1}
  float tr = 0.f, f = 0.f;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    c[r] = cscale(c[r], rl * eqs[R * w + r]);
    f += cabs2(c[r]);
    if (R * w + r == l) tr = -c[r].x;
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    tr += __shfl_xor_sync(0xffffffffu, tr, m);
    f += __shfl_xor_sync(0xffffffffu, f, m);
  }
  if (l == 0) { red[0][w] = tr; red[1][w] = f; }
  __syncthreads();
  tr = (red[0][0] + red[0][1]) + (red[0][2] + red[0][3]);
  f = (red[1][0] + red[1][1]) + (red[1][2] + red[1][3]);
  // Lemma 1, Eq. (6):  beta^2 = Es/rho^2 (tr A^{-1} - kappa ||A^{-1}||_F^2)
  const float rad = a.coef * (tr - a.kappa * f);
  const bool ok = (bad == 0) && (rad > 0.f) && (rad < INFINITY);
  const float beta = ok ? sqrtf(rad) : 1.f;
  const float ib = ok ? -__fdividef(1.f, beta) : 0.f;   // -: c holds -A^{-1}; failed problems: z = 0
  if (a.Wout) {                                         // prepare: cache W = A^{-1} / beta (upper, packed)
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (R * w + r <= l) a.Wout[(size_t)p * NP + pidx(U, R * w + r, l)] = cscale(c[r], ib);
    if (tid == 0) {
      a.beta[p] = ok ? beta : qnan();
      if (!ok) atomicAdd(a.bad, 1);
    }
    pdl_trigger();
    return;
  }

  // ---- whitening z_k[l] = (1/beta) sum_v A^{-1}[l][v] s_k[v], A^{-1}[l][v] = conj(A^{-1}[v][l])
  float2 *zo = a.zout + (size_t)p * a.K * U;
  for (int k0 = 0; k0 < a.K; k0 += KC) {
    float2 acc[KC];
#pragma unroll
    for (int j = 0; j < KC; ++j) {
      acc[j] = make_float2(0.f, 0.f);
      const float2 *sk = ss + (size_t)min(k0 + j, a.K - 1) * U + R * w;
#pragma unroll
      for (int r = 0; r < R; r += 2) {
        const float4 sv = *reinterpret_cast<const float4 *>(sk + r);
        cfma_cj(acc[j], c[r], lo2(sv));
        cfma_cj(acc[j], c[r + 1], hi2(sv));
      }
    }
#pragma unroll
    for (int j = 0; j < KC; ++j) part[(w * KC + j) * U + l] = acc[j];
    __syncthreads();
    for (int i = tid; i < KC * U; i += SMW_THREADS) {
      const int j = i / U, u = i % U;
      if (k0 + j < a.K) {
        const float2 s0 = part[(0 * KC + j) * U + u], s1 = part[(1 * KC + j) * U + u];
        const float2 s2 = part[(2 * KC + j) * U + u], s3 = part[(3 * KC + j) * U + u];
        const float zr = ((s0.x + s1.x) + (s2.x + s3.x)) * ib, zi = ((s0.y + s1.y) + (s2.y + s3.y)) * ib;
        zo[(size_t)(k0 + j) * U + u] = make_float2(zr, zi);
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    a.beta[p] = ok ? beta : qnan();
    if (!ok) atomicAdd(a.bad, 1);
  }
  pdl_trigger();
}

}  // namespace dpk
