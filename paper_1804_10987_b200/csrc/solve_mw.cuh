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
// Here lane l of warp w holds column l, rows (32/NW) w .. : with NW = 2 a pivot costs
// each warp 16 row updates instead of 32, twice as many warps are resident, and the
// pivot chain is a 64-thread named barrier plus one shared-memory round trip (NW = 4
// halves the rows again but doubles the per-pivot overhead instructions).
//
// Pivot k lives in warp k/R, register k%R: the R pivots of a row block are unrolled
// (compile-time registers) inside a runtime loop over the NW blocks, so the code stays
// small.  Look-ahead: during pivot k the owner of row k+1 applies pivot k to that
// row first, publishes it (and the reciprocal of its diagonal) into the other half of
// a double-buffered slot; one __syncthreads per pivot separates the buffers' reads
// and writes.  The owner recomputes the same row again in the common update loop
// (bit-identical operands), which keeps the loop free of warp-dependent skips.
#pragma once

namespace dpk {

constexpr int SMW_THREADS = 128;

// complex elements of dynamic smem per CTA (4 / NW problems)
__host__ __device__ inline int smw_smem_elems(int K, int KC, int NW) {
  return (4 / NW) * (npacked(32) + K * 32 + NW * KC * 32);
}

// The solve of one problem by NW warps (rows 32/NW per warp, lane l = column l), shared by
// solve_mw_kernel and the fused PD Gram+solve epilogue (gram_tc2.cuh).  On entry c holds
// column l, rows R w .. R w + R-1, of A = G + kappa I; `bad` is 0 and visible; `psync`
// synchronises the NW warps of the problem; ss holds s_k of the problem's subcarrier
// ([K][U], unless a.Wout) and `part` has NW KC U complex of scratch.  Writes z (or W for
// a prepare call) and beta of problem p.
// Blocked form of the same sweep (NW = 4, R = 8 rows per warp, lane l = column l): the pivots are
// taken in 4 blocks B = [8kb, 8kb + 8) (the sweep of a block is the composition of its 8 scalar
// sweeps, so the arithmetic is the scalar sweep's, regrouped):
//   A_BB <- -A_BB^{-1},  A_BR <- A_BB^{-1} A_BR,  A_RB <- A_RB A_BB^{-1},  A_RR <- A_RR - A_RB A_BB^{-1} A_BR.
// Phase A (warp kb, which owns rows B): the 8 scalar pivots of the block applied to rows B of every
//   column (one-pivot look-ahead, __syncwarp only) -> y_l = new rows B of column l, published.
// Phase B (the other warps): new A_il = sigma_l A_il - sum_{b in B} A_ib y_l[b]  (sigma_l = 0 for
//   l in B, whose y_l is -A_BB^{-1} e_l), with the old A_iB of the warp's rows staged in shared
//   memory by its lanes l in B: 8 complex MACs per row, no per-pivot barrier.
// One CTA barrier per block (4 per problem instead of 32) and ~40% of the instructions of the
// row-split scalar loop below.  ybuf: 2 x [4][32][2] complex; stage: this warp's [8][8] complex.
template <typename Sync>
__device__ __forceinline__ void mw_sweep_blk(float2 (&c)[8], int w, int l, float2 (*slot)[32], float2 *ybuf,
                                             float2 *stage, int &bad, Sync psync) {
#pragma unroll 1
  for (int kb = 0; kb < 4; ++kb) {
    const int b0 = 8 * kb;
    const bool inB = (unsigned)(l - b0) < 8u;
    float2 *yb = ybuf + (kb & 1) * 256;
    if (w == kb) {
      if (inB) slot[0][l - b0] = c[0];                       // pivot row b0 at the columns of B
      __syncwarp();
      float id;
      {
        const float d0 = slot[0][0].x;
        const bool g = (d0 > 0.f) && (d0 < INFINITY);
        if (!g) bad = 1;
        id = __fdividef(1.f, g ? d0 : 1.f);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float2 *cur = slot[j & 1];                     // cur[r] = a_{b0+j, b0+r}
        float2 *nxt = slot[(j + 1) & 1];
        const bool piv = (l == b0 + j);
        const float2 sig = piv ? make_float2(1.f - id, 0.f) : cscale(c[j], id);
        float idn = 1.f;
        if (j + 1 < 8) {                                     // look-ahead: row b0+j+1 first
          cfms_cj(c[j + 1], cur[j + 1], sig);
          if (inB) nxt[l - b0] = c[j + 1];
          __syncwarp();
          const float dn = nxt[j + 1].x;
          const bool g = (dn > 0.f) && (dn < INFINITY);
          if (!g) bad = 1;
          idn = __fdividef(1.f, g ? dn : 1.f);
        }
#pragma unroll
        for (int r = 0; r < 8; ++r)
          if (r != j && r != j + 1) cfms_cj(c[r], cur[r], sig);
        c[j] = piv ? make_float2(-id, 0.f) : cscale(c[j], id);
        id = idn;
        __syncwarp();
      }
      float4 *yo = reinterpret_cast<float4 *>(yb);
#pragma unroll
      for (int q = 0; q < 4; ++q) yo[q * 32 + l] = make_float4(c[2 * q].x, c[2 * q].y, c[2 * q + 1].x, c[2 * q + 1].y);
    } else if (inB) {                                        // old A_iB of this warp's rows
#pragma unroll
      for (int r = 0; r < 8; ++r) stage[r * 8 + (l - b0)] = c[r];   // [row r][b - b0]
    }
    psync();
    if (w != kb) {
      float2 y[8];
      const float4 *yi = reinterpret_cast<const float4 *>(yb);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 v = yi[q * 32 + l];
        y[2 * q] = lo2(v);
        y[2 * q + 1] = hi2(v);
      }
      const float sgm = inB ? 0.f : 1.f;
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        float2 t = cscale(c[r], sgm);
        const float4 *sr = reinterpret_cast<const float4 *>(stage + 8 * r);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 v = sr[q];
          cfms(t, lo2(v), y[2 * q]);
          cfms(t, hi2(v), y[2 * q + 1]);
        }
        c[r] = t;
      }
      __syncwarp();                                          // stage reads done before the next block's writes
    }
  }
}

template <int KC, int NW, typename Sync, bool BLK = false>
__device__ __forceinline__ void mw_solve(const Args &a, float2 (&c)[32 / NW], int w, int l, int pt, int p,
                                         bool active, float2 (*slot)[32], float *pinv, float *eqs,
                                         float (*red)[NW], int &bad, const float2 *ss, float2 *part, Sync psync,
                                         float2 *ybuf = nullptr, float2 *stage = nullptr) {
  constexpr int U = 32, R = U / NW;
  constexpr int NP = npacked(U);
  // Jacobi equilibration A' = D^{-1/2} A D^{-1/2} (unit diagonal)
  if (l / R == w) {
    float dl = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (R * w + r == l) dl = c[r].x;
    const bool g = (dl > 0.f) && (dl < INFINITY);
    if (!g) bad = 1;
    eqs[l] = g ? rsqrtf(dl) : 1.f;
  }
  psync();
  const float rl = eqs[l];
#pragma unroll
  for (int r = 0; r < R; ++r) c[r] = cscale(c[r], rl * eqs[R * w + r]);
  if constexpr (BLK) {
    static_assert(NW == 4, "blocked sweep: 4 warps x 8 rows");
    mw_sweep_blk(c, w, l, slot, ybuf, stage + 64 * w, bad, psync);
  } else {
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
  psync();

  // ---- sweep: after pivot k, c holds the columns of the partially swept matrix
#pragma unroll 1
  for (int kb = 0; kb < NW; ++kb) {
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
      psync();
    }
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
  psync();
  tr = 0.f;
  f = 0.f;
#pragma unroll
  for (int i = 0; i < NW; ++i) { tr += red[0][i]; f += red[1][i]; }
  // Lemma 1, Eq. (6):  beta^2 = Es/rho^2 (tr A^{-1} - kappa ||A^{-1}||_F^2)
  const float rad = a.coef * (tr - a.kappa * f);
  const bool ok = (bad == 0) && (rad > 0.f) && (rad < INFINITY);
  const float beta = ok ? sqrtf(rad) : 1.f;
  const float ib = ok ? -__fdividef(1.f, beta) : 0.f;   // -: c holds -A^{-1}; failed problems: z = 0
  if (a.Wout) {                                         // prepare: cache W = A^{-1} / beta (upper, packed)
    if (active) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (R * w + r <= l) a.Wout[(size_t)p * NP + pidx(U, R * w + r, l)] = cscale(c[r], ib);
      if (pt == 0) {
        a.beta[p] = ok ? beta : qnan();
        if (!ok) atomicAdd(a.bad, 1);
      }
    }
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
    psync();
    for (int i = pt; i < KC * U; i += NW * 32) {
      const int j = i / U, u = i % U;
      if (active && k0 + j < a.K) {
        float zr = 0.f, zi = 0.f;
#pragma unroll
        for (int ww = 0; ww < NW; ++ww) {
          const float2 v = part[(ww * KC + j) * U + u];
          zr += v.x;
          zi += v.y;
        }
        zo[(size_t)(k0 + j) * U + u] = make_float2(zr * ib, zi * ib);
      }
    }
    psync();
  }
  if (active && pt == 0) {
    a.beta[p] = ok ? beta : qnan();
    if (!ok) atomicAdd(a.bad, 1);
  }
}

// NW warps per problem (rows 32/NW per warp), 4/NW problems per 128-thread CTA; the
// warps of one problem synchronise on their own named barrier (id 1 + problem in CTA).
template <int KC, int NW, bool BLK = false>
__global__ void __launch_bounds__(SMW_THREADS, NW == 4 ? 9 : 5) solve_mw_kernel(Args a) {
  pdl_trigger();   // early: the next kernel may launch once every CTA of this grid has started
                   // (it still waits for this grid's completion in griddepcontrol.wait)   // 1200 problems in one wave
  constexpr int U = 32, R = U / NW, PPC = 4 / NW;
  constexpr int NP = npacked(U);
  extern __shared__ __align__(16) float2 smw[];
  __shared__ __align__(16) float2 slot_[PPC][2][U];
  __shared__ float pinv_[PPC][2];
  __shared__ float eqs_[PPC][U];
  __shared__ float red_[PPC][2][NW];
  __shared__ int bad_[PPC];
  __shared__ __align__(16) float2 ybuf_[BLK ? 512 : 1], stage_[BLK ? 256 : 1];   // blocked sweep (NW = 4)
  const int tid = threadIdx.x, l = tid & 31;
  const int q = (tid >> 5) / NW, w = (tid >> 5) % NW;       // problem in CTA, warp within problem
  const int pt = tid - q * NW * 32;                         // thread index within the problem
  const int nprob = a.n_sc * a.groups;
  const int pr = blockIdx.x * PPC + q;
  const bool active = pr < nprob;
  const int p = active ? pr : nprob - 1;
  const int sc = p / a.groups;
  float2 *Gs = smw + (size_t)q * (NP + a.K * U + NW * KC * U);
  float2 *ss = Gs + NP;             // s_k of its subcarrier, [K][U]
  float2 *part = ss + a.K * U;      // whitening partials [NW][KC][U]
  int &bad = bad_[q];
  auto psync = [&]() {
    if (NW == 4) __syncthreads();
    else asm volatile("bar.sync %0, %1;" ::"r"(1 + q), "r"(NW * 32) : "memory");
  };
  if (pt == 0) bad = 0;
  // s is an input of the call (unless a collective on the stream produced it: a.s_wait), so it is
  // fetched before griddepcontrol.wait; G is the Gram kernel's output, fetched after it
  const bool s_early = !a.Wout && !a.s_wait;            // prepare calls have no symbols
  if (s_early)
    for (int i = pt; i < a.K * U / 2; i += NW * 32) cp_async16(ss + 2 * i, a.s + (size_t)sc * a.K * U + 2 * i);
  pdl_wait();
  for (int i = pt; i < NP / 2; i += NW * 32) cp_async16(Gs + 2 * i, a.G + (size_t)p * NP + 2 * i);
  if (!a.Wout && !s_early)
    for (int i = pt; i < a.K * U / 2; i += NW * 32) cp_async16(ss + 2 * i, a.s + (size_t)sc * a.K * U + 2 * i);
  cp_async_wait_all();
  psync();
  // column l of A = G + kappa I, rows R w .. R w + R-1 (Hermitian: lower part mirrored)
  float2 c[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int u = R * w + r;
    float2 g = (u <= l) ? Gs[pidx(U, u, l)] : cconj(Gs[pidx(U, l, u)]);
    if (u == l) g = make_float2(g.x + a.kappa, 0.f);
    c[r] = g;
  }
  mw_solve<KC, NW, decltype(psync), BLK>(a, c, w, l, pt, p, active, slot_[q], pinv_[q], eqs_[q], red_[q], bad, ss,
                                          part, psync, ybuf_, stage_);
  pdl_trigger();
}

}  // namespace dpk
