// exch_lsa.cuh — PD whitening node with the cross-GPU exchange fused in (DP_PD_NVLINK, U = 32).
//
// The PD adder tree G = sum_c G_c spans the clusters of all GPUs, and every GPU then
// needs the whitened symbols z of every subcarrier.  The paper and
// the other topologies of this library do that with collectives between kernels (reduce /
// allreduce / reduce-scatter of the packed Gram, broadcast / all-gather of z).  Here rank r
// owns the subcarrier block [r nb, (r+1) nb), nb = n_sc / world, and its solve kernel does the
// exchange itself over NVLink load/store, through NCCL 2.28's device API (symmetric windows
// registered with NCCL_WIN_COLL_SYMMETRIC, ncclGetLsaPointer, ncclLsaBarrierSession):
//
//   1. per-CTA cross-GPU barrier (CTA i of every rank): every rank's Gram kernel -- which wrote
//      that rank's partial packed Gram of ALL subcarriers into its window -- has completed;
//   2. the CTA's subcarrier Gram is summed straight from every peer's window in rank order
//      (the reduce-scatter, fused into the solve's loads; the same fixed order on every rank);
//   3. the solve (mw_solve: equilibrated Hermitian sweep, Lemma-1 beta, z = A^{-1} s / beta);
//   4. z and beta are stored into every peer's window (the all-gather, fused into the epilogue);
//   5. per-CTA barrier again: when this kernel has completed on a rank, CTA i of every peer has
//      finished its stores into this rank's window (for every i), so the precode that follows
//      on the stream sees all of z.  Frame t+1's Gram cannot overwrite a window a peer is still
//      reading: that peer passed barrier 5 only after this rank's loads of frame t.
//
// No data atomics and a fixed summation order: the result is bit-identical on every rank and
// across world sizes that produce the same partial Grams.
#pragma once
#include <nccl_device.h>

#include "solve_mw.cuh"

namespace dpk {

struct LsaArgs {
  ncclDevComm dc;
  ncclWindow_t wg, wz, wb;   // packed Gram [n_sc][NP], z [n_sc][K][U], beta [n_sc] windows
  int sc0;                   // this rank's first subcarrier
};

template <int KC>
__global__ void __launch_bounds__(SMW_THREADS, 9) solve_lsa_kernel(Args a, const __grid_constant__ LsaArgs x) {
  pdl_trigger();
  constexpr int U = 32, NW = 4, R = U / NW, NP = npacked(U);
  extern __shared__ __align__(16) float2 smw[];
  __shared__ __align__(16) float2 slot_[2][U];
  __shared__ float pinv_[2];
  __shared__ float eqs_[U];
  __shared__ float red_[2][NW];
  __shared__ int bad_;
  const int tid = threadIdx.x, l = tid & 31, w = tid >> 5;
  const int p = blockIdx.x;                                  // problem within this rank's block
  const int sc = x.sc0 + p;                                  // its subcarrier
  float2 *Gs = smw, *ss = Gs + NP, *part = ss + a.K * U;
  auto psync = [&]() { __syncthreads(); };
  if (tid == 0) bad_ = 0;
  ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), x.dc, ncclTeamTagLsa(), (uint32_t)blockIdx.x);
  pdl_wait();                                                // this rank's Gram (and s landing) complete
  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);       // ... and every peer's
  // s of the subcarrier (async) while the Gram is summed over the peers' windows, in rank order
  for (int i = tid; i < a.K * U / 2; i += SMW_THREADS) cp_async16(ss + 2 * i, a.s + (size_t)sc * a.K * U + 2 * i);
  const size_t goff = (size_t)sc * NP * sizeof(float2);
  for (int i = tid; i < NP / 2; i += SMW_THREADS) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int r = 0; r < x.dc.lsaSize; ++r) {
      const float4 v = *reinterpret_cast<const float4 *>(static_cast<const char *>(ncclGetLsaPointer(x.wg, goff, r)) +
                                                         16 * (size_t)i);
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    reinterpret_cast<float4 *>(Gs)[i] = acc;
  }
  cp_async_wait_all();
  psync();
  float2 c[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int u = R * w + r;
    float2 g = (u <= l) ? Gs[pidx(U, u, l)] : cconj(Gs[pidx(U, l, u)]);
    if (u == l) g = make_float2(g.x + a.kappa, 0.f);
    c[r] = g;
  }
  // a.zout / a.beta point at this rank's block inside its own windows (problem p <-> subcarrier sc)
  mw_solve<KC, NW>(a, c, w, l, tid, p, true, slot_, pinv_, eqs_, red_, bad_, ss, part, psync);
  __syncthreads();                                           // z, beta of subcarrier sc written (global)
  // all-gather: z and beta of this subcarrier into every other rank's windows
  const size_t zoff = (size_t)sc * a.K * U * sizeof(float2);
  const float4 *zl = reinterpret_cast<const float4 *>(a.zout + (size_t)p * a.K * U);
  for (int r = 0; r < x.dc.lsaSize; ++r) {
    if (r == x.dc.lsaRank) continue;
    float4 *zr = reinterpret_cast<float4 *>(ncclGetLsaPointer(x.wz, zoff, r));
    for (int i = tid; i < a.K * U / 2; i += SMW_THREADS) zr[i] = zl[i];
    if (tid == 0)
      *static_cast<float *>(ncclGetLsaPointer(x.wb, (size_t)sc * sizeof(float), r)) = __ldcg(a.beta + p);
  }
  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);       // every peer's stores into this window done
  pdl_trigger();
}

}  // namespace dpk
