// k_solve.cu — launchers of the whitening node: kernel (b) (regularise, equilibrated Hermitian
// sweep = LDL^H elimination fused with its substitutions P:285-286, Lemma-1 beta Eq. 6,
// z = A^{-1} s / beta P:174-177, or W = A^{-1}/beta for a prepare call) and the apply-time
// whitening z = W s.  U = 32 uses the multi-warp solve (solve_mw.cuh).
#include "dp_internal.cuh"
#include "solve_mw.cuh"

namespace dpi {

template <int U, int KC>
int launch_solve(dp_ctx *c, const Args &a, cudaStream_t st) {
  const int nprob = a.n_sc * a.groups;
  if constexpr (U == 32) {
    static const bool sg_only = getenv("DP_SOLVE_SG") != nullptr;   // A/B: one warp per problem
    static const int nw_env = getenv("DP_SOLVE_NW") ? atoi(getenv("DP_SOLVE_NW")) : 4;
    static const bool blk = getenv("DP_SOLVE_BLK") && atoi(getenv("DP_SOLVE_BLK")) == 1;   // A/B: 1 = blocked sweep
    if (!sg_only) {                                                  // 4 (or 2) warps per problem (solve_mw.cuh)
      const int NW = nw_env == 2 ? 2 : 4;
      // whitening in symbol chunks of at most 8: at 9 CTAs / SM (56 registers) 14 or 16
      // accumulators spilled
      constexpr int KS = KC > 8 ? KC / 2 : KC;
      const size_t sm = (size_t)dpk::smw_smem_elems(a.K, KS, NW) * sizeof(float2);
      auto kern = NW == 4 ? (blk ? dpk::solve_mw_kernel<KS, 4, true> : dpk::solve_mw_kernel<KS, 4, false>)
                          : dpk::solve_mw_kernel<KS, 2>;
      CK(set_smem(kern, sm));
      LaunchScope ls(c, DP_KERNEL_SOLVE, st);
      CK(launch_pdl(kern, dim3((nprob + 4 / NW - 1) / (4 / NW)), dim3(dpk::SMW_THREADS), sm, st, a));
      return DP_OK;
    }
  }
  // few problems (PD: one per subcarrier): one warp per CTA spreads the ~9k-instruction
  // warps evenly over the SMs (4-warp CTAs left some SMs with 50% more work)
  static const int wpc_env = getenv("DP_SOLVE_WPC") ? atoi(getenv("DP_SOLVE_WPC")) : 0;   // A/B: warps per CTA
  const int wpc = (wpc_env == 1 || wpc_env == 2 || wpc_env == 4) ? wpc_env
                  : (nprob / (32 / U) <= 16 * c->num_sms) ? 1 : 4;
  const int per = wpc * (32 / U);
  const size_t sm = smem_solve(U, a.K) / 4 * wpc;
  auto kern = dpk::solve_kernel<U, KC>;
  CK(set_smem(kern, sm));
  LaunchScope ls(c, DP_KERNEL_SOLVE, st);
  CK(launch_pdl(kern, dim3((nprob + per - 1) / per), dim3(32 * wpc), sm, st, a));
  return DP_OK;
}
template <int U, int KC> struct Solve {
  static int run(dp_ctx *c, const Args &a, cudaStream_t st) { return launch_solve<U, KC>(c, a, st); }
};
int launch_solve_any(dp_ctx *c, const Args &a, cudaStream_t st) { return dispatch<Solve>(c->cfg.U, a.K, c, a, st); }

template <int U, int KC>
int launch_whiten(dp_ctx *c, const Args &a, cudaStream_t st) {
  const int nprob = a.n_sc * a.groups;
  const int per = 4 * (32 / U);
  const size_t sm = (size_t)per * (dpk::npacked(U) + a.K * U + U * dpk::ZL<KC>::zs(a.K)) * sizeof(float2);
  auto kern = dpk::whiten_kernel<U, KC>;
  CK(set_smem(kern, sm));
  LaunchScope ls(c, DP_KERNEL_SOLVE, st);
  CK(launch_pdl(kern, dim3((nprob + per - 1) / per), dim3(128), sm, st, a));
  return DP_OK;
}
template <int U, int KC> struct Whiten {
  static int run(dp_ctx *c, const Args &a, cudaStream_t st) { return launch_whiten<U, KC>(c, a, st); }
};
int launch_whiten_any(dp_ctx *c, const Args &a, cudaStream_t st) { return dispatch<Whiten>(c->cfg.U, a.K, c, a, st); }

}  // namespace dpi
