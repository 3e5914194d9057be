// k_fd_small.cu — launcher of the FD small-cluster branch B_c = S < U (fd_small.cuh).
#include "dp_internal.cuh"
#include "fd_small.cuh"

namespace dpi {

template <int S, int U, int KC>
int launch_fd_small_t(dp_ctx *c, const Args &a, cudaStream_t st) {
  constexpr int NSG = 4 * (32 / S);                      // 4 warps per CTA
  const size_t sm = (size_t)NSG * dpk::fds_size<S, U, KC>(a.K) * sizeof(float2);
  if (sm > 227 * 1024) return fail(DP_ERR_UNSUPPORTED, "FD small-cluster tiles need %zu B of shared memory", sm);
  auto kern = dpk::fd_small_kernel<S, U, KC>;
  CK(set_smem(kern, sm));
  const int nprob = a.n_sc * a.nchunks;
  LaunchScope ls(c, DP_KERNEL_FUSED_FD, st);
  CK(launch_pdl(kern, dim3((nprob + NSG - 1) / NSG), dim3(128), sm, st, a));
  return DP_OK;
}
template <int S, int U>
int launch_fd_small_kc(dp_ctx *c, const Args &a, cudaStream_t st) {
  switch (kc_of(a.K)) {
    case 7: return launch_fd_small_t<S, U, 7>(c, a, st);
    case 8: return launch_fd_small_t<S, U, 8>(c, a, st);
    case 14: return launch_fd_small_t<S, U, 14>(c, a, st);
    default: return launch_fd_small_t<S, U, 16>(c, a, st);
  }
}
int launch_fd_small(dp_ctx *c, const Args &a, cudaStream_t st) {
  const int S = a.S, U = c->cfg.U;
  if (S == 4 && U == 8) return launch_fd_small_kc<4, 8>(c, a, st);
  if (S == 4 && U == 16) return launch_fd_small_kc<4, 16>(c, a, st);
  if (S == 4 && U == 32) return launch_fd_small_kc<4, 32>(c, a, st);
  if (S == 8 && U == 16) return launch_fd_small_kc<8, 16>(c, a, st);
  if (S == 8 && U == 32) return launch_fd_small_kc<8, 32>(c, a, st);
  if (S == 16 && U == 32) return launch_fd_small_kc<16, 32>(c, a, st);
  return fail(DP_ERR_UNSUPPORTED, "FD small-cluster branch: B_c=%d, U=%d (need B_c in {4, 8, 16} < U)", S, U);
}

}  // namespace dpi
