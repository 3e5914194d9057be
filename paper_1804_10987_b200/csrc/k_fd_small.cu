// k_fd_small.cu — launcher of the FD small-cluster branch B_c = S < U (fd_small.cuh).
#include "dp_internal.cuh"
#include "fd_small.cuh"

namespace dpi {

template <int S, int U, int KC>
int launch_fd_small_t(dp_ctx *c, const Args &a, cudaStream_t st) {
  const size_t per = (size_t)(32 / S) * dpk::fds_size<S, U, KC>(a.K) * sizeof(float2);   // one warp's SGs
  int nw = 4;                                            // warps per CTA: fewer when the tiles do not fit
  while (nw > 1 && nw * per > 160 * 1024) nw >>= 1;
  const size_t sm = nw * per;
  if (sm > 227 * 1024) return fail(DP_ERR_UNSUPPORTED, "FD small-cluster tiles need %zu B of shared memory", sm);
  auto kern = dpk::fd_small_kernel<S, U, KC>;
  CK(set_smem(kern, sm));
  const int nprob = a.n_sc * a.nchunks, NSG = nw * (32 / S);
  LaunchScope ls(c, DP_KERNEL_FUSED_FD, st);
  CK(launch_pdl(kern, dim3((nprob + NSG - 1) / NSG), dim3(32 * nw), sm, st, a));
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
// sub-group size: the power of two >= B_c (lanes >= B_c pad, fd_small.cuh)
int launch_fd_small(dp_ctx *c, const Args &a, cudaStream_t st) {
  const int S = a.S, U = c->cfg.U;
  if (S < 1 || S >= U) return fail(DP_ERR_UNSUPPORTED, "FD small-cluster branch: B_c=%d, U=%d (need 1 <= B_c < U)", S, U);
  const int SP = S <= 4 ? 4 : S <= 8 ? 8 : S <= 16 ? 16 : 32;
  switch (U) {
    case 4: return launch_fd_small_kc<4, 4>(c, a, st);
    case 8: return SP == 4 ? launch_fd_small_kc<4, 8>(c, a, st) : launch_fd_small_kc<8, 8>(c, a, st);
    case 16:
      return SP == 4 ? launch_fd_small_kc<4, 16>(c, a, st) : SP == 8 ? launch_fd_small_kc<8, 16>(c, a, st)
                                                              : launch_fd_small_kc<16, 16>(c, a, st);
    case 32:
      return SP == 4 ? launch_fd_small_kc<4, 32>(c, a, st) : SP == 8 ? launch_fd_small_kc<8, 32>(c, a, st)
             : SP == 16 ? launch_fd_small_kc<16, 32>(c, a, st) : launch_fd_small_kc<32, 32>(c, a, st);
  }
  return fail(DP_ERR_UNSUPPORTED, "FD small-cluster branch: U=%d", U);
}

}  // namespace dpi
