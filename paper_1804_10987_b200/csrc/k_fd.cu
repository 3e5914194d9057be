// k_fd.cu — launchers of the SIMT FD-WF single pass (fd_fused_kernel, kernels.cuh; Sec. III-C,
// P:210-234), the fully-distributed MRT baseline (mrt_kernel, Fig. 2) and the per-subcarrier
// scalar kernels (fd_finish_kernel, fd_var_finish_kernel, read_scalars_kernel).
#include "dp_internal.cuh"

namespace dpi {

template <int U, int KC>
int launch_fd_fused(dp_ctx *c, const Args &a, cudaStream_t st, int nw_, int kid) {
  const int nw = nw_ > 0 ? nw_ : c->fd_nw;
  const int nsg = nw * (32 / U);
  const int nprob = a.n_sc * a.nchunks;
  static const size_t pad = getenv("DP_FD_SMEM_PAD") ? (size_t)atoi(getenv("DP_FD_SMEM_PAD")) : 0;   // occupancy experiments
  const size_t sm = smem_fd_fused(U, a.S, a.K, nw) + pad;
  auto kern = dpk::fd_fused_kernel<U, KC>;
  CK(set_smem(kern, sm));
  LaunchScope ls(c, kid, st);
  CK(launch_pdl(kern, dim3((nprob + nsg - 1) / nsg), dim3(nw * 32), sm, st, a));
  return DP_OK;
}
template <int U, int KC> struct FdFused {
  static int run(dp_ctx *c, const Args &a, cudaStream_t st, int nw, int kid) {
    return launch_fd_fused<U, KC>(c, a, st, nw, kid);
  }
};
int launch_fd_fused_any(dp_ctx *c, const Args &a, cudaStream_t st, int nw, int kid) {
  return dispatch<FdFused>(c->cfg.U, a.K, c, a, st, nw, kid);
}

template <int U>
int launch_mrt(dp_ctx *c, const Args &a, cudaStream_t st) {
  const size_t sm = (size_t)4 * a.K * U * sizeof(float2);
  auto kern = dpk::mrt_kernel<U>;
  CK(set_smem(kern, sm));
  LaunchScope ls(c, DP_KERNEL_FUSED_FD, st);
  CK(launch_pdl(kern, dim3((a.n_sc * a.nchunks + 3) / 4), dim3(128), sm, st, a));
  return DP_OK;
}
int launch_mrt_u(dp_ctx *c, const Args &a, cudaStream_t st) {
  switch (c->cfg.U) {
    case 4: return launch_mrt<4>(c, a, st);
    case 8: return launch_mrt<8>(c, a, st);
    case 16: return launch_mrt<16>(c, a, st);
    default: return launch_mrt<32>(c, a, st);
  }
}

int launch_fd_finish(dp_ctx *c, const Args &a, cudaStream_t st) {
  LaunchScope ls(c, DP_KERNEL_FINISH, st);
  CK(launch_pdl(dpk::fd_finish_kernel, dim3((a.n_sc + 127) / 128), dim3(128), 0, st, a));
  return DP_OK;
}

int launch_fd_var_finish(dp_ctx *c, const Args &a, const dpk::VarRuns &vr, cudaStream_t st) {
  LaunchScope ls(c, DP_KERNEL_FINISH, st);
  CK(launch_pdl(dpk::fd_var_finish_kernel, dim3((a.n_sc + 3) / 4), dim3(128), 0, st, a, vr));
  return DP_OK;
}

int launch_read_scalars(const float *fin, int n_sc, int which, float *dst, cudaStream_t st) {
  dpk::read_scalars_kernel<<<(n_sc + 127) / 128, 128, 0, st>>>(fin, n_sc, which, dst);
  CK(cudaGetLastError());
  return DP_OK;
}

}  // namespace dpi
