// k_fd.cu — launchers of the SIMT FD-WF single pass (fd_fused_kernel, kernels.cuh; Sec. III-C,
// P:210-234), the fully-distributed MRT baseline (mrt_kernel, Fig. 2) and the per-subcarrier
// scalar kernels (fd_finish_kernel, fd_var_finish_kernel, read_scalars_kernel).
#include "dp_internal.cuh"

namespace dpi {

// Sub-groups per problem of fd_fused_kernel: replicate while the grid would have fewer than two
// waves of warps (12 resident per SM), every lane keeps at least two precode rows (the replicas
// repeat the sweep and the whitening, which must stay the smaller part: cfg2 FD with 16 rows was
// 18.9 -> 23.7 us at R = 2, fig2a FD with 128 rows 53.7 -> 44.2 us, cfg2 PD single pass with 64 rows
// 19.0 -> 16.9 us at R = 4), and the replicas fit in one warp (DP_FD_REP=<R> forces R for A/B runs).
int fd_rep(const dp_ctx *c, const Args &a, int nw) {
  const int U = c->cfg.U, PPW = 32 / U;
  static const int env = getenv("DP_FD_REP") ? atoi(getenv("DP_FD_REP")) : 0;
  const long long nprob = (long long)a.n_sc * a.nchunks, target = 2LL * 12 * c->num_sms;
  auto fits = [&](int R) { return R <= PPW && (nw * PPW) % R == 0 && a.S % R == 0 && a.S >= 2 * R * U; };
  if (env > 0) return fits(env) ? env : 1;
  int R = 1;
  while (fits(2 * R) && nprob * 2 * R * U / 32 <= target) R *= 2;
  return R;
}

template <int U, int KC>
int launch_fd_fused(dp_ctx *c, const Args &a, cudaStream_t st, int nw_, int kid) {
  const int nw = nw_ > 0 ? nw_ : c->fd_nw;
  Args b = a;
  b.rep = fd_rep(c, a, nw);
  const int npb = nw * (32 / U) / b.rep;                  // problems per CTA
  const int nprob = a.n_sc * a.nchunks;
  static const size_t pad = getenv("DP_FD_SMEM_PAD") ? (size_t)atoi(getenv("DP_FD_SMEM_PAD")) : 0;   // occupancy experiments
  const size_t sm = smem_fd_fused(U, a.S, a.K, nw, b.rep) + pad;
  auto kern = dpk::fd_fused_kernel<U, KC>;
  CK(set_smem(kern, sm));
  LaunchScope ls(c, kid, st);
  CK(launch_pdl(kern, dim3((nprob + npb - 1) / npb), dim3(nw * 32), sm, st, b));
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
  Args b = a;                                              // b.rep = lanes per subcarrier (fd_finish_kernel)
  const int mx = std::max(a.nbeta, a.nchunks);
  b.rep = 1;
  while (b.rep < mx) b.rep *= 2;
  if (b.rep > 32) b.rep = 0;                               // many small clusters: thread per subcarrier
  const long long nt = (long long)a.n_sc * (b.rep ? b.rep : 1);
  CK(launch_pdl(dpk::fd_finish_kernel, dim3((unsigned)((nt + 127) / 128)), dim3(128), 0, st, b));
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
