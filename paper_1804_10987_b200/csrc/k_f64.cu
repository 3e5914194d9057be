// k_f64.cu — launchers of the DP_FLAG_FP64 kernels (f64.cuh): FD per cluster (B_c >= U) and the PD
// Gram -> [cross-rank sum] -> whitening node -> precode chain with fp64 accumulation.
#include "dp_internal.cuh"
#include "f64.cuh"

namespace dpi {

template <int U>
int launch_fd_f64_t(dp_ctx *c, const Args &a, cudaStream_t st) {
  constexpr int PPW = 32 / U;
  const size_t per = dpk::f64_sg_bytes(a.S, U, a.K);
  int nw = 4;
  while (nw > 1 && (size_t)nw * PPW * per > 110 * 1024) nw >>= 1;
  const size_t sm = (size_t)nw * PPW * per;
  if (sm > 227 * 1024) return fail(DP_ERR_UNSUPPORTED, "DP_FLAG_FP64: cluster tile B_c=%d x U=%d needs %zu B", a.S, U, sm);
  auto kern = dpk::fd_f64_kernel<U>;
  CK(set_smem(kern, sm));
  const int nsg = nw * PPW, nprob = a.n_sc * a.nchunks;
  LaunchScope ls(c, DP_KERNEL_FUSED_FD, st);
  CK(launch_pdl(kern, dim3((nprob + nsg - 1) / nsg), dim3(32 * nw), sm, st, a));
  return DP_OK;
}
int launch_fd_f64(dp_ctx *c, const Args &a, cudaStream_t st) {
  switch (c->cfg.U) {
    case 4: return launch_fd_f64_t<4>(c, a, st);
    case 8: return launch_fd_f64_t<8>(c, a, st);
    case 16: return launch_fd_f64_t<16>(c, a, st);
    case 32: return launch_fd_f64_t<32>(c, a, st);
  }
  return fail(DP_ERR_UNSUPPORTED, "U=%d", c->cfg.U);
}

template <int U>
int launch_gram_f64_t(dp_ctx *c, const Args &a, double2 *G64, cudaStream_t st) {
  const size_t sm = (size_t)a.Bl * U * 8;
  if (sm > 227 * 1024) return fail(DP_ERR_UNSUPPORTED, "DP_FLAG_FP64: Gram tile of %d antennas", a.Bl);
  auto kern = dpk::gram_f64_kernel<U>;
  CK(set_smem(kern, sm));
  LaunchScope ls(c, DP_KERNEL_GRAM, st);
  CK(launch_pdl(kern, dim3(a.n_sc), dim3(128), sm, st, a, G64));
  return DP_OK;
}
int launch_gram_f64(dp_ctx *c, const Args &a, double2 *G64, cudaStream_t st) {
  switch (c->cfg.U) {
    case 4: return launch_gram_f64_t<4>(c, a, G64, st);
    case 8: return launch_gram_f64_t<8>(c, a, G64, st);
    case 16: return launch_gram_f64_t<16>(c, a, G64, st);
    case 32: return launch_gram_f64_t<32>(c, a, G64, st);
  }
  return fail(DP_ERR_UNSUPPORTED, "U=%d", c->cfg.U);
}

template <int U>
int launch_solve_f64_t(dp_ctx *c, const Args &a, const double2 *G64, double2 *z64, cudaStream_t st) {
  constexpr int NSG = 4 * (32 / U);
  const size_t sm = (size_t)NSG * ((size_t)a.K * U * 8 + U * 16);
  auto kern = dpk::solve_f64_kernel<U>;
  CK(set_smem(kern, sm));
  LaunchScope ls(c, DP_KERNEL_SOLVE, st);
  CK(launch_pdl(kern, dim3((a.n_sc + NSG - 1) / NSG), dim3(128), sm, st, a, G64, z64));
  return DP_OK;
}
int launch_solve_f64(dp_ctx *c, const Args &a, const double2 *G64, double2 *z64, cudaStream_t st) {
  switch (c->cfg.U) {
    case 4: return launch_solve_f64_t<4>(c, a, G64, z64, st);
    case 8: return launch_solve_f64_t<8>(c, a, G64, z64, st);
    case 16: return launch_solve_f64_t<16>(c, a, G64, z64, st);
    case 32: return launch_solve_f64_t<32>(c, a, G64, z64, st);
  }
  return fail(DP_ERR_UNSUPPORTED, "U=%d", c->cfg.U);
}

template <int U>
int launch_precode_f64_t(dp_ctx *c, const Args &a, const double2 *z64, cudaStream_t st) {
  const size_t sm = (size_t)a.K * U * 16;
  auto kern = dpk::precode_f64_kernel<U>;
  CK(set_smem(kern, sm));
  LaunchScope ls(c, DP_KERNEL_PRECODE, st);
  CK(launch_pdl(kern, dim3(a.n_sc), dim3(128), sm, st, a, z64));
  return DP_OK;
}
int launch_precode_f64(dp_ctx *c, const Args &a, const double2 *z64, cudaStream_t st) {
  switch (c->cfg.U) {
    case 4: return launch_precode_f64_t<4>(c, a, z64, st);
    case 8: return launch_precode_f64_t<8>(c, a, z64, st);
    case 16: return launch_precode_f64_t<16>(c, a, z64, st);
    case 32: return launch_precode_f64_t<32>(c, a, z64, st);
  }
  return fail(DP_ERR_UNSUPPORTED, "U=%d", c->cfg.U);
}

}  // namespace dpi
