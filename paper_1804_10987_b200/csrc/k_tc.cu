// k_tc.cu — launchers of the tensor-core (tcgen05 / TMEM / TMA) kernels: the persistent PD Gram
// (gram_tc2.cuh), the persistent PD precode (precode_tc2.cuh) and the FD single pass at
// U = B_c = 32 (fd_tc.cuh), plus the TMA tensor maps over H they read.
#include "dp_internal.cuh"
#include "fd_tc.cuh"
#include "gram_tc2.cuh"
#include "precode_tc2.cuh"

namespace dpi {

// 2-D tensor map over H_local viewed as fp32 [rows][2U], box_rows-row x 32-float boxes with
// the given swizzle (SWIZZLE_128B: the canonical K-major SW128 UMMA layout; SWIZZLE_128B_ATOM_32B:
// the MN-major tf32 layout of the Gram operands).
static int encode_h_tmap(const float2 *H, int rows, CUtensorMap *tm, int box_rows, CUtensorMapSwizzle sw, int U) {
  static PFN_cuTensorMapEncodeTiled encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&encode, cudaEnableDefault, &q) != cudaSuccess ||
        !encode)
      return fail(DP_ERR_CUDA, "cuTensorMapEncodeTiled not available");
  }
  cuuint64_t dims[2] = {(cuuint64_t)(2 * U), (cuuint64_t)rows};   // fp32 [rows][2U]
  cuuint64_t strides[1] = {(cuuint64_t)(2 * U * 4)};
  cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)H, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DP_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return DP_OK;
}

// cached per context by (pointer, rows, box, swizzle, U): per-frame host overhead
static int make_h_tmap(dp_ctx *c, const float2 *H, int rows, CUtensorMap *tm, int box_rows, CUtensorMapSwizzle sw,
                       int U = 32) {
  const int key = (int)sw + 16 * U;
  for (const auto &e : c->tmaps)
    if (e.p == H && e.rows == rows && e.box == box_rows && e.sw == key) {
      *tm = e.tm;
      return DP_OK;
    }
  RET(encode_h_tmap(H, rows, tm, box_rows, sw, U));
  if (c->tmaps.size() >= 16) c->tmaps.erase(c->tmaps.begin());
  c->tmaps.push_back({H, rows, box_rows, key, *tm});
  return DP_OK;
}

// ---------------------------------------------------------------- (a) Gram on the tensor cores
template <int CH, int U>
int launch_gram_tc2(dp_ctx *c, const Args &b, cudaStream_t st) {
  using T = dpk::GT2<CH, U>;
  CUtensorMap tm;
  RET(make_h_tmap(c, b.H, b.n_sc * b.Bl, &tm, CH, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, U));
  auto kern = dpk::gram_tc2_kernel<CH, U>;
  CK(set_smem(kern, T::SMEM));
  LaunchScope ls(c, DP_KERNEL_GRAM, st);
  CK(launch_pdl(kern, dim3(std::min(b.n_sc * b.nchunks, c->num_sms)), dim3(T::THREADS), T::SMEM, st, tm, b));
  return DP_OK;
}
int launch_gram_tc2_any(dp_ctx *c, const Args &b, cudaStream_t st) {
  if (c->cfg.U == 32) return (b.S % 64 == 0) ? launch_gram_tc2<64, 32>(c, b, st) : launch_gram_tc2<32, 32>(c, b, st);
  if (c->cfg.U == 16) return (b.S % 64 == 0) ? launch_gram_tc2<64, 16>(c, b, st) : launch_gram_tc2<32, 16>(c, b, st);
  return fail(DP_ERR_UNSUPPORTED, "tensor-core Gram: U=%d", c->cfg.U);
}

// ---------------------------------------------------------------- (c) PD precode on the tensor cores
// U = 32, one z per subcarrier, K <= 16, 128-antenna blocks
bool precode_tc2_ok(const dp_ctx *c, const Args &a) {
  static const bool off = getenv("DP_NO_PC2") != nullptr;
  return !off && c->use_tc && c->cfg.U == 32 && a.K <= 16 && a.Bl % dpk::PC2_ROWS == 0 && a.zgroups == 1;
}

int launch_precode_tc2(dp_ctx *c, const Args &a, cudaStream_t st) {
  CUtensorMap tm;
  RET(make_h_tmap(c, a.H, a.n_sc * a.Bl, &tm, dpk::PC2_ROWS, CU_TENSOR_MAP_SWIZZLE_128B));
  static const bool smem_hs = getenv("DP_PC2_SMEM_HS") != nullptr;   // A/B: residual plane in shared memory
  auto kern = smem_hs ? dpk::precode_tc2_kernel<false> : dpk::precode_tc2_kernel<true>;
  const size_t smem = dpk::pc2_smem(!smem_hs);
  CK(set_smem(kern, smem));
  LaunchScope ls(c, DP_KERNEL_PRECODE, st);
  CK(launch_pdl(kern, dim3(std::min(a.n_sc, c->num_sms)), dim3(dpk::PC2_THREADS), smem, st, tm, a));
  return DP_OK;
}

// ---------------------------------------------------------------- FD with the cluster Gram on the tensor cores
// U = 32, S = 32 (fd_tc.cuh)
bool fd_tc_ok(const dp_ctx *c, const Args &a) {
  static const bool off = getenv("DP_NO_TC_FD") != nullptr;
  return !off && c->use_tc && c->cfg.U == 32 && a.S == 32 && a.K <= 16;
}

// fd_tc folds the per-subcarrier scalars into the kernel (no fd_finish_kernel) when a CTA holds
// whole subcarriers (Cl = 1, 2, 4); with DP_FD_CLUSTER_FOLD also when the rank's clusters of a
// subcarrier fill a thread-block cluster of Cl/4 CTAs (Cl = 8, 16, 32).  Returns CTAs per
// subcarrier, 0 = off (fd_finish_kernel after the FD kernel).
int fd_fold_of(const dp_ctx *c, const Args &a) {
  static const bool off = getenv("DP_NO_FOLD") != nullptr;
  static const bool cl_fold = getenv("DP_FD_CLUSTER_FOLD") != nullptr;   // A/B: thread-block-cluster fold
  if (off || a.Gout || !c->vruns.empty()) return 0;
  const int Cl = a.nchunks;
  if (Cl == 4) return 1;                                   // one CTA = one subcarrier: in-CTA fold
  // Cl = 8, 16, 32: a CTA cluster of Cl/4 waits for its slowest CTA before the sums (cfg4: FD kernel
  // 137.8 us with the 2-CTA cluster fold, 133.8 us without + fd_finish_kernel); opt-in
  if (cl_fold && (Cl == 8 || Cl == 16 || Cl == 32)) return Cl / 4;
  if (4 % Cl == 0) return 1;
  return 0;
}

template <int KC, bool WTC>
int launch_fd_tc(dp_ctx *c, const Args &a, cudaStream_t st) {
  CUtensorMap tm;
  RET(make_h_tmap(c, a.H, a.n_sc * a.Bl - a.hrow_off, &tm, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B));
  auto kern = dpk::fd_tc_kernel<KC, WTC>;
  static const size_t pad = getenv("DP_FD_SMEM_PAD") ? (size_t)atoi(getenv("DP_FD_SMEM_PAD")) : 0;   // occupancy experiments
  const size_t smem = dpk::FDT_SMEM + pad;
  CK(set_smem(kern, smem));
  const int nprob = a.n_sc * a.nchunks;
  Args b = a;
  // resident CTAs: 3 per SM; the L2 prefetch assumes contiguous clusters (off for unequal runs)
  static const int pf_waves = getenv("DP_FD_PF") ? atoi(getenv("DP_FD_PF")) : 3;   // A/B: CTAs ahead / num_sms
  b.pf_dist = a.Bl == a.nchunks * 32 ? pf_waves * c->num_sms : 0;
  b.fold = fd_fold_of(c, a);
  LaunchScope ls(c, DP_KERNEL_FUSED_FD, st);
  if (b.fold > 1)
    CK(launch_pdl_cluster(kern, dim3((nprob + 3) / 4), dim3(dpk::FDT_THREADS), smem, b.fold, st, tm, b));
  else
    CK(launch_pdl(kern, dim3((nprob + 3) / 4), dim3(dpk::FDT_THREADS), smem, st, tm, b));
  return DP_OK;
}
int launch_fd_tc_kc(dp_ctx *c, const Args &a, cudaStream_t st) {
  static const bool simt_w = getenv("DP_FD_SIMT_WHITEN") != nullptr;   // A/B: SIMT whitening
  // tensor-core whitening stacks a CTA's 4 problems on one s: they must share the subcarrier
  if (simt_w || a.nchunks % 4 != 0) {
    switch (kc_of(a.K)) {
      case 7: return launch_fd_tc<7, false>(c, a, st);
      case 8: return launch_fd_tc<8, false>(c, a, st);
      case 14: return launch_fd_tc<14, false>(c, a, st);
      default: return launch_fd_tc<16, false>(c, a, st);
    }
  }
  switch (kc_of(a.K)) {
    case 7: return launch_fd_tc<7, true>(c, a, st);
    case 8: return launch_fd_tc<8, true>(c, a, st);
    case 14: return launch_fd_tc<14, true>(c, a, st);
    default: return launch_fd_tc<16, true>(c, a, st);
  }
}

}  // namespace dpi
