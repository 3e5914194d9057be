// k_pd.cu — launchers of the SIMT per-subcarrier Gram (kernel (a): G_c = H_c H_c^H, per
// cluster or summed over the rank's clusters) and precode (kernel (c): x_c = H_c^H z, P:178,
// P:296) of kernels.cuh.  At U = 32 (and U = 16 on request) the Gram runs on the tensor cores
// (launch_gram_tc2_any, k_tc.cu).
#include "dp_internal.cuh"

namespace dpi {

template <int U, bool PER_CHUNK>
int launch_gram(dp_ctx *c, const Args &a, int nw, cudaStream_t st) {
  if constexpr (U == 32 || U == 16) {
    Args b = a;                                   // work item = (subcarrier, group)
    if (!PER_CHUNK) {
      b.S = a.Bl;                                 // one group: all local antennas
      b.nchunks = 1;
    }
    // tensor-core Gram, operands straight from TMA.  U = 16 (M = 64 UMMAs) is correct but measured
    // no faster than the SIMT kernel at cfg3 (17.3 vs 15.5 us: 128-antenna items are too small to
    // amortise the per-item epilogue), so it is opt-in (DP_GRAM_TC16)
    static const bool tc16 = getenv("DP_GRAM_TC16") != nullptr;
    if (c->use_tc && b.S % 32 == 0 && (U == 32 || tc16)) return launch_gram_tc2_any(c, b, st);
  }
  const size_t sm = smem_gram(U, a.Bl, nw);
  if (sm > 227 * 1024) return fail(DP_ERR_UNSUPPORTED, "Gram tile needs %zu B of shared memory", sm);
  auto kern = dpk::gram_kernel<U, PER_CHUNK>;
  CK(set_smem(kern, sm));
  LaunchScope ls(c, DP_KERNEL_GRAM, st);
  CK(launch_pdl(kern, dim3(a.n_sc), dim3(nw * 32), sm, st, a));
  return DP_OK;
}

int launch_gram_any(dp_ctx *c, const Args &a, int nw, bool per_chunk, cudaStream_t st) {
  switch (c->cfg.U) {
    case 4: return per_chunk ? launch_gram<4, true>(c, a, nw, st) : launch_gram<4, false>(c, a, nw, st);
    case 8: return per_chunk ? launch_gram<8, true>(c, a, nw, st) : launch_gram<8, false>(c, a, nw, st);
    case 16: return per_chunk ? launch_gram<16, true>(c, a, nw, st) : launch_gram<16, false>(c, a, nw, st);
    case 32: return per_chunk ? launch_gram<32, true>(c, a, nw, st) : launch_gram<32, false>(c, a, nw, st);
  }
  return fail(DP_ERR_UNSUPPORTED, "U=%d", c->cfg.U);
}

template <int U, int KC>
int launch_precode(dp_ctx *c, const Args &a, int nw, cudaStream_t st) {
  const size_t sm = smem_precode(U, a.Bl, a.K, a.zgroups);
  if (sm > 227 * 1024) return fail(DP_ERR_UNSUPPORTED, "precode tile needs %zu B of shared memory", sm);
  auto kern = dpk::precode_kernel<U, KC>;
  CK(set_smem(kern, sm));
  LaunchScope ls(c, DP_KERNEL_PRECODE, st);
  CK(launch_pdl(kern, dim3(a.n_sc), dim3(nw * 32), sm, st, a));
  return DP_OK;
}
template <int U, int KC> struct Precode {
  static int run(dp_ctx *c, const Args &a, int nw, cudaStream_t st) { return launch_precode<U, KC>(c, a, nw, st); }
};
int launch_precode_any(dp_ctx *c, const Args &a, int nw, cudaStream_t st) {
  return dispatch<Precode>(c->cfg.U, a.K, c, a, nw, st);
}

}  // namespace dpi
