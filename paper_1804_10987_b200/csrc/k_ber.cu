// k_ber.cu — the uncoded-BER harness entry points of the C-ABI (include/dp.h, SURVEY.md §8 f1;
// Sec. IV-D): device-side frame synthesis and the UE receiver + bit-error count
// (ber.cuh).  Not part of the precoder.
#include "dp_internal.cuh"
#include "ber.cuh"

extern "C" {

// ---------------------------------------------------------------- BER harness (f1)
namespace {
using dpi::fail;
int qam_of(int M, dpk::Qam *q) {
  int hb = 0;
  while ((1 << (2 * hb)) < M) ++hb;
  if (M != 4 && M != 16 && M != 64 && M != 256) return fail(DP_ERR_INVALID, "M=%d: square QAM with M in {4,16,64,256}", M);
  q->hb = hb;
  q->m = 1 << hb;
  q->scale = (float)std::sqrt(3.0 / (2.0 * (M - 1)));
  return DP_OK;
}
int check_dims(int n_sc, int B, int U, int K) {
  if (n_sc <= 0 || B <= 0 || U <= 0 || K <= 0 || U > 32 || B > 256 || K > 16)
    return fail(DP_ERR_INVALID, "dims n_sc=%d B=%d U=%d K=%d (need > 0, U <= 32, B <= 256, K <= 16)", n_sc, B, U, K);
  return DP_OK;
}
}  // namespace

int dp_synth_frame(unsigned long long seed, unsigned long long frame, int n_sc, int B, int U, int K, int M, double N0,
                   dp_c32 *H, dp_c32 *s, unsigned char *idx, dp_c32 *noise, void *stream) {
  dpi::clear_error();
  RET(check_dims(n_sc, B, U, K));
  if (!H || !s || !idx) return fail(DP_ERR_INVALID, "H, s and idx must be device pointers");
  if (!(N0 >= 0) || !std::isfinite(N0)) return fail(DP_ERR_INVALID, "N0 must be finite and >= 0");
  dpk::SynthArgs a;
  RET(qam_of(M, &a.q));
  a.seed = seed;
  a.frame = (uint32_t)frame;
  a.n_sc = n_sc; a.B = B; a.U = U; a.K = K;
  a.sigma_n = (float)std::sqrt(N0 / 2.0);
  a.H = reinterpret_cast<float2 *>(H);
  a.s = reinterpret_cast<float2 *>(s);
  a.noise = reinterpret_cast<float2 *>(noise);
  a.idx = idx;
  const size_t n = std::max((size_t)n_sc * B * U, (size_t)n_sc * K * U);
  const size_t thr = (n + 1) / 2;
  dpk::synth_kernel<<<(unsigned)((thr + 255) / 256), 256, 0, (cudaStream_t)stream>>>(a);
  CK(cudaGetLastError());
  return DP_OK;
}

int dp_receive_count(int n_sc, int B, int U, int K, int M, const dp_c32 *H, const dp_c32 *x, const dp_c32 *noise,
                     const float *rx, const unsigned char *idx, unsigned long long *errors, void *stream) {
  dpi::clear_error();
  RET(check_dims(n_sc, B, U, K));
  if (!H || !x || !rx || !idx || !errors) return fail(DP_ERR_INVALID, "NULL argument");
  dpk::RxArgs a;
  RET(qam_of(M, &a.q));
  a.n_sc = n_sc; a.B = B; a.U = U; a.K = K;
  a.H = reinterpret_cast<const float2 *>(H);
  a.x = reinterpret_cast<const float2 *>(x);
  a.noise = reinterpret_cast<const float2 *>(noise);
  a.rx = rx;
  a.idx = idx;
  a.errors = errors;
  const size_t sm = ((size_t)B * U + (size_t)K * B) * sizeof(float2);
  CK(dpi::set_smem(dpk::rx_count_kernel, sm));
  dpk::rx_count_kernel<<<n_sc, 256, sm, (cudaStream_t)stream>>>(a);
  CK(cudaGetLastError());
  return DP_OK;
}

}  // extern "C"
