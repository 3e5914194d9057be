// ber.cuh — device-side uncoded-BER harness (Fig. 2):
// synthetic Rayleigh frames drawn on the GPU, and the UE-side receiver + bit-error
// count.  Not part of the precoder: it feeds dp_precode_pd / dp_precode_fd and
// scores their outputs the way the paper's simulations do.
//
// Random numbers: Philox4x32-10 (Salmon et al., SC'11), counter = (index lo, index hi,
// stream id, frame), key = (seed lo, seed hi).  Every value is a pure function of
// (seed, frame, stream, index), so frames are reproducible and independent of the
// launch shape.  Streams: 0 = channel H, 1 = symbol indices, 2 = noise.
//   H[sc][b][u] ~ CN(0, 1)     (re, im ~ N(0, 1/2), Box-Muller)        (P:237 Rayleigh, reading R16)
//   idx ~ U{0..M-1}, s = Gray-mapped square QAM, Es = 1                 (P:237 64-QAM, readings R1, R17)
//   n ~ CN(0, N0)
// Receiver (Eq. 1 with the joint UE scaling of P:106-114, reading R9 for FD):
//   s_hat[sc][k][u] = rx[sc] (sum_b H[sc][b][u] x[sc][k][b] + n[sc][k][u]);
//   per-axis nearest-level decision, Gray label, bit errors = popcount(label_tx ^ label_rx).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace dpk {

struct Philox {
  __device__ static uint4 round(uint4 c, uint2 k) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    const uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    return make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  __device__ static uint4 gen(uint64_t seed, uint32_t stream, uint32_t frame, uint64_t i) {
    uint4 c = make_uint4((uint32_t)i, (uint32_t)(i >> 32), stream, frame);
    uint2 k = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      c = round(c, k);
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    return c;
  }
};

// uniform in (0, 1]
__device__ __forceinline__ float u01(uint32_t v) { return ((float)(v >> 8) + 1.0f) * (1.0f / 16777216.0f); }
// two independent N(0, sigma^2) from two uniforms (Box-Muller)
__device__ __forceinline__ float2 gauss2(uint32_t a, uint32_t b, float sigma) {
  const float r = sqrtf(-2.0f * logf(u01(a))) * sigma;
  float sn, cs;
  sincospif(2.0f * u01(b), &sn, &cs);
  return make_float2(r * cs, r * sn);
}

// square Gray QAM, symbol index i = (label_I << (bits/2)) | label_Q; a label g sits at
// level position p with p ^ (p >> 1) = g; amplitude (2p - (m - 1)) * scale
__device__ __forceinline__ int gray_inverse(int g) {
  int p = g;
  for (int s = 1; s < 16; s <<= 1) p ^= p >> s;
  return p;
}
struct Qam {
  int m, hb;     // levels per axis, bits per axis
  float scale;   // sqrt(3 / (2 (M - 1)))
  __device__ float2 point(int idx) const {
    const int pi = gray_inverse(idx >> hb), pq = gray_inverse(idx & (m - 1));
    return make_float2((float)(2 * pi - (m - 1)) * scale, (float)(2 * pq - (m - 1)) * scale);
  }
  __device__ int label(float v) const {   // nearest level, ties to the lower one, Gray label
    float p = floorf((v / scale + (float)(m - 1)) * 0.5f + 0.5f - 1e-6f);
    p = fminf(fmaxf(p, 0.f), (float)(m - 1));
    const int q = (int)p;
    return q ^ (q >> 1);
  }
};

struct SynthArgs {
  uint64_t seed;
  uint32_t frame;
  int n_sc, B, U, K;
  Qam q;
  float sigma_n;          // sqrt(N0 / 2)
  float2 *H, *s, *noise;
  uint8_t *idx;
};

// one thread per pair of complex entries of each stream
__global__ void synth_kernel(SynthArgs a) {
  const size_t nH = (size_t)a.n_sc * a.B * a.U, nS = (size_t)a.n_sc * a.K * a.U;
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const float sh = 0.70710678118654752f;   // sqrt(1/2)
  if (2 * t < nH) {
    const uint4 r = Philox::gen(a.seed, 0, a.frame, t);
    a.H[2 * t] = gauss2(r.x, r.y, sh);
    if (2 * t + 1 < nH) a.H[2 * t + 1] = gauss2(r.z, r.w, sh);
  }
  if (2 * t < nS) {
    const uint4 r = Philox::gen(a.seed, 1, a.frame, t);
    const int M = a.q.m * a.q.m;
    for (int j = 0; j < 2 && 2 * t + j < nS; ++j) {
      const uint32_t v = j ? r.y : r.x;
      const int id = (int)(((uint64_t)v * (uint64_t)M) >> 32);   // uniform on 0..M-1 (M | 2^32)
      a.idx[2 * t + j] = (uint8_t)id;
      a.s[2 * t + j] = a.q.point(id);
    }
    if (a.noise) {
      const uint4 g = Philox::gen(a.seed, 2, a.frame, t);
      a.noise[2 * t] = gauss2(g.x, g.y, a.sigma_n);
      if (2 * t + 1 < nS) a.noise[2 * t + 1] = gauss2(g.z, g.w, a.sigma_n);
    }
  }
}

struct RxArgs {
  int n_sc, B, U, K;
  Qam q;
  const float2 *H, *x, *noise;
  const float *rx;
  const uint8_t *idx;
  unsigned long long *errors;
};

// one CTA per subcarrier: H[sc] and x[sc] staged in shared memory, thread (k, u)
__global__ void rx_count_kernel(RxArgs a) {
  extern __shared__ float2 sm_rx[];
  const int sc = blockIdx.x;
  float2 *Hs = sm_rx, *xs = Hs + (size_t)a.B * a.U;
  for (int i = threadIdx.x; i < a.B * a.U; i += blockDim.x) Hs[i] = a.H[(size_t)sc * a.B * a.U + i];
  for (int i = threadIdx.x; i < a.K * a.B; i += blockDim.x) xs[i] = a.x[(size_t)sc * a.K * a.B + i];
  __syncthreads();
  const float r = a.rx[sc];
  int err = 0;
  for (int e = threadIdx.x; e < a.K * a.U; e += blockDim.x) {
    const int k = e / a.U, u = e % a.U;
    float yr = 0.f, yi = 0.f;
    for (int b = 0; b < a.B; ++b) {          // y_u = sum_b H^paper_{u,b} x_b = sum_b H[b][u] x[b]
      const float2 h = Hs[b * a.U + u], v = xs[k * a.B + b];
      yr = fmaf(h.x, v.x, fmaf(-h.y, v.y, yr));
      yi = fmaf(h.x, v.y, fmaf(h.y, v.x, yi));
    }
    const size_t o = ((size_t)sc * a.K + k) * a.U + u;
    const float2 n = a.noise ? a.noise[o] : make_float2(0.f, 0.f);
    const float sr = r * (yr + n.x), si = r * (yi + n.y);
    const int tx = a.idx[o];
    const int rxi = (a.q.label(sr) << a.q.hb) | a.q.label(si);
    err += __popc((unsigned)(tx ^ rxi));
  }
  for (int m = 16; m >= 1; m >>= 1) err += __shfl_xor_sync(0xffffffffu, err, m);
  if ((threadIdx.x & 31) == 0 && err) atomicAdd(a.errors, (unsigned long long)err);
}

}  // namespace dpk
