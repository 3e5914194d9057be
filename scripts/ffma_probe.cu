// FFMA throughput probe: 3-distinct-register FFMA chains vs shared-operand (reuse) chains.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float *out, int iters, float s) {
  float a[16], x[16], y[16];
  for (int i = 0; i < 16; ++i) { a[i] = threadIdx.x * 1e-3f + i; x[i] = s + i * 1e-4f; y[i] = 1.0f - i * 1e-5f; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) a[i] = fmaf(x[i], y[i], a[i]);          // 3 distinct sources per FFMA
      else if (MODE == 1) a[i] = fmaf(x[0], y[0], a[i]);     // 2 shared sources (reuse)
      else a[i] = fmaf(x[i & 1], y[0], a[i]);                // complex-MAC-like: 2 of 3 shared across pairs
    }
  }
  float r = 0; for (int i = 0; i < 16; ++i) r += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
int main() {
  float *o; cudaMalloc(&o, 148 * 8 * 1024 * 4);
  int iters = 20000;
  for (int mode = 0; mode < 3; ++mode) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) k<0><<<148 * 8, 256>>>(o, iters, 0.5f);
      if (mode == 1) k<1><<<148 * 8, 256>>>(o, iters, 0.5f);
      if (mode == 2) k<2><<<148 * 8, 256>>>(o, iters, 0.5f);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double flops = 2.0 * 16 * iters * 148.0 * 8 * 256;
      if (rep) printf("mode %d: %.1f TFLOP/s (%.3f ms)\n", mode, flops / ms / 1e9, ms);
    }
  }
  return 0;
}
