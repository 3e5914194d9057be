// FFMA vs FFMA2 (fma.rn.f32x2, sm_100a) throughput probe, and a complex-MAC mix:
// mode 0: 16 independent FFMA chains; mode 1: 16 independent FFMA2 chains (32 FMAs);
// mode 2: complex MAC acc += conj(o) * v as 2 FFMA2 (broadcast + swapped operand);
// mode 3: 16 independent DFMA chains (fp64 pipe, the DP_FLAG_FP64 kernels).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/ffma2_probe.cu -o /tmp/ffma2_probe
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void fma2(u64 &d, u64 a, u64 b) { asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b)); }
__device__ __forceinline__ float lo(u64 v) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); return a + b; }
template <int MODE>
__global__ void k(float *out, int iters, float s) {
  float r = 0;
  if (MODE == 0) {
    float a[16], x[16], y[16];
    for (int i = 0; i < 16; ++i) { a[i] = threadIdx.x * 1e-3f + i; x[i] = s + i * 1e-4f; y[i] = 1.0f - i * 1e-5f; }
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = fmaf(x[i], y[i], a[i]);
    for (int i = 0; i < 16; ++i) r += a[i];
  } else if (MODE == 1) {
    u64 a[16], x[16], y[16];
    for (int i = 0; i < 16; ++i) { a[i] = pk(threadIdx.x * 1e-3f + i, i); x[i] = pk(s + i * 1e-4f, s); y[i] = pk(1.0f - i * 1e-5f, 1.f); }
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 16; ++i) fma2(a[i], x[i], y[i]);
    for (int i = 0; i < 16; ++i) r += lo(a[i]);
  } else if (MODE == 3) {
    double a[16], x[16], y[16];
    for (int i = 0; i < 16; ++i) { a[i] = threadIdx.x * 1e-3 + i; x[i] = s + i * 1e-4; y[i] = 1.0 - i * 1e-5; }
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = fma(x[i], y[i], a[i]);
    for (int i = 0; i < 16; ++i) r += (float)a[i];
  } else {
    u64 a[8], v[8];
    const float ox = s, oy = s * 0.5f;
    for (int i = 0; i < 8; ++i) { a[i] = pk(threadIdx.x * 1e-3f + i, i); v[i] = pk(1.0f - i * 1e-5f, 1e-3f * i); }
    const u64 oxx = pk(ox, ox), oyn = pk(oy, -oy);
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float vx, vy; asm("mov.b64 {%0,%1}, %2;" : "=f"(vx), "=f"(vy) : "l"(v[i]));
        fma2(a[i], oxx, v[i]);
        fma2(a[i], oyn, pk(vy, vx));
      }
    for (int i = 0; i < 8; ++i) r += lo(a[i]);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
int main() {
  float *o; cudaMalloc(&o, 148 * 8 * 1024 * 4);
  int iters = 20000;
  for (int mode = 0; mode < 4; ++mode) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) k<0><<<148 * 8, 256>>>(o, iters, 0.5f);
      if (mode == 1) k<1><<<148 * 8, 256>>>(o, iters, 0.5f);
      if (mode == 2) k<2><<<148 * 8, 256>>>(o, iters, 0.5f);
      if (mode == 3) k<3><<<148 * 8, 256>>>(o, iters / 4, 0.5f);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double fmas = (mode == 0 ? 16.0 : mode == 3 ? 16.0 / 4 : 32.0) * iters * 148.0 * 8 * 256;
      double instr = (mode == 3 ? 4.0 : 16.0) * iters * 148.0 * 8 * 256 / 32;   // warp instructions
      if (rep) printf("mode %d: %.1f TFLOP/s  %.2f warp-instr/clk/SM @1.965GHz (%.3f ms)\n", mode, 2 * fmas / ms / 1e9,
                      instr / (ms * 1e-3) / 148 / 1.965e9, ms);
    }
  }
  return 0;
}
