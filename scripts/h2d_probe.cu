// h2d_probe.cu — pinned host -> device copy bandwidth for a cfg4-sized H (78.6 MB), split into
// `chunks` pieces issued round-robin on `nstreams` streams (one DMA queue each), CUDA events.
#include <cuda_runtime.h>
#include <cstdio>
int main() {
  const size_t bytes = 1200ull * 256 * 32 * 8;
  void *h, *d;
  cudaHostAlloc(&h, bytes, cudaHostAllocDefault);
  cudaMalloc(&d, bytes);
  memset(h, 1, bytes);
  cudaStream_t st[8];
  for (int i = 0; i < 8; ++i) cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int ns_list[] = {1, 2, 4, 8}, ch_list[] = {1, 8, 32};
  for (int ns : ns_list)
    for (int ch : ch_list) {
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaDeviceSynchronize();
        cudaEventRecord(e0, 0);
        for (int s = 0; s < ns; ++s) cudaStreamWaitEvent(st[s], e0, 0);
        const size_t per = bytes / ch;
        for (int c = 0; c < ch; ++c)
          cudaMemcpyAsync((char *)d + c * per, (char *)h + c * per, per, cudaMemcpyHostToDevice, st[c % ns]);
        for (int s = 0; s < ns; ++s) {
          cudaEvent_t ej;
          cudaEventCreateWithFlags(&ej, cudaEventDisableTiming);
          cudaEventRecord(ej, st[s]);
          cudaStreamWaitEvent(0, ej, 0);
          cudaEventDestroy(ej);
        }
        cudaEventRecord(e1, 0);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("streams %d chunks %2d: %.3f ms  %.1f GB/s\n", ns, ch, best, bytes / best / 1e6);
    }
  // D2H for reference
  float ms; cudaEventRecord(e0, 0); cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, 0); cudaEventRecord(e1, 0);
  cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); printf("D2H 1 stream: %.1f GB/s\n", bytes / ms / 1e6);
  return 0;
}
