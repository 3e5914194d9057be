// TMA streaming-bandwidth probe (sm_100a): 148 persistent CTAs stream a 1 GiB fp32
// matrix [rows][64] through an NS-stage shared-memory ring; one consumer warp frees
// each stage as soon as it lands.  Modes: 0 = 2-D tensor boxes SWIZZLE_128B_ATOM_32B
// (gram_tc2 operands), 1 = 2-D SWIZZLE_128B (precode_tc2 operands), 2 = 1-D bulk copy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/tma_bw_probe scripts/tma_bw_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *m, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(m)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t *m, uint32_t ph) {
  asm volatile("{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}\n" ::"r"(su32(m)), "r"(ph) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t *m, uint32_t b) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(m)), "r"(b) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t *m) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(m)) : "memory");
}

__global__ void read_flush(const float4 *p, size_t n, float *out) {
  float acc = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) acc += p[i].x;
  if (acc == 12345.f) out[0] = acc;
}
__device__ int my_chunks(int nchunks, int per) {
  int n = 0;
  for (int i = 0;; ++i) {
    const int c = per == 1 ? blockIdx.x + i * gridDim.x : ((i / per) * gridDim.x + blockIdx.x) * per + i % per;
    if (c >= nchunks) return n;
    ++n;
  }
}
template <int MODE, int CHAIN>
__global__ void __launch_bounds__(192, 1) probe(const __grid_constant__ CUtensorMap tm, const float *src, int nchunks,
                                               int rows_per_chunk, int ns, float *sink, int getenv_item) {
  extern __shared__ __align__(1024) uint8_t sm_[];
  uint8_t *sm = sm_ + ((1024u - (su32(sm_) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full[32], freeb[32], mid[32];
  const int chunk_bytes = rows_per_chunk * 256;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ns; ++i) { mbar_init(&full[i], 1); mbar_init(&freeb[i], 1); mbar_init(&mid[i], 128); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0, ph = 0, g = 0;
    const int per = getenv_item;   // chunks per item (item-major order, items strided over CTAs)
    for (int i = 0; i < (nchunks + gridDim.x * per - 1) / (gridDim.x * per) * per; ++i, ++g) {
      const int c = per == 1 ? blockIdx.x + i * gridDim.x : ((i / per) * gridDim.x + blockIdx.x) * per + i % per;
      if (c >= nchunks) break;
      if (g >= ns) mbar_wait(&freeb[s], ph ^ 1);
      uint8_t *st = sm + (size_t)s * chunk_bytes;
      expect_tx(&full[s], chunk_bytes);
      if (MODE == 2) {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(st)),
                     "l"(src + (size_t)c * rows_per_chunk * 64), "r"(chunk_bytes), "r"(su32(&full[s])) : "memory");
      } else {
        for (int h = 0; h < 2; ++h)
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                           su32(st + h * chunk_bytes / 2)),
                       "l"(reinterpret_cast<uint64_t>(&tm)), "r"(32 * h), "r"(c * rows_per_chunk), "r"(su32(&full[s])) : "memory");
      }
      if (++s == ns) { s = 0; ph ^= 1; }
    }
  } else if (CHAIN == 0 && threadIdx.x == 32) {
    int s = 0, ph = 0;
    float acc = 0.f;
    for (int c = 0, nmy = my_chunks(nchunks, getenv_item); c < nmy; ++c) {
      mbar_wait(&full[s], ph);
      acc += *reinterpret_cast<const float *>(sm + (size_t)s * chunk_bytes + 4 * (c & 63));
      arrive(&freeb[s]);
      if (++s == ns) { s = 0; ph ^= 1; }
    }
    sink[blockIdx.x] = acc;
  } else if (CHAIN && threadIdx.x >= 64) {
    // chained hand-off as in gram_tc2: 128 threads wait full -> arrive mid; one thread waits mid -> free
    int s = 0, ph = 0;
    float acc = 0.f;
    for (int c = 0, nmy = my_chunks(nchunks, getenv_item); c < nmy; ++c) {
      mbar_wait(&full[s], ph);
      acc += *reinterpret_cast<const float *>(sm + (size_t)s * chunk_bytes + 4 * (threadIdx.x & 63));
      if (CHAIN == 2) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      arrive(&mid[s]);
      if (++s == ns) { s = 0; ph ^= 1; }
    }
    sink[blockIdx.x * 256 + threadIdx.x] = acc;
  } else if (CHAIN && threadIdx.x == 32) {
    int s = 0, ph = 0;
    for (int c = 0, nmy = my_chunks(nchunks, getenv_item); c < nmy; ++c) {
      mbar_wait(&mid[s], ph);
      arrive(&freeb[s]);
      if (++s == ns) { s = 0; ph ^= 1; }
    }
  }
}

int main() {
  const size_t rows = getenv("ROWS") ? (size_t)atol(getenv("ROWS")) : ((size_t)1 << 22);   // default 4M rows x 256 B = 1 GiB
  float *src, *sink;
  cudaMalloc(&src, rows * 256);
  cudaMemset(src, 0, rows * 256);
  cudaMalloc(&sink, 148 * 256 * 4);
  PFN_cuTensorMapEncodeTiled enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float *flush;
  cudaMalloc(&flush, (size_t)512 << 20);
  for (int per : {1, 4})
  for (int chain = 0; chain < 2; ++chain)
  for (int mode = 0; mode < 1; mode += 2)
    for (int rpc : {64})
      for (int ns : {5, 8}) {
        const size_t smem = (size_t)ns * rpc * 256 + 1024;
        if (smem > 227 * 1024 || (mode < 2 && rpc > 256)) continue;
        CUtensorMap tm;
        cuuint64_t dims[2] = {64, rows};
        cuuint64_t str[1] = {256};
        cuuint32_t box[2] = {32, (cuuint32_t)rpc}, es[2] = {1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, src, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            mode == 0 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const int nchunks = (int)(rows / rpc);
        auto k = mode == 0 ? (chain == 0 ? probe<0, 0> : chain == 1 ? probe<0, 1> : probe<0, 2>)
                           : (chain == 0 ? probe<2, 0> : chain == 1 ? probe<2, 1> : probe<2, 2>);
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        float best = 1e9;
        for (int rep = 0; rep < 4; ++rep) {
          if (getenv("DIRTY")) cudaMemsetAsync(flush, rep, (size_t)512 << 20);
          else read_flush<<<nsm * 8, 256>>>((const float4 *)flush, ((size_t)512 << 20) / 16, sink);
          cudaEventRecord(a);
          k<<<nsm, 192, smem>>>(tm, src, nchunks, rpc, ns, sink, per);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (rep && ms < best) best = ms;
        }
        printf("per %d chain %d mode %d rows/chunk %3d (%5d B) stages %2d (%6zu B in flight/SM): %7.1f GB/s  %s\n", per, chain, mode, rpc, rpc * 256, ns,
               (size_t)ns * rpc * 256, rows * 256 / best / 1e6, cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
