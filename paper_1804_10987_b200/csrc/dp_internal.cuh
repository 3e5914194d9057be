// dp_internal.cuh — library-internal declarations shared by the translation units of
// libdp.so (dp_api.cu: the C-ABI host side; k_*.cu: kernel launchers, one group of
// kernels per unit so the library compiles in parallel).  Not installed, not part of
// the C-ABI (include/dp.h is).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "dp.h"
#include "kernels.cuh"

namespace dpi {

// record a thread-local error message (dp_last_error) and return `code`  (dp_api.cu)
int fail(int code, const char *fmt, ...);
void clear_error();

#define CK(call)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess) return dpi::fail(DP_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call, \
                                            cudaGetErrorString(e_));                              \
  } while (0)
#define NK(call)                                                                                  \
  do {                                                                                            \
    ncclResult_t r_ = (call);                                                                     \
    if (r_ != ncclSuccess) return dpi::fail(DP_ERR_NCCL, "%s:%d %s: %s", __FILE__, __LINE__, #call, \
                                            ncclGetErrorString(r_));                              \
  } while (0)
#define RET(call)                 \
  do {                            \
    int rc_ = (call);             \
    if (rc_ != DP_OK) return rc_; \
  } while (0)

// count a collective's payload (floats) in the context's exchange ledger
#define LEDGER(c, kind, nfloats) ((c)->ledger[(kind)] += (long long)(nfloats))

struct ProfRec {
  int kid;
  cudaEvent_t a, b;
};

}  // namespace dpi

struct dp_ctx {
  dp_config cfg;
  int Bl = 0;        // antennas on this rank
  int Cl = 0;        // clusters on this rank
  int S = 0;         // cluster size B / C
  int pd_chunk = 0;  // rows per SG chunk in the per-subcarrier PD kernels
  int pd_nchunks = 0;
  int pd_nw = 0;     // warps per CTA of the per-subcarrier PD kernels
  int fd_nw = 0;     // warps per CTA of the FD fused kernel
  int fdu_nw = 0;    // warps of the FD unfused per-subcarrier kernels (chunk = cluster)
  int pdf_nw = 0;    // warps per CTA of the single-pass PD kernel at world 1 (0: not used)
  bool comm_on = false;
  bool use_tc = true;        // tensor-core paths where available (env DP_NO_TC=1 disables)
  int num_sms = 148;
  ncclComm_t comm = nullptr;
  // device workspace
  float2 *s_buf = nullptr;   // broadcast landing buffer for s
  float2 *G = nullptr;       // packed Grams
  float2 *z = nullptr;       // whitened symbols (unfused / T1)
  float *beta = nullptr;     // per problem beta
  float *pw = nullptr;       // power partials
  float *fin = nullptr;      // [n_sc][2] per-subcarrier scalars
  int *bad = nullptr;        // non-HPD counter
  size_t pw_len = 0;
  // DP_FLAG_FP64 workspace (fp64 Gram / z of the PD kernels), sized at dp_init when the flag is set
  double2 *G64 = nullptr;    // packed fp64 Grams [n_sc][U(U+1)/2]
  double2 *z64 = nullptr;    // fp64 z [n_sc][K][U]
  // host staging (host-pointer calls)
  float2 *h_dev = nullptr, *s_dev = nullptr, *x_dev = nullptr;
  cudaStream_t st_h2d = nullptr, st_d2h = nullptr;   // host-pointer pipeline copy streams
  // DP_FLAG_HOST_ASYNC: per-chunk completion of the last call (kernels on chunk i, D2H of chunk i)
  static constexpr int HP_MAXCH = 64;
  cudaEvent_t hp_kdone[HP_MAXCH] = {}, hp_d2h[HP_MAXCH] = {};
  int hp_nch = 0;                                    // chunks of the last async call (0: none pending)
  cudaStream_t st_side = nullptr;                    // side stream: s broadcast beside the PD Gram
  cudaEvent_t ev_side0 = nullptr, ev_side1 = nullptr;
  // host-side caches (per-frame host overhead): tensor maps by (pointer, rows, box, swizzle),
  // device-ness of recently seen pointers
  struct TmapEntry { const void *p; int rows, box, sw; CUtensorMap tm; };
  std::vector<TmapEntry> tmaps;
  std::vector<std::pair<const void *, bool>> ptr_kind;
  // unequal clusters (dp_set_clusters; Eq. 9): this rank's clusters as maximal
  // runs of equal (size, power share, tau); empty = the equal split B/C, rho^2/C, cfg.tau
  struct VarRun { int cl0, len, S, off; double w, tau; };
  std::vector<VarRun> vruns;
  std::vector<int> vsizes;   // all C cluster sizes (global) when set
  cudaStream_t st_run[3] = {nullptr, nullptr, nullptr};   // concurrent runs (fork / join on events)
  cudaEvent_t ev_fork = nullptr, ev_join[3] = {nullptr, nullptr, nullptr};
  bool run_streams = false;  // st_run / ev_* all created (dp_set_clusters)
  float *vb = nullptr;       // per-run beta / power scratch [2][n_sc][Cl] (dp_set_clusters)
  float *rd_buf = nullptr;   // dp_read_scalars staging for host destinations [n_sc]
  // last call
  int last_mode = -1;        // 0 pd, 1 fd
  int prepared = -1;         // W cached in G by dp_prepare_pd (0) / dp_prepare_fd (1); -1 none
  // profiling
  std::vector<dpi::ProfRec> prof;
  std::vector<cudaEvent_t> ev_pool;
  double prof_ms[DP_NUM_KERNELS] = {0};
  long long prof_n[DP_NUM_KERNELS] = {0};
  long long launches = 0;
  // DP_PD_NVLINK (k_lsa.cu): symmetric windows over G, z, beta (ncclMemAlloc'd) and the device communicator
  ncclWindow_t win_g = nullptr, win_z = nullptr, win_b = nullptr;
  ncclDevComm *devcomm = nullptr;
  bool lsa = false;
  // exchange ledger: float payload elements handed to each kind of collective by this rank
  long long ledger[DP_NUM_COMM] = {0};
};

namespace dpi {

using dpk::Args;

inline int next_pow2(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

// precode/whitening symbol chunk KC: one chunk for K <= 16 (7, 8, 14 or 16), else chunks of 16
inline int kc_of(int K) { return K == 7 ? 7 : K == 14 ? 14 : K <= 8 ? 8 : 16; }

template <int KC>
int zs_of(int K) { return dpk::ZL<KC>::zs(K); }
inline int zs_rt(int K) {
  switch (kc_of(K)) {
    case 7: return zs_of<7>(K);
    case 8: return zs_of<8>(K);
    case 14: return zs_of<14>(K);
    default: return zs_of<16>(K);
  }
}
template <int U>
int fd_scr_rt(int K) {
  switch (kc_of(K)) {
    case 7: return dpk::fd_scr_size<U, 7>(K);
    case 8: return dpk::fd_scr_size<U, 8>(K);
    case 14: return dpk::fd_scr_size<U, 14>(K);
    default: return dpk::fd_scr_size<U, 16>(K);
  }
}
template <int U>
int solve_scr_rt(int K) {
  switch (kc_of(K)) {
    case 7: return dpk::solve_scr_size<U, 7>(K);
    case 8: return dpk::solve_scr_size<U, 8>(K);
    case 14: return dpk::solve_scr_size<U, 14>(K);
    default: return dpk::solve_scr_size<U, 16>(K);
  }
}
inline int fd_scr_u(int U, int K) {
  return U == 4 ? fd_scr_rt<4>(K) : U == 8 ? fd_scr_rt<8>(K) : U == 16 ? fd_scr_rt<16>(K) : fd_scr_rt<32>(K);
}
inline int solve_scr_u(int U, int K) {
  return U == 4 ? solve_scr_rt<4>(K) : U == 8 ? solve_scr_rt<8>(K) : U == 16 ? solve_scr_rt<16>(K)
                                                                            : solve_scr_rt<32>(K);
}

// ---------------------------------------------------------------- smem sizes (bytes)
// fd_fused_kernel: per problem [tile S x U][rep scratch]; nw warps of 32 / U sub-groups
inline size_t smem_fd_fused(int U, int S, int K, int nw, int rep = 1) {
  const int nsg = nw * (32 / U);
  return ((size_t)(nsg / rep) * S * U + (size_t)nsg * fd_scr_u(U, K)) * sizeof(float2);
}
inline size_t smem_gram(int U, int Bl, int nw) {
  return ((size_t)Bl * U + (size_t)(nw / 2) * 32 * (U / 2 + U / 4)) * sizeof(float2);
}
inline size_t smem_solve(int U, int K) { return (size_t)4 * (32 / U) * solve_scr_u(U, K) * sizeof(float2); }
inline size_t smem_precode(int U, int Bl, int K, int zgroups) {
  return ((size_t)Bl * U + (size_t)zgroups * U * zs_rt(K)) * sizeof(float2);
}

// ---------------------------------------------------------------- profiling helpers
inline cudaEvent_t take_event(dp_ctx *c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

struct LaunchScope {
  dp_ctx *c;
  int kid;
  cudaStream_t st;
  cudaEvent_t a = nullptr, b = nullptr;
  LaunchScope(dp_ctx *c_, int kid_, cudaStream_t st_) : c(c_), kid(kid_), st(st_) {
    c->launches++;
    if (c->cfg.flags & DP_FLAG_PROFILE) {
      a = take_event(c);
      b = take_event(c);
      cudaEventRecord(a, st);
    }
  }
  ~LaunchScope() {
    if (a) {
      cudaEventRecord(b, st);
      c->prof.push_back({kid, a, b});
    }
  }
};

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and size (host overhead
// per frame matters when a rank's share of the frame is small, e.g. 8 GPUs)
template <typename Kern>
cudaError_t set_smem(Kern kern, size_t bytes) {
  static std::mutex mu;
  static std::unordered_map<const void *, size_t> done;
  std::lock_guard<std::mutex> g(mu);
  auto it = done.find((const void *)kern);
  if (it != done.end() && it->second >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) done[(const void *)kern] = bytes;
  return e;
}

// Launch with programmatic dependent launch (PDL): the kernel may be scheduled while
// its predecessor on the stream drains; every kernel starts with griddepcontrol.wait.
template <typename Kern, typename... KArgs>
cudaError_t launch_pdl(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t st, const KArgs &...args) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  static const bool use_pdl = getenv("DP_NO_PDL") == nullptr;
  cfg.attrs = attr;
  cfg.numAttrs = use_pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

// PDL launch with a thread-block cluster shape (cluster_x CTAs along x)
template <typename Kern, typename... KArgs>
cudaError_t launch_pdl_cluster(Kern kern, dim3 grid, dim3 block, size_t smem, int cluster_x, cudaStream_t st,
                               const KArgs &...args) {
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = cluster_x;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  static const bool use_pdl = getenv("DP_NO_PDL") == nullptr;
  cfg.attrs = use_pdl ? attr : attr + 1;
  cfg.numAttrs = use_pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

// ---------------------------------------------------------------- U / KC dispatch
template <template <int, int> class F, int U, typename... T>
int dispatch_kc(int K, T... args) {
  switch (kc_of(K)) {
    case 7: return F<U, 7>::run(args...);
    case 8: return F<U, 8>::run(args...);
    case 14: return F<U, 14>::run(args...);
    default: return F<U, 16>::run(args...);
  }
}
template <template <int, int> class F, typename... T>
int dispatch(int U, int K, T... args) {
  switch (U) {
    case 4: return dispatch_kc<F, 4>(K, args...);
    case 8: return dispatch_kc<F, 8>(K, args...);
    case 16: return dispatch_kc<F, 16>(K, args...);
    case 32: return dispatch_kc<F, 32>(K, args...);
  }
  return fail(DP_ERR_UNSUPPORTED, "U=%d: kernels are instantiated for U in {4, 8, 16, 32}", U);
}

// ---------------------------------------------------------------- launchers (k_*.cu)
// Every launcher dispatches on the context's U and the args' K (a.K), counts the launch
// and brackets it with profiling events (LaunchScope).
// k_fd.cu: SIMT FD single pass (U <= 32, B_c >= U), MRT, the FD scalar finish kernels
int launch_fd_fused_any(dp_ctx *c, const Args &a, cudaStream_t st, int nw = 0,   // nw 0: c->fd_nw
                        int kid = DP_KERNEL_FUSED_FD);
int launch_mrt_u(dp_ctx *c, const Args &a, cudaStream_t st);
int launch_fd_finish(dp_ctx *c, const Args &a, cudaStream_t st);
int launch_fd_var_finish(dp_ctx *c, const Args &a, const dpk::VarRuns &vr, cudaStream_t st);
int launch_read_scalars(const float *fin, int n_sc, int which, float *dst, cudaStream_t st);
// k_fd_small.cu: FD small clusters B_c < U
int launch_fd_small(dp_ctx *c, const Args &a, cudaStream_t st);
// k_pd.cu: SIMT Gram (per chunk or summed) and precode
int launch_gram_any(dp_ctx *c, const Args &a, int nw, bool per_chunk, cudaStream_t st);
int launch_precode_any(dp_ctx *c, const Args &a, int nw, cudaStream_t st);
// k_solve.cu: regularised solve + beta + whitening (or W for prepare), apply-time whitening
int launch_solve_any(dp_ctx *c, const Args &a, cudaStream_t st);
int launch_whiten_any(dp_ctx *c, const Args &a, cudaStream_t st);
// k_tc.cu: tensor-core kernels (tcgen05 / TMEM / TMA)
int launch_gram_tc2_any(dp_ctx *c, const Args &b, cudaStream_t st);   // b.S % 32 == 0, U in {16, 32}
bool precode_tc2_ok(const dp_ctx *c, const Args &a);
int lsa_setup(dp_ctx *c);
int fd_rep(const dp_ctx *c, const Args &a, int nw);
void lsa_teardown(dp_ctx *c);
int launch_solve_lsa(dp_ctx *c, const Args &a, int sc0, cudaStream_t st);
int launch_precode_tc2(dp_ctx *c, const Args &a, cudaStream_t st);
bool fd_tc_ok(const dp_ctx *c, const Args &a);
int fd_fold_of(const dp_ctx *c, const Args &a);
int launch_fd_tc_kc(dp_ctx *c, const Args &a, cudaStream_t st);
// k_f64.cu: DP_FLAG_FP64 (fp64 Gram / solve / whitening / precode accumulation)
int launch_fd_f64(dp_ctx *c, const Args &a, cudaStream_t st);                 // FD, B_c >= U
int launch_gram_f64(dp_ctx *c, const Args &a, double2 *G64, cudaStream_t st);   // PD partial Gram
int launch_solve_f64(dp_ctx *c, const Args &a, const double2 *G64, double2 *z64, cudaStream_t st);
int launch_precode_f64(dp_ctx *c, const Args &a, const double2 *z64, cudaStream_t st);

}  // namespace dpi
