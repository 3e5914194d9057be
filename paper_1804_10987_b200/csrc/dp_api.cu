// dp_api.cu — C-ABI of libdp.so (see include/dp.h for the contract).
//
// Host side of the B200-native decentralized WF precoders (arXiv 1804.10987):
// argument validation, workspace ownership, kernel dispatch over U, NCCL
// exchange steps (PD: Gram reduction P:280-281 and, in the paper's topology,
// z broadcast P:296; FD: s broadcast P:255/P:299 and a 2*n_sc scalar
// allreduce), host-pointer staging and kernel-level profiling.
#include "dp_internal.cuh"

namespace dpi {

thread_local std::string g_err;

int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}
void clear_error() { g_err.clear(); }

}  // namespace dpi

using namespace dpi;

namespace {

int drain_profile(dp_ctx *c) {
  for (auto &r : c->prof) {
    CK(cudaEventSynchronize(r.b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, r.a, r.b));
    c->prof_ms[r.kid] += ms;
    c->prof_n[r.kid] += 1;
    c->ev_pool.push_back(r.a);
    c->ev_pool.push_back(r.b);
  }
  c->prof.clear();
  return DP_OK;
}

// ---------------------------------------------------------------- helpers
int alloc(void **p, size_t bytes) {
  if (bytes == 0) bytes = 16;
  CK(cudaMalloc(p, bytes));
  CK(cudaMemset(*p, 0, bytes));
  return DP_OK;
}

bool is_device_ptr(const void *p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}
// cached per context (an address does not change between device and host memory under UVA)
bool is_device_ptr(dp_ctx *c, const void *p) {
  for (const auto &e : c->ptr_kind)
    if (e.first == p) return e.second;
  const bool d = is_device_ptr(p);
  if (c->ptr_kind.size() >= 64) c->ptr_kind.erase(c->ptr_kind.begin());
  c->ptr_kind.push_back({p, d});
  return d;
}

int validate_call(dp_ctx *c, const void *H, const void *s, double N0, double rho2, void *x) {
  if (!c) return fail(DP_ERR_INVALID, "ctx is NULL");
  if (!H || !x) return fail(DP_ERR_INVALID, "H_local and x_local must be non-NULL");
  const bool need_s = c->cfg.s_on_all_ranks || c->cfg.rank == 0;
  if (need_s && !s) return fail(DP_ERR_INVALID, "s must be non-NULL on this rank");
  if (!(N0 >= 0.0) || !std::isfinite(N0)) return fail(DP_ERR_INVALID, "N0 must be finite and >= 0 (got %g)", N0);
  if (!(rho2 > 0.0) || !std::isfinite(rho2)) return fail(DP_ERR_INVALID, "rho2 must be finite and > 0 (got %g)", rho2);
  return DP_OK;
}

// regulariser kappa and Lemma-1 coefficient Es / rho_x^2 of a call (fp32 for the default kernels,
// fp64 for the DP_FLAG_FP64 ones)
void set_params(Args &a, double kappa, double coef) {
  a.kappa = (float)kappa;
  a.coef = (float)coef;
  a.kappa64 = kappa;
  a.coef64 = coef;
}

Args base_args(dp_ctx *c) {
  Args a;
  memset(&a, 0, sizeof(a));
  a.n_sc = c->cfg.n_sc;
  a.Bl = c->Bl;
  a.K = c->cfg.K;
  a.beta = c->beta;
  a.pw = c->pw;
  a.bad = c->bad;
  a.fin = c->fin;
  a.fin_inv_beta = 1;
  return a;
}

// Stage host pointers into device buffers (H2D on st).  Returns device views.
int stage_in(dp_ctx *c, const dp_c32 *H, const dp_c32 *s, dp_c32 *x, cudaStream_t st, bool *host,
             const float2 **Hd, const float2 **sd, float2 **xd) {
  const bool hdev = is_device_ptr(c, H), xdev = is_device_ptr(c, x);
  const bool sdev = s ? is_device_ptr(c, s) : hdev;
  if (hdev != xdev || hdev != sdev)
    return fail(DP_ERR_INVALID, "H_local, s and x_local must all be device pointers or all host pointers");
  *host = !hdev;
  const size_t nH = (size_t)c->cfg.n_sc * c->Bl * c->cfg.U, nS = (size_t)c->cfg.n_sc * c->cfg.K * c->cfg.U,
               nX = (size_t)c->cfg.n_sc * c->cfg.K * c->Bl;
  if (hdev) {
    *Hd = reinterpret_cast<const float2 *>(H);
    *sd = reinterpret_cast<const float2 *>(s);
    *xd = reinterpret_cast<float2 *>(x);
    return DP_OK;
  }
  if (!c->h_dev) {
    RET(alloc((void **)&c->h_dev, nH * 8));
    RET(alloc((void **)&c->s_dev, nS * 8));
    RET(alloc((void **)&c->x_dev, nX * 8));
  }
  CK(cudaMemcpyAsync(c->h_dev, H, nH * 8, cudaMemcpyHostToDevice, st));
  if (s) CK(cudaMemcpyAsync(c->s_dev, s, nS * 8, cudaMemcpyHostToDevice, st));
  *Hd = c->h_dev;
  *sd = s ? c->s_dev : nullptr;
  *xd = c->x_dev;
  return DP_OK;
}

int stage_out(dp_ctx *c, bool host, dp_c32 *x, cudaStream_t st) {
  if (!host) return DP_OK;
  const size_t nX = (size_t)c->cfg.n_sc * c->cfg.K * c->Bl;
  CK(cudaMemcpyAsync(x, c->x_dev, nX * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return DP_OK;
}

// s broadcast from rank 0 ("the vector s is the only signal that must be broadcast")
int distribute_s(dp_ctx *c, const float2 *s, cudaStream_t st, const float2 **s_use, int K = 0) {
  if (!c->comm_on || c->cfg.s_on_all_ranks) {
    *s_use = s;
    return DP_OK;
  }
  const size_t n = (size_t)c->cfg.n_sc * (K > 0 ? K : c->cfg.K) * c->cfg.U * 2;
  if (c->cfg.rank == 0) {
    NK(ncclBroadcast(s, (void *)s, n, ncclFloat, 0, c->comm, st));
    LEDGER(c, DP_COMM_S_BCAST, n);
    *s_use = s;
  } else {
    NK(ncclBroadcast(nullptr, c->s_buf, n, ncclFloat, 0, c->comm, st));
    LEDGER(c, DP_COMM_S_BCAST, n);
    *s_use = c->s_buf;
  }
  return DP_OK;
}

int finish_call(dp_ctx *c, bool host, dp_c32 *x, cudaStream_t st) {
  RET(stage_out(c, host, x, st));
  if (c->cfg.flags & DP_FLAG_SYNC) {
    CK(cudaStreamSynchronize(st));
    int nb = 0;
    CK(cudaMemcpy(&nb, c->bad, sizeof(int), cudaMemcpyDeviceToHost));
    if (nb > 0) {
      CK(cudaMemset(c->bad, 0, sizeof(int)));
      return fail(DP_ERR_NUMERIC, "%d (subcarrier, cluster) problems had a non-HPD regularised Gram", nb);
    }
  }
  return DP_OK;
}

// FD frame on device pointers (everything after the host staging)
// Unequal clusters (dp_set_clusters): one launch per run of equal (B_c, rho_c^2 share, tau_c)
// -- the same kernels as the equal split, H / x offset to the run's first antenna with the
// rank's row stride Bl -- into per-run beta / power scratch, then fd_var_finish_kernel
// (beta_c in [sc][Cl] order, fin = {sum_c 1/beta_c, sum_c power_c}).  mrt: the MRT precoder.
// FD / MRT need cluster sizes: the equal split, or dp_set_clusters when C does not divide B
int need_split(const dp_ctx *c) {
  if (c->S == 0 && c->vruns.empty())
    return fail(DP_ERR_INVALID, "B=%d not divisible by C=%d: set the cluster sizes with dp_set_clusters", c->cfg.B,
                c->cfg.C);
  return DP_OK;
}
int fd_var_runs(dp_ctx *c, const float2 *Hd, const float2 *s_use, double N0, double rho2, float2 *xd, bool mrt,
                cudaStream_t st) {
  const dp_config &k = c->cfg;
  const bool fp64 = (k.flags & DP_FLAG_FP64) != 0;
  const size_t n = (size_t)k.n_sc * c->Cl;
  float *vb = c->vb;                                      // allocated by dp_set_clusters (no allocation here)
  dpk::VarRuns vr;
  memset(&vr, 0, sizeof(vr));
  vr.n = (int)c->vruns.size();
  vr.Cl = c->Cl;
  vr.vb = vb;
  vr.vp = vb + n;
  // the runs touch disjoint H rows, x columns and scratch: up to 3 run on the context's own streams
  // (created by dp_set_clusters) so their partial waves overlap; fork on an event, join before the finish
  static const bool serial = getenv("DP_VAR_SERIAL") != nullptr;
  const int nfork = (serial || !c->run_streams) ? 0 : std::min(vr.n, 3);
  if (nfork > 1) {
    CK(cudaEventRecord(c->ev_fork, st));
    for (int j = 0; j < nfork; ++j) CK(cudaStreamWaitEvent(c->st_run[j], c->ev_fork, 0));
  }
  int rc = DP_OK;
  for (int i = 0; i < vr.n && rc == DP_OK; ++i) {
    const cudaStream_t sr = nfork > 1 ? c->st_run[i % nfork] : st;
    const auto &r = c->vruns[i];
    const double rho_c2 = r.w * rho2;                     // rho_c^2 = w_c rho^2, sum_c w_c = 1
    Args a = base_args(c);
    a.H = Hd + (size_t)r.off * k.U;
    a.hrow_off = r.off;
    a.s = s_use;
    a.s_wait = c->comm_on && !k.s_on_all_ranks;
    a.x = xd + r.off;
    a.S = r.S;
    a.nchunks = r.len;
    a.nbeta = r.len;
    set_params(a, (r.tau * k.U * N0 / rho_c2), (k.Es / rho_c2));  // Eq. 9 with the cluster's tau_c, rho_c^2
    a.beta = vb + (size_t)k.n_sc * r.cl0;
    a.pw = vb + n + (size_t)k.n_sc * r.cl0;
    a.fold = 0;
    vr.cl0[i] = r.cl0;
    vr.len[i] = r.len;
    if (mrt) rc = launch_mrt_u(c, a, sr);
    else if (fp64 && r.S < k.U) rc = fail(DP_ERR_UNSUPPORTED, "DP_FLAG_FP64: FD branch B_c < U is fp32 only");
    else if (fp64) rc = launch_fd_f64(c, a, sr);
    else if (r.S < k.U) rc = launch_fd_small(c, a, sr);
    else if (fd_tc_ok(c, a)) rc = launch_fd_tc_kc(c, a, sr);
    else rc = launch_fd_fused_any(c, a, sr);
  }
  if (nfork > 1)                                          // join even after a failed launch
    for (int j = 0; j < nfork; ++j) {
      const cudaError_t e1 = cudaEventRecord(c->ev_join[j], c->st_run[j]);
      const cudaError_t e2 = e1 == cudaSuccess ? cudaStreamWaitEvent(st, c->ev_join[j], 0) : e1;
      if (e2 != cudaSuccess && rc == DP_OK) rc = fail(DP_ERR_CUDA, "fork/join: %s", cudaGetErrorString(e2));
    }
  if (rc == DP_OK) rc = launch_fd_var_finish(c, base_args(c), vr, st);
  return rc;
}

int precode_fd_dev(dp_ctx *c, const float2 *Hd, const float2 *sd, double N0, double rho2, float2 *xd,
                   cudaStream_t st) {
  const dp_config &k = c->cfg;
  RET(need_split(c));
  const float2 *s_use;
  RET(distribute_s(c, sd, st, &s_use));
  // FD parameters (Sec. III-C): rho_c^2 = rho^2/C, kappa_c = tau U N0 / rho_c^2 (Eq. 9)
  const double rho_c2 = rho2 / k.C;
  Args a = base_args(c);
  a.H = Hd;
  a.s = s_use;
  a.s_wait = c->comm_on && !k.s_on_all_ranks;             // s landed by ncclBroadcast on this stream
  a.x = xd;
  a.S = c->S;
  a.nchunks = c->Cl;
  set_params(a, (k.tau * k.U * N0 / rho_c2), (k.Es / rho_c2));
  a.nbeta = c->Cl;
  if (!c->vruns.empty()) {
    if ((k.flags & DP_FLAG_UNFUSED) && !(k.flags & DP_FLAG_FP64))
      return fail(DP_ERR_UNSUPPORTED, "DP_FLAG_UNFUSED with unequal clusters");
    RET(fd_var_runs(c, Hd, s_use, N0, rho2, xd, false, st));
  } else if (k.flags & DP_FLAG_FP64) {
    // accuracy option: the whole per-cluster chain with fp64 accumulation (f64.cuh)
    if (c->S < k.U) return fail(DP_ERR_UNSUPPORTED, "DP_FLAG_FP64: FD branch B_c < U is fp32 only");
    RET(launch_fd_f64(c, a, st));
    RET(launch_fd_finish(c, a, st));
  } else if (c->S < k.U) {
    // small clusters (B_c < U): B_c x B_c regularised Gram per cluster
    RET(launch_fd_small(c, a, st));
    RET(launch_fd_finish(c, a, st));
  } else if (k.flags & DP_FLAG_UNFUSED) {
    // (a) per-cluster Grams -> (b) solve+whiten per cluster -> (c) precode
    a.Gout = c->G;
    RET(launch_gram_any(c, a, c->fdu_nw, true, st));
    a.G = c->G;
    a.groups = c->Cl;
    a.zout = c->z;
    RET(launch_solve_any(c, a, st));
    a.zin = c->z;
    a.zgroups = c->Cl;
    a.chunks_per_zgroup = 1;
    RET(launch_precode_any(c, a, c->fdu_nw, st));
  } else {
    const bool tc = fd_tc_ok(c, a);
    // SIMT kernel: fold the scalars when every CTA holds whole subcarriers
    const int nsg = c->fd_nw * (32 / k.U);
    const int npb = nsg / fd_rep(c, a, c->fd_nw);          // problems per CTA of the SIMT kernel
    const bool simt_fold = !tc && npb <= 32 && npb % c->Cl == 0 && getenv("DP_NO_FOLD") == nullptr;
    if (tc) RET(launch_fd_tc_kc(c, a, st));
    else {
      a.fold = simt_fold ? 1 : 0;
      RET(launch_fd_fused_any(c, a, st));
      a.fold = 0;
    }
    if ((tc && fd_fold_of(c, a) == 0) || (!tc && !simt_fold))   // scalars not folded into the kernel
      RET(launch_fd_finish(c, a, st));
  }
  if (c->comm_on) {
    NK(ncclAllReduce(c->fin, c->fin, (size_t)k.n_sc * 2, ncclFloat, ncclSum, c->comm, st));
    LEDGER(c, DP_COMM_SCALARS, (size_t)k.n_sc * 2);
  }
  c->last_mode = 1;
  c->prepared = -1;                                       // G workspace reused
  return DP_OK;
}

// Fully-distributed MRT frame (Fig. 2 baseline) on device pointers
int precode_mrt_dev(dp_ctx *c, const float2 *Hd, const float2 *sd, double N0, double rho2, float2 *xd,
                    cudaStream_t st) {
  (void)N0;                                               // MRT ignores the noise level
  const dp_config &k = c->cfg;
  RET(need_split(c));
  const float2 *s_use;
  RET(distribute_s(c, sd, st, &s_use));
  Args a = base_args(c);
  a.H = Hd;
  a.s = s_use;
  a.x = xd;
  a.S = c->S;
  a.nchunks = c->Cl;
  set_params(a, 0.0, k.Es / (rho2 / k.C));                // Es / rho_c^2, rho_c^2 = rho^2 / C
  a.nbeta = c->Cl;
  if (!c->vruns.empty()) {
    RET(fd_var_runs(c, Hd, s_use, 0.0, rho2, xd, true, st));
  } else {
    RET(launch_mrt_u(c, a, st));
    RET(launch_fd_finish(c, a, st));
  }
  if (c->comm_on) {
    NK(ncclAllReduce(c->fin, c->fin, (size_t)k.n_sc * 2, ncclFloat, ncclSum, c->comm, st));
    LEDGER(c, DP_COMM_SCALARS, (size_t)k.n_sc * 2);
  }
  c->last_mode = 1;                                       // scalars laid out as FD's
  c->prepared = -1;
  return DP_OK;
}

// PD frame on device pointers (everything after the host staging)
int precode_pd_dev(dp_ctx *c, const float2 *Hd, const float2 *sd, double N0, double rho2, float2 *xd,
                   cudaStream_t st) {
  const dp_config &k = c->cfg;
  // PD parameters (Theorem 1, Eq. 5): kappa = U N0 / rho^2 ; beta via Lemma 1 with rho^2
  Args a = base_args(c);
  a.H = Hd;
  a.x = xd;
  a.s_wait = c->comm_on;                                   // s may come from a collective on the stream
  a.S = c->pd_chunk;
  a.nchunks = c->pd_nchunks;
  set_params(a, (k.U * N0 / rho2), (k.Es / rho2));
  a.groups = 1;
  a.nbeta = 1;
  a.fin_inv_beta = (k.rank == 0) ? 1 : 0;   // 1/beta contributed once to the scalar allreduce
  if (!c->comm_on && c->pdf_nw > 0 && !(k.flags & (DP_FLAG_UNFUSED | DP_FLAG_FP64))) {
    // one GPU holds every cluster: the adder tree G = sum_c G_c runs inside the per-subcarrier
    // Gram accumulation, and the whole PD chain -- Gram over all B antennas, A = G + kappa I, sweep,
    // Lemma-1 beta, z = A^{-1} s / beta, x_c = H_c^H z for every cluster -- is one single-pass kernel
    // (fd_fused_kernel with one "cluster" of all B antennas and PD's kappa / coefficient): H is read once
    a.S = c->Bl;
    a.nchunks = 1;
    a.fold = 1;                                           // fin[sc] = {1/beta, power} in-kernel
    a.s = sd;
    RET(launch_fd_fused_any(c, a, st, c->pdf_nw, DP_KERNEL_FUSED_PD));
    c->last_mode = 0;
    c->prepared = -1;
    return DP_OK;
  }
  if (k.flags & DP_FLAG_FP64) {
    // accuracy option (f64.cuh): fp64 partial Gram -> allreduce (ncclDouble) -> fp64 solve and
    // whitening on every rank -> fp64-accumulated local precode
    const float2 *s_use = sd;
    RET(distribute_s(c, sd, st, &s_use));
    a.s = s_use;
    RET(launch_gram_f64(c, a, c->G64, st));
    if (c->comm_on) {
      const size_t n64 = (size_t)k.n_sc * dpk::npacked(k.U) * 2;
      NK(ncclAllReduce(c->G64, c->G64, n64, ncclDouble, ncclSum, c->comm, st));
      LEDGER(c, DP_COMM_GRAM, 2 * n64);                   // fp32-sized units: one double = two floats
    }
    RET(launch_solve_f64(c, a, c->G64, c->z64, st));
    RET(launch_precode_f64(c, a, c->z64, st));
    if (c->comm_on) {
      NK(ncclAllReduce(c->fin, c->fin, (size_t)k.n_sc * 2, ncclFloat, ncclSum, c->comm, st));
      LEDGER(c, DP_COMM_SCALARS, (size_t)k.n_sc * 2);
    }
    c->last_mode = 0;
    c->prepared = -1;
    return DP_OK;
  }
  const bool topo_t1 = c->comm_on && k.pd_topology == DP_PD_REDUCE_BCAST;
  const bool topo_t3 = c->comm_on && k.pd_topology == DP_PD_SCATTER_GATHER;
  const bool topo_nvl = c->comm_on && k.pd_topology == DP_PD_NVLINK && c->lsa && !(k.flags & DP_FLAG_FP64);
  const float2 *s_use = sd;
  // s broadcast (allreduce / scatter-gather topologies): issued on the context's side stream so it
  // overlaps the Gram kernel (s is not needed before the whitening node); joined before the Gram
  // exchange, so two collectives of the one communicator never run concurrently
  const bool side = !topo_t1 && c->comm_on && !k.s_on_all_ranks && c->st_side;
  if (side) {
    CK(cudaEventRecord(c->ev_side0, st));
    CK(cudaStreamWaitEvent(c->st_side, c->ev_side0, 0));
    RET(distribute_s(c, sd, c->st_side, &s_use));
    CK(cudaEventRecord(c->ev_side1, c->st_side));
  } else if (!topo_t1) {
    RET(distribute_s(c, sd, st, &s_use));
  }
  a.s = s_use;
  // (a) Gram of this rank's antennas: first levels of the adder tree G = sum_c G_c
  const size_t nG = (size_t)k.n_sc * dpk::npacked(k.U) * 2;
  a.Gout = c->G;
  RET(launch_gram_any(c, a, c->pd_nw, false, st));
  if (side) CK(cudaStreamWaitEvent(st, c->ev_side1, 0));
  a.G = c->G;
  a.zout = c->z;
  if (topo_nvl) {
    // subcarrier-split whitening node with the exchange inside the kernel (exch_lsa.cuh): rank r sums
    // its block's partial Grams straight from the peers' windows, solves, and stores z and beta into
    // every peer's window -- the reduce-scatter and the all-gather of DP_PD_SCATTER_GATHER without a
    // collective between kernels
    const int nb = k.n_sc / k.world, sc0 = k.rank * nb;
    Args b = a;
    b.n_sc = nb;
    b.zout = c->z + (size_t)sc0 * k.K * k.U;
    b.beta = c->beta + sc0;
    RET(launch_solve_lsa(c, b, sc0, st));
    LEDGER(c, DP_COMM_GRAM, nG);                          // the same payload the collectives would move
    LEDGER(c, DP_COMM_Z_BCAST, (size_t)nb * k.K * k.U * 2 + (size_t)nb);
  } else if (topo_t3) {
    // subcarrier-split whitening node: rank r receives sum_c G_c of its n_sc/world subcarriers
    // (reduce-scatter, in place), solves and whitens them, and the z / beta blocks are
    // all-gathered: the solve scales with the GPU count instead of running on every rank
    const int nb = k.n_sc / k.world, sc0 = k.rank * nb;
    const size_t blkG = (size_t)nb * dpk::npacked(k.U) * 2, blkZ = (size_t)nb * k.K * k.U * 2;
    NK(ncclReduceScatter(c->G, c->G + (size_t)sc0 * dpk::npacked(k.U), blkG, ncclFloat, ncclSum, c->comm, st));
    LEDGER(c, DP_COMM_GRAM, nG);
    Args b = a;
    b.n_sc = nb;
    b.G = c->G + (size_t)sc0 * dpk::npacked(k.U);
    b.s = s_use + (size_t)sc0 * k.K * k.U;
    b.zout = c->z + (size_t)sc0 * k.K * k.U;
    b.beta = c->beta + sc0;
    RET(launch_solve_any(c, b, st));
    NK(ncclGroupStart());
    NK(ncclAllGather(c->z + (size_t)sc0 * k.K * k.U, c->z, blkZ, ncclFloat, c->comm, st));
    NK(ncclAllGather(c->beta + sc0, c->beta, (size_t)nb, ncclFloat, c->comm, st));
    NK(ncclGroupEnd());
    LEDGER(c, DP_COMM_Z_BCAST, blkZ + (size_t)nb);
  } else if (c->comm_on && !topo_t1) {
    // cross-rank adder tree on every rank; every rank whitens redundantly
    NK(ncclAllReduce(c->G, c->G, nG, ncclFloat, ncclSum, c->comm, st));
    LEDGER(c, DP_COMM_GRAM, nG);
  } else if (topo_t1) {
    // paper topology: reduce the Grams to the master GPU
    NK(ncclReduce(c->G, c->G, nG, ncclFloat, ncclSum, 0, c->comm, st));
    LEDGER(c, DP_COMM_GRAM, nG);
  }
  // (b) whitening node: A = G + kappa I, LDL^H, A^{-1}, beta (Lemma 1), z = A^{-1} s / beta
  if (!topo_t3 && !topo_nvl && (!topo_t1 || k.rank == 0)) RET(launch_solve_any(c, a, st));
  if (topo_t1) {
    // master broadcasts z and beta
    NK(ncclGroupStart());
    NK(ncclBroadcast(c->z, c->z, (size_t)k.n_sc * k.K * k.U * 2, ncclFloat, 0, c->comm, st));
    NK(ncclBroadcast(c->beta, c->beta, (size_t)k.n_sc, ncclFloat, 0, c->comm, st));
    NK(ncclGroupEnd());
    LEDGER(c, DP_COMM_Z_BCAST, (size_t)k.n_sc * k.K * k.U * 2 + (size_t)k.n_sc);
  }
  // (c) local precode x_c = H_c^H z on every rank
  a.zin = c->z;
  a.zgroups = 1;
  a.chunks_per_zgroup = c->pd_nchunks;
  if (precode_tc2_ok(c, a)) {
    RET(launch_precode_tc2(c, a, st));               // tensor-core precode, writes the scalars
  } else {
    RET(launch_precode_any(c, a, c->pd_nw, st));
  }
  // per-subcarrier scalars (written by the precode kernel): power summed over ranks
  if (c->comm_on) {
    NK(ncclAllReduce(c->fin, c->fin, (size_t)k.n_sc * 2, ncclFloat, ncclSum, c->comm, st));
    LEDGER(c, DP_COMM_SCALARS, (size_t)k.n_sc * 2);
  }
  c->last_mode = 0;
  c->prepared = -1;
  return DP_OK;
}

// Host-pointer frames, world = 1: the frame is cut into subcarrier chunks (subcarriers are
// independent problems) and H2D of chunk i+1, the kernels of chunk i and D2H of chunk i-1
// overlap on three streams (copy engines both ways + compute), instead of copy-all /
// compute / copy-all.  The scalar outputs (beta, fin) are written at the chunk's offset;
// the other workspace is reused chunk after chunk on the compute stream.
using DevFn = int (*)(dp_ctx *, const float2 *, const float2 *, double, double, float2 *, cudaStream_t);
int host_pipelined(dp_ctx *c, DevFn fn, int groups, const dp_c32 *H, const dp_c32 *s, double N0, double rho2,
                   dp_c32 *x, cudaStream_t st) {
  const dp_config k = c->cfg;
  static const int nch_env = getenv("DP_HOST_CHUNKS") ? atoi(getenv("DP_HOST_CHUNKS")) : 8;
  const int nch = std::max(1, std::min(std::min(nch_env, k.n_sc), (int)dp_ctx::HP_MAXCH));
  const bool async = (k.flags & DP_FLAG_HOST_ASYNC) != 0;
  const size_t rowH = (size_t)c->Bl * k.U, rowS = (size_t)k.K * k.U, rowX = (size_t)k.K * c->Bl;
  if (!c->h_dev) {
    RET(alloc((void **)&c->h_dev, (size_t)k.n_sc * rowH * 8));
    RET(alloc((void **)&c->s_dev, (size_t)k.n_sc * rowS * 8));
    RET(alloc((void **)&c->x_dev, (size_t)k.n_sc * rowX * 8));
  }
  if (!c->st_h2d) {
    CK(cudaStreamCreateWithFlags(&c->st_h2d, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->st_d2h, cudaStreamNonBlocking));
  }
  if (async && !c->hp_kdone[0])
    for (int i = 0; i < dp_ctx::HP_MAXCH; ++i) {
      CK(cudaEventCreateWithFlags(&c->hp_kdone[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->hp_d2h[i], cudaEventDisableTiming));
    }
  const bool chain = async && c->hp_nch == nch;            // previous async call with the same chunks
  cudaEvent_t ev_start = take_event(c);
  CK(cudaEventRecord(ev_start, st));                       // after the caller's prior work
  if (!chain) CK(cudaStreamWaitEvent(c->st_h2d, ev_start, 0));
  else CK(cudaStreamWaitEvent(st, c->hp_kdone[nch - 1], 0));   // the workspace: previous call's kernels done
                                                                // (a no-op when both calls use one stream)
  float *beta0 = c->beta, *fin0 = c->fin;
  int rc = DP_OK;
  std::vector<cudaEvent_t> evs;
  for (int i = 0; i < nch && rc == DP_OK; ++i) {
    const int sc0 = (int)((long long)k.n_sc * i / nch), sc1 = (int)((long long)k.n_sc * (i + 1) / nch);
    const int n = sc1 - sc0;
    cudaEvent_t ein = take_event(c), eout = take_event(c);
    evs.push_back(ein);
    evs.push_back(eout);
    if (chain) CK(cudaStreamWaitEvent(c->st_h2d, c->hp_kdone[i], 0));   // staging chunk i free
    CK(cudaMemcpyAsync(c->h_dev + sc0 * rowH, H + sc0 * rowH, n * rowH * 8, cudaMemcpyHostToDevice, c->st_h2d));
    CK(cudaMemcpyAsync(c->s_dev + sc0 * rowS, s + sc0 * rowS, n * rowS * 8, cudaMemcpyHostToDevice, c->st_h2d));
    CK(cudaEventRecord(ein, c->st_h2d));
    CK(cudaStreamWaitEvent(st, ein, 0));
    if (chain) CK(cudaStreamWaitEvent(st, c->hp_d2h[i], 0));   // x staging chunk i copied out
    c->cfg.n_sc = n;                                        // chunk view of the context
    c->beta = beta0 + (size_t)sc0 * groups;
    c->fin = fin0 + (size_t)sc0 * 2;
    rc = fn(c, c->h_dev + sc0 * rowH, c->s_dev + sc0 * rowS, N0, rho2, c->x_dev + sc0 * rowX, st);
    c->cfg.n_sc = k.n_sc;
    c->beta = beta0;
    c->fin = fin0;
    if (rc != DP_OK) break;
    CK(cudaEventRecord(eout, st));
    CK(cudaStreamWaitEvent(c->st_d2h, eout, 0));
    CK(cudaMemcpyAsync(x + sc0 * rowX, c->x_dev + sc0 * rowX, n * rowX * 8, cudaMemcpyDeviceToHost, c->st_d2h));
    if (async) {
      CK(cudaEventRecord(c->hp_kdone[i], st));
      CK(cudaEventRecord(c->hp_d2h[i], c->st_d2h));
    }
  }
  if (async) {                                             // syncing `stream` covers the last D2H
    c->hp_nch = rc == DP_OK ? nch : 0;
    if (rc == DP_OK) CK(cudaStreamWaitEvent(st, c->hp_d2h[nch - 1], 0));
  } else {
    c->hp_nch = 0;
    CK(cudaStreamSynchronize(c->st_d2h));
    CK(cudaStreamSynchronize(st));
  }
  for (auto e : evs) c->ev_pool.push_back(e);
  c->ev_pool.push_back(ev_start);
  return rc;
}

int precode_entry(dp_ctx *c, int mode, const dp_c32 *H, const dp_c32 *s, double N0, double rho2, dp_c32 *x,
                  void *stream) {
  g_err.clear();
  RET(validate_call(c, H, s, N0, rho2, x));
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaSetDevice(c->cfg.device));
  const bool fd = mode != 0;                              // 0 PD, 1 FD, 2 MRT (per-cluster scalars)
  DevFn fn = mode == 0 ? precode_pd_dev : mode == 1 ? precode_fd_dev : precode_mrt_dev;
  const bool hdev = is_device_ptr(c, H);
  static const bool no_pipe = getenv("DP_NO_HOST_PIPELINE") != nullptr;
  if (!hdev && !c->comm_on && !no_pipe && s && !is_device_ptr(c, x) && !is_device_ptr(c, s) && c->cfg.n_sc >= 16) {
    RET(host_pipelined(c, fn, fd ? c->Cl : 1, H, s, N0, rho2, x, st));
    return finish_call(c, false, x, st);                    // numeric check (DP_FLAG_SYNC); data already home
  }
  bool host;
  const float2 *Hd, *sd;
  float2 *xd;
  RET(stage_in(c, H, s, x, st, &host, &Hd, &sd, &xd));
  RET(fn(c, Hd, sd, N0, rho2, xd, st));
  return finish_call(c, host, x, st);
}
}  // namespace

// ====================================================================== C ABI
extern "C" {

const char *dp_last_error(void) { return g_err.c_str(); }

int dp_get_unique_id(void *out128) {
  if (!out128) return fail(DP_ERR_INVALID, "out128 is NULL");
  ncclUniqueId id;
  NK(ncclGetUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  memcpy(out128, &id, sizeof(id));
  return DP_OK;
}

int dp_init(const dp_config *cfg, dp_ctx **out) {
  g_err.clear();
  if (!out) return fail(DP_ERR_INVALID, "out is NULL");
  *out = nullptr;
  if (!cfg) return fail(DP_ERR_INVALID, "cfg is NULL");
  const dp_config &k = *cfg;
  if (k.n_sc <= 0 || k.B <= 0 || k.U <= 0 || k.K <= 0 || k.C <= 0)
    return fail(DP_ERR_INVALID, "dims must be positive (n_sc=%d B=%d U=%d K=%d C=%d)", k.n_sc, k.B, k.U, k.K, k.C);
  if (k.K > 64) return fail(DP_ERR_INVALID, "K=%d > 64", k.K);
  if (k.world <= 0 || k.rank < 0 || k.rank >= k.world) return fail(DP_ERR_INVALID, "rank %d / world %d", k.rank, k.world);
  if (k.B % k.world) return fail(DP_ERR_INVALID, "B=%d not divisible by world=%d", k.B, k.world);
  if (k.C % k.world) return fail(DP_ERR_INVALID, "C=%d not divisible by world=%d", k.C, k.world);
  if (!(k.Es > 0.0) || !std::isfinite(k.Es)) return fail(DP_ERR_INVALID, "Es must be > 0");
  if (!(k.tau >= 0.0) || !std::isfinite(k.tau)) return fail(DP_ERR_INVALID, "tau must be >= 0");
  if (k.pd_topology != DP_PD_ALLREDUCE && k.pd_topology != DP_PD_REDUCE_BCAST && k.pd_topology != DP_PD_SCATTER_GATHER &&
      k.pd_topology != DP_PD_NVLINK)
    return fail(DP_ERR_INVALID, "pd_topology %d", k.pd_topology);
  if ((k.pd_topology == DP_PD_SCATTER_GATHER || k.pd_topology == DP_PD_NVLINK) && k.n_sc % k.world)
    return fail(DP_ERR_INVALID, "pd_topology %d needs n_sc=%d divisible by world=%d", k.pd_topology, k.n_sc, k.world);
  if (k.pd_topology == DP_PD_NVLINK && k.U != 32)
    return fail(DP_ERR_UNSUPPORTED, "DP_PD_NVLINK: U=%d (the fused-exchange whitening kernel is U = 32)", k.U);
  if (k.U != 4 && k.U != 8 && k.U != 16 && k.U != 32)
    return fail(DP_ERR_UNSUPPORTED, "U=%d: supported U are 4, 8, 16, 32", k.U);
  // equal split S = B / C (P:157 with w_c = 1/C); 0 when C does not divide B: the sizes then come
  // from dp_set_clusters before any FD / MRT call
  const int S = (k.B % k.C) ? 0 : k.B / k.C;
  const bool comm_on = k.world > 1 || (k.flags & DP_FLAG_FORCE_COMM);
  if (comm_on && !k.nccl_id) return fail(DP_ERR_INVALID, "nccl_id is required when world > 1 or DP_FLAG_FORCE_COMM");

  CK(cudaSetDevice(k.device));
  dp_ctx *c = new dp_ctx();
  c->cfg = k;
  c->comm_on = comm_on;
  c->use_tc = getenv("DP_NO_TC") == nullptr;
  CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, k.device));
  c->Bl = k.B / k.world;
  c->Cl = k.C / k.world;
  c->S = S;
  // per-subcarrier PD kernels: split clusters into chunks (>= U rows) until the
  // CTA has >= 256 threads of SGs
  int chunk = S ? S : c->Bl;
  if (S && S < k.U) {                        // small clusters: PD chunks span several clusters (>= U rows)
    chunk = c->Bl;
    for (int m = S; m < c->Bl; m += S)
      if (m >= k.U && c->Bl % m == 0) { chunk = m; break; }
  }
  while ((c->Bl / chunk) * k.U < 256 && chunk % 16 == 0 && chunk / 2 >= k.U) chunk /= 2;
  c->pd_chunk = chunk;
  c->pd_nchunks = c->Bl / chunk;
  c->pd_nw = next_pow2((c->pd_nchunks * k.U + 31) / 32);
  c->fdu_nw = next_pow2((c->Cl * k.U + 31) / 32);
  // FD fused: 4 warps, fewer if smem would not fit
  c->fd_nw = 4;
  const int S_fd = S ? S : k.U;
  while (c->fd_nw > 1 && smem_fd_fused(k.U, S_fd, k.K, c->fd_nw) > 100 * 1024) c->fd_nw >>= 1;
  if (smem_fd_fused(k.U, S_fd, k.K, c->fd_nw) > 227 * 1024) {
    delete c;
    return fail(DP_ERR_UNSUPPORTED, "cluster tile S=%d x U=%d does not fit in shared memory", S, k.U);
  }
  // single-pass PD at world 1 (fd_fused_kernel with one problem of S = B per subcarrier, its rows split
  // over up to 32/U sub-groups, fd_rep): used for B U <= 1024 (cfg2; Fig. 2(d) B = 64, U = 16: 17.8 ->
  // 15.7 us per frame, p50 33.5 -> 26.8 us); at cfg3 (B U = 2048) it is 31.5 vs ~29 us per frame
  // and the three-kernel path stays.
  // DP_PD_FUSED=1 / 0 forces it on (any U < 32) / off.  0: not used
  c->pdf_nw = 0;
  {
    const char *ev = getenv("DP_PD_FUSED");
    const bool want = ev ? (atoi(ev) != 0) : (c->Bl * k.U <= 1024);
    if (!comm_on && k.U < 32 && want)
      for (int nw = 4; nw >= 1; nw >>= 1)
        if (smem_fd_fused(k.U, c->Bl, k.K, nw) <= (nw > 1 ? 100 * 1024 : 227 * 1024)) {
          c->pdf_nw = nw;
          break;
        }
  }
  if (c->pd_nw > 8) {
    delete c;
    return fail(DP_ERR_UNSUPPORTED, "B/world=%d antennas per rank need %d warps per subcarrier (max 8)", c->Bl, c->pd_nw);
  }
  const int NP = dpk::npacked(k.U);
  const size_t n_sc = k.n_sc;
  const size_t groups = std::max(c->Cl, 1);
  int rc = DP_OK;
  auto A = [&](void **p, size_t b) {
    if (rc == DP_OK) rc = alloc(p, b);
  };
  if (comm_on && !k.s_on_all_ranks) A((void **)&c->s_buf, n_sc * k.K * k.U * 8);
  const bool nvl = comm_on && k.pd_topology == DP_PD_NVLINK;   // G, z, beta: symmetric windows (lsa_setup)
  if (!nvl) {
    A((void **)&c->G, n_sc * groups * NP * 8);
    A((void **)&c->z, n_sc * groups * k.K * k.U * 8);
    A((void **)&c->beta, n_sc * groups * 4);
  }
  c->pw_len = n_sc * std::max<size_t>(std::max(c->pd_nchunks, c->Cl), 1);
  A((void **)&c->pw, c->pw_len * 4);
  A((void **)&c->fin, n_sc * 2 * 4);
  A((void **)&c->bad, 4);
  A((void **)&c->rd_buf, n_sc * 4);
  if (k.flags & DP_FLAG_FP64) {
    A((void **)&c->G64, n_sc * NP * 16);
    A((void **)&c->z64, n_sc * k.K * k.U * 16);
  }
  if (rc != DP_OK) {
    std::string e = g_err;
    dp_finalize(c);
    g_err = e;
    return rc;
  }
  if (comm_on) {
    if (cudaStreamCreateWithFlags(&c->st_side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_side0, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_side1, cudaEventDisableTiming) != cudaSuccess) {
      dp_finalize(c);
      return fail(DP_ERR_CUDA, "side stream / events for the s broadcast");
    }
    ncclUniqueId id;
    memcpy(&id, k.nccl_id, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&c->comm, k.world, id, k.rank);
    if (r != ncclSuccess) {
      dp_finalize(c);
      return fail(DP_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
    }
    if (k.pd_topology == DP_PD_NVLINK) {
      const int rl = lsa_setup(c);
      if (rl != DP_OK) {
        std::string e = g_err;
        dp_finalize(c);
        g_err = e;
        return rl;
      }
    }
  }
  *out = c;
  return DP_OK;
}

int dp_precode_fd(dp_ctx *c, const dp_c32 *H, const dp_c32 *s, double N0, double rho2, dp_c32 *x, void *stream) {
  return precode_entry(c, 1, H, s, N0, rho2, x, stream);
}
int dp_precode_pd(dp_ctx *c, const dp_c32 *H, const dp_c32 *s, double N0, double rho2, dp_c32 *x, void *stream) {
  return precode_entry(c, 0, H, s, N0, rho2, x, stream);
}
int dp_precode_mrt(dp_ctx *c, const dp_c32 *H, const dp_c32 *s, double N0, double rho2, dp_c32 *x, void *stream) {
  return precode_entry(c, 2, H, s, N0, rho2, x, stream);
}


int dp_read_scalars(dp_ctx *c, int which, float *dst, void *stream) {
  g_err.clear();
  if (!c || !dst) return fail(DP_ERR_INVALID, "ctx/dst is NULL");
  if (c->last_mode < 0) return fail(DP_ERR_INVALID, "no precode call yet");
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaSetDevice(c->cfg.device));
  const bool dev = is_device_ptr(dst);
  const int n_sc = c->cfg.n_sc;
  if (which == DP_SCALAR_BETA) {
    const size_t n = (size_t)n_sc * (c->last_mode == 1 ? c->Cl : 1);
    CK(cudaMemcpyAsync(dst, c->beta, n * 4, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
  } else if (which == DP_SCALAR_RX || which == DP_SCALAR_POWER) {
    float *d = dev ? dst : c->rd_buf;                     // host dst: through the context's staging buffer
    RET(launch_read_scalars(c->fin, n_sc, which, d, st));
    if (!dev) CK(cudaMemcpyAsync(dst, c->rd_buf, (size_t)n_sc * 4, cudaMemcpyDeviceToHost, st));
  } else {
    return fail(DP_ERR_INVALID, "unknown scalar %d", which);
  }
  if (!dev) CK(cudaStreamSynchronize(st));
  return DP_OK;
}

int dp_status(dp_ctx *c, int *n_bad) {
  g_err.clear();
  if (!c) return fail(DP_ERR_INVALID, "ctx is NULL");
  CK(cudaSetDevice(c->cfg.device));
  CK(cudaDeviceSynchronize());
  if (c->comm) {
    ncclResult_t async_err;
    NK(ncclCommGetAsyncError(c->comm, &async_err));
    if (async_err != ncclSuccess) return fail(DP_ERR_NCCL, "NCCL async error: %s", ncclGetErrorString(async_err));
  }
  int nb = 0;
  CK(cudaMemcpy(&nb, c->bad, sizeof(int), cudaMemcpyDeviceToHost));
  CK(cudaMemset(c->bad, 0, sizeof(int)));
  if (n_bad) *n_bad = nb;
  if (nb > 0) return fail(DP_ERR_NUMERIC, "%d (subcarrier, cluster) problems had a non-HPD regularised Gram", nb);
  return DP_OK;
}

int dp_profile_read(dp_ctx *c, double *ms, long long *launches, int reset) {
  g_err.clear();
  if (!c) return fail(DP_ERR_INVALID, "ctx is NULL");
  RET(drain_profile(c));
  for (int i = 0; i < DP_NUM_KERNELS; ++i) {
    if (ms) ms[i] = c->prof_ms[i];
    if (launches) launches[i] = c->prof_n[i];
    if (reset) {
      c->prof_ms[i] = 0;
      c->prof_n[i] = 0;
    }
  }
  return DP_OK;
}

long long dp_launch_count(dp_ctx *c) { return c ? c->launches : 0; }

int dp_comm_info(dp_ctx *c, int *nranks, int *nccl_version) {
  g_err.clear();
  if (!c) return fail(DP_ERR_INVALID, "ctx is NULL");
  if (nranks) {
    *nranks = 0;
    if (c->comm) NK(ncclCommCount(c->comm, nranks));
  }
  if (nccl_version) NK(ncclGetVersion(nccl_version));
  return DP_OK;
}

int dp_comm_ledger(dp_ctx *c, long long *floats, int reset) {
  g_err.clear();
  if (!c || !floats) return fail(DP_ERR_INVALID, "NULL argument");
  for (int i = 0; i < DP_NUM_COMM; ++i) {
    floats[i] = c->ledger[i];
    if (reset) c->ledger[i] = 0;
  }
  return DP_OK;
}

int dp_set_clusters(dp_ctx *c, const int *B_c, const double *power, const double *tau) {
  g_err.clear();
  if (!c) return fail(DP_ERR_INVALID, "ctx is NULL");
  const dp_config &k = c->cfg;
  const int C = k.C;
  std::vector<int> sz(C);
  std::vector<double> w(C), t(C);
  long long sum = 0;
  double wsum = 0.0;
  bool equal = true;
  if (!B_c && c->S == 0) return fail(DP_ERR_INVALID, "B=%d not divisible by C=%d: B_c is required", k.B, C);
  for (int i = 0; i < C; ++i) {
    sz[i] = B_c ? B_c[i] : c->S;
    w[i] = power ? power[i] : 1.0 / C;
    t[i] = tau ? tau[i] : k.tau;
    if (sz[i] <= 0) return fail(DP_ERR_INVALID, "B_c[%d]=%d must be positive", i, sz[i]);
    if (!(w[i] > 0.0) || !std::isfinite(w[i])) return fail(DP_ERR_INVALID, "power[%d] must be > 0", i);
    if (!(t[i] >= 0.0) || !std::isfinite(t[i])) return fail(DP_ERR_INVALID, "tau[%d] must be >= 0", i);
    if (sz[i] >= k.U && !(c->use_tc && k.U == 32 && sz[i] == 32 && k.K <= 16) &&
        smem_fd_fused(k.U, sz[i], k.K, c->fd_nw) > 227 * 1024)
      return fail(DP_ERR_UNSUPPORTED, "B_c[%d]=%d: the FD tile needs more than 227 KB of shared memory", i, sz[i]);
    sum += sz[i];
    wsum += w[i];
    equal = equal && sz[i] == c->S && std::fabs(w[i] - 1.0 / C) <= 1e-12 && t[i] == k.tau;
  }
  if (sum != k.B) return fail(DP_ERR_INVALID, "sum of B_c = %lld != B = %d", sum, k.B);
  if (std::fabs(wsum - 1.0) > 1e-9) return fail(DP_ERR_INVALID, "sum of power shares = %.12g != 1", wsum);
  const int c0 = k.rank * c->Cl;
  long long local = 0;
  for (int i = c0; i < c0 + c->Cl; ++i) local += sz[i];
  if (local != c->Bl)
    return fail(DP_ERR_INVALID, "rank %d: its clusters hold %lld antennas, need B/world = %d", k.rank, local, c->Bl);
  std::vector<dp_ctx::VarRun> runs;
  int off = 0;
  for (int i = c0; i < c0 + c->Cl; ++i) {
    if (!runs.empty()) {
      auto &r = runs.back();
      if (r.S == sz[i] && r.w == w[i] && r.tau == t[i]) {
        ++r.len;
        off += sz[i];
        continue;
      }
    }
    runs.push_back({i - c0, 1, sz[i], off, w[i], t[i]});
    off += sz[i];
  }
  if (!equal && (int)runs.size() > dpk::VAR_MAX_RUNS)
    return fail(DP_ERR_UNSUPPORTED, "%d runs of equal clusters > %d", (int)runs.size(), dpk::VAR_MAX_RUNS);
  if (!equal) {
    // run scratch and the fork/join streams are created here, once, so FD / MRT calls with
    // unequal clusters allocate nothing (dp.h: no allocation in precode calls)
    CK(cudaSetDevice(k.device));
    if (!c->vb) RET(alloc((void **)&c->vb, 2 * (size_t)k.n_sc * c->Cl * sizeof(float)));
    if (runs.size() > 1 && !c->run_streams) {
      for (int j = 0; j < 3; ++j) {
        if (!c->st_run[j]) CK(cudaStreamCreateWithFlags(&c->st_run[j], cudaStreamNonBlocking));
        if (!c->ev_join[j]) CK(cudaEventCreateWithFlags(&c->ev_join[j], cudaEventDisableTiming));
      }
      if (!c->ev_fork) CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
      c->run_streams = true;                              // only once every stream and event exists
    }
  }
  if (equal) {
    c->vruns.clear();
    c->vsizes.clear();
  } else {
    c->vruns = runs;
    c->vsizes = sz;
  }
  if (c->prepared == 1) c->prepared = -1;                 // a cached FD W no longer matches
  return DP_OK;
}

int dp_finalize(dp_ctx *c) {
  if (!c) return DP_OK;
  cudaSetDevice(c->cfg.device);
  cudaDeviceSynchronize();
  drain_profile(c);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  if (c->comm && (c->lsa || c->devcomm || c->win_g || c->win_z || c->win_b)) lsa_teardown(c);
  if (c->comm) ncclCommDestroy(c->comm);
  for (int i = 0; i < dp_ctx::HP_MAXCH; ++i) {
    if (c->hp_kdone[i]) cudaEventDestroy(c->hp_kdone[i]);
    if (c->hp_d2h[i]) cudaEventDestroy(c->hp_d2h[i]);
  }
  if (c->st_h2d) cudaStreamDestroy(c->st_h2d);
  if (c->st_d2h) cudaStreamDestroy(c->st_d2h);
  for (int j = 0; j < 3; ++j) {
    if (c->st_run[j]) cudaStreamDestroy(c->st_run[j]);
    if (c->ev_join[j]) cudaEventDestroy(c->ev_join[j]);
  }
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->st_side) cudaStreamDestroy(c->st_side);
  if (c->ev_side0) cudaEventDestroy(c->ev_side0);
  if (c->ev_side1) cudaEventDestroy(c->ev_side1);
  void *bufs[] = {c->s_buf, c->G, c->z, c->beta, c->pw, c->fin, c->bad, c->h_dev, c->s_dev, c->x_dev, c->vb, c->rd_buf, c->G64, c->z64};
  for (void *b : bufs)
    if (b) cudaFree(b);
  delete c;
  return DP_OK;
}

// ---------------------------------------------------------------- test-only step exports
int dp_debug_gram(dp_ctx *c, const dp_c32 *H, int per_cluster, dp_c32 *G, void *stream) {
  g_err.clear();
  if (!c || !H || !G) return fail(DP_ERR_INVALID, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  Args a = base_args(c);
  a.H = reinterpret_cast<const float2 *>(H);
  a.Gout = reinterpret_cast<float2 *>(G);
  if (per_cluster) {
    RET(need_split(c));
    if (!c->vruns.empty()) return fail(DP_ERR_UNSUPPORTED, "dp_debug_gram per cluster: unequal clusters");
    a.S = c->S;
    a.nchunks = c->Cl;
    if (fd_tc_ok(c, a)) RET(launch_fd_tc_kc(c, a, st));   // the FD path's own (tensor-core) Gram
    else RET(launch_gram_any(c, a, c->fdu_nw, true, st));
  } else {
    a.S = c->pd_chunk;
    a.nchunks = c->pd_nchunks;
    RET(launch_gram_any(c, a, c->pd_nw, false, st));
  }
  return DP_OK;
}

int dp_debug_solve(dp_ctx *c, const dp_c32 *G, int groups, const dp_c32 *s, double kappa, double rho_x2,
                   float *beta, dp_c32 *z, void *stream) {
  g_err.clear();
  if (!c || !G || !s || !beta || !z || groups <= 0) return fail(DP_ERR_INVALID, "bad argument");
  cudaStream_t st = (cudaStream_t)stream;
  Args a = base_args(c);
  a.G = reinterpret_cast<const float2 *>(G);
  a.s = reinterpret_cast<const float2 *>(s);
  a.groups = groups;
  a.zout = reinterpret_cast<float2 *>(z);
  a.beta = beta;
  set_params(a, kappa, c->cfg.Es / rho_x2);
  RET(launch_solve_any(c, a, st));
  return DP_OK;
}

// ---------------------------------------------------------------- prepare / apply (f2)
// Prepare from a Gram the caller already has (uplink reuse): G_packed holds this rank's
// partial Gram(s) in the packed layout of dp_debug_gram; it is copied into the context and the
// prepare continues as from the Gram kernel's output.
int prepare_from_gram(dp_ctx *c, int fd, const dp_c32 *G, double N0, double rho2, cudaStream_t st) {
  const dp_config &k = c->cfg;
  if (fd) RET(need_split(c));
  if (fd && !c->vruns.empty()) return fail(DP_ERR_UNSUPPORTED, "prepare/apply: unequal clusters run fused only");
  const int groups = fd ? c->Cl : 1;
  const size_t nG = (size_t)k.n_sc * groups * dpk::npacked(k.U);
  CK(cudaMemcpyAsync(c->G, G, nG * sizeof(float2), cudaMemcpyDeviceToDevice, st));
  Args a = base_args(c);
  if (fd) {
    const double rho_c2 = rho2 / k.C;
    set_params(a, (k.tau * k.U * N0 / rho_c2), (k.Es / rho_c2));  // Eq. 9
  } else {
    set_params(a, (k.U * N0 / rho2), (k.Es / rho2));  // Eq. 5
    if (c->comm_on) {
      NK(ncclAllReduce(c->G, c->G, nG * 2, ncclFloat, ncclSum, c->comm, st));
      LEDGER(c, DP_COMM_GRAM, nG * 2);
    }
  }
  a.groups = groups;
  a.nbeta = groups;
  a.G = c->G;
  a.Wout = c->G;
  a.s = nullptr;
  RET(launch_solve_any(c, a, st));
  c->prepared = fd;
  return DP_OK;
}

int dp_prepare_pd(dp_ctx *c, const dp_c32 *H, double N0, double rho2, void *stream) {
  g_err.clear();
  if (!c || !H) return fail(DP_ERR_INVALID, "ctx and H_local must be non-NULL");
  if (c->cfg.flags & DP_FLAG_FP64) return fail(DP_ERR_UNSUPPORTED, "prepare / apply: not with DP_FLAG_FP64");
  if (!is_device_ptr(H)) return fail(DP_ERR_INVALID, "dp_prepare_pd takes device pointers");
  if (!(N0 >= 0.0) || !std::isfinite(N0)) return fail(DP_ERR_INVALID, "N0 must be finite and >= 0");
  if (!(rho2 > 0.0) || !std::isfinite(rho2)) return fail(DP_ERR_INVALID, "rho2 must be finite and > 0");
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaSetDevice(c->cfg.device));
  const dp_config &k = c->cfg;
  Args a = base_args(c);
  a.H = reinterpret_cast<const float2 *>(H);
  a.S = c->pd_chunk;
  a.nchunks = c->pd_nchunks;
  set_params(a, (k.U * N0 / rho2), (k.Es / rho2));  // Eq. 5
  a.groups = 1;
  a.nbeta = 1;
  a.Gout = c->G;
  RET(launch_gram_any(c, a, c->pd_nw, false, st));   // G_c summed over local clusters
  if (c->comm_on) {                                       // every rank holds sum_c G_c
    NK(ncclAllReduce(c->G, c->G, (size_t)k.n_sc * dpk::npacked(k.U) * 2, ncclFloat, ncclSum, c->comm, st));
    LEDGER(c, DP_COMM_GRAM, (size_t)k.n_sc * dpk::npacked(k.U) * 2);
  }
  a.G = c->G;
  a.Wout = c->G;                                          // W = A^{-1}/beta in place of G
  a.s = nullptr;
  RET(launch_solve_any(c, a, st));
  c->prepared = 0;
  return DP_OK;
}

int dp_prepare_fd(dp_ctx *c, const dp_c32 *H, double N0, double rho2, void *stream) {
  g_err.clear();
  if (!c || !H) return fail(DP_ERR_INVALID, "ctx and H_local must be non-NULL");
  if (c->cfg.flags & DP_FLAG_FP64) return fail(DP_ERR_UNSUPPORTED, "prepare / apply: not with DP_FLAG_FP64");
  if (!is_device_ptr(H)) return fail(DP_ERR_INVALID, "dp_prepare_fd takes device pointers");
  if (!(N0 >= 0.0) || !std::isfinite(N0)) return fail(DP_ERR_INVALID, "N0 must be finite and >= 0");
  if (!(rho2 > 0.0) || !std::isfinite(rho2)) return fail(DP_ERR_INVALID, "rho2 must be finite and > 0");
  RET(need_split(c));
  if (c->S < c->cfg.U) return fail(DP_ERR_UNSUPPORTED, "prepare/apply: FD branch B_c < U runs fused only");
  if (!c->vruns.empty()) return fail(DP_ERR_UNSUPPORTED, "prepare/apply: unequal clusters run fused only");
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaSetDevice(c->cfg.device));
  const dp_config &k = c->cfg;
  const double rho_c2 = rho2 / k.C;
  Args a = base_args(c);
  a.H = reinterpret_cast<const float2 *>(H);
  a.S = c->S;
  a.nchunks = c->Cl;
  set_params(a, (k.tau * k.U * N0 / rho_c2), (k.Es / rho_c2));  // Eq. 9
  a.groups = c->Cl;
  a.nbeta = c->Cl;
  a.Gout = c->G;
  RET(launch_gram_any(c, a, c->fdu_nw, true, st));  // G_c per local cluster
  a.Gout = nullptr;
  a.G = c->G;
  a.Wout = c->G;
  a.s = nullptr;
  RET(launch_solve_any(c, a, st));
  c->prepared = 1;
  return DP_OK;
}

int dp_prepare_from_gram(dp_ctx *c, int fd, const dp_c32 *G_packed, double N0, double rho2, void *stream) {
  g_err.clear();
  if (!c || !G_packed) return fail(DP_ERR_INVALID, "ctx and G_packed must be non-NULL");
  if (c->cfg.flags & DP_FLAG_FP64) return fail(DP_ERR_UNSUPPORTED, "prepare / apply: not with DP_FLAG_FP64");
  if (!is_device_ptr(c, G_packed)) return fail(DP_ERR_INVALID, "dp_prepare_from_gram takes device pointers");
  if (!(N0 >= 0.0) || !std::isfinite(N0)) return fail(DP_ERR_INVALID, "N0 must be finite and >= 0");
  if (!(rho2 > 0.0) || !std::isfinite(rho2)) return fail(DP_ERR_INVALID, "rho2 must be finite and > 0");
  if (fd != 0 && fd != 1) return fail(DP_ERR_INVALID, "fd must be 0 (PD) or 1 (FD)");
  if (fd) RET(need_split(c));
  if (fd && c->S < c->cfg.U) return fail(DP_ERR_UNSUPPORTED, "prepare/apply: FD branch B_c < U runs fused only");
  CK(cudaSetDevice(c->cfg.device));
  return prepare_from_gram(c, fd, G_packed, N0, rho2, (cudaStream_t)stream);
}

int dp_apply(dp_ctx *c, const dp_c32 *H, const dp_c32 *s, int Ka, dp_c32 *x, void *stream) {
  g_err.clear();
  if (!c || !H || !x) return fail(DP_ERR_INVALID, "ctx, H_local and x_local must be non-NULL");
  if (c->prepared < 0) return fail(DP_ERR_INVALID, "no prepared channel (dp_prepare_pd / dp_prepare_fd first)");
  if (Ka < 1 || Ka > c->cfg.K) return fail(DP_ERR_INVALID, "Ka=%d must be in [1, K=%d]", Ka, c->cfg.K);
  const bool need_s = c->cfg.s_on_all_ranks || c->cfg.rank == 0;
  if (need_s && !s) return fail(DP_ERR_INVALID, "s must be non-NULL on this rank");
  if (!is_device_ptr(H) || !is_device_ptr(x) || (s && !is_device_ptr(s)))
    return fail(DP_ERR_INVALID, "dp_apply takes device pointers");
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaSetDevice(c->cfg.device));
  const dp_config &k = c->cfg;
  const float2 *s_use;
  RET(distribute_s(c, reinterpret_cast<const float2 *>(s), st, &s_use, Ka));
  const bool fd = c->prepared == 1;
  Args a = base_args(c);
  a.H = reinterpret_cast<const float2 *>(H);
  a.x = reinterpret_cast<float2 *>(x);
  a.s = s_use;
  a.K = Ka;
  a.G = c->G;                                             // cached W
  a.zout = c->z;
  a.groups = fd ? c->Cl : 1;
  a.nbeta = fd ? c->Cl : 1;
  a.fin_inv_beta = (fd || k.rank == 0) ? 1 : 0;
  RET(launch_whiten_any(c, a, st));                // z = W s
  a.zin = c->z;
  if (fd) {
    a.S = c->S;
    a.nchunks = c->Cl;
    a.zgroups = c->Cl;
    a.chunks_per_zgroup = 1;
    RET(launch_precode_any(c, a, c->fdu_nw, st));  // x_c = H_c^H z_c
  } else {
    a.S = c->pd_chunk;
    a.nchunks = c->pd_nchunks;
    a.zgroups = 1;
    a.chunks_per_zgroup = c->pd_nchunks;
    if (precode_tc2_ok(c, a)) RET(launch_precode_tc2(c, a, st));
    else RET(launch_precode_any(c, a, c->pd_nw, st));
  }
  if (c->comm_on) {
    NK(ncclAllReduce(c->fin, c->fin, (size_t)k.n_sc * 2, ncclFloat, ncclSum, c->comm, st));
    LEDGER(c, DP_COMM_SCALARS, (size_t)k.n_sc * 2);
  }
  c->last_mode = c->prepared;
  if (k.flags & DP_FLAG_SYNC) {
    CK(cudaStreamSynchronize(st));
    int nb = 0;
    CK(cudaMemcpy(&nb, c->bad, sizeof(int), cudaMemcpyDeviceToHost));
    if (nb > 0) {
      CK(cudaMemset(c->bad, 0, sizeof(int)));
      return fail(DP_ERR_NUMERIC, "%d (subcarrier, cluster) problems had a non-HPD regularised Gram", nb);
    }
  }
  return DP_OK;
}

}  // extern "C"
