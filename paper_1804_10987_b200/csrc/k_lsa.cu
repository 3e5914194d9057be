// k_lsa.cu — launcher of the PD whitening node with the cross-GPU exchange fused in
// (DP_PD_NVLINK, exch_lsa.cuh), and the symmetric-window setup it needs (NCCL 2.28 device API).
#include "dp_internal.cuh"
#include "exch_lsa.cuh"

namespace dpi {

// Symmetric windows over the packed Gram, z and beta workspaces (collective over the ranks: every
// rank calls this with the same sizes), and a device communicator with one LSA barrier per CTA
// of the solve grid.  The workspaces are allocated with ncclMemAlloc (VMM memory NCCL can map
// into every peer's address space).
int lsa_setup(dp_ctx *c) {
  const dp_config &k = c->cfg;
  // the same sizes as the cudaMalloc'd workspaces they replace (FD paths use them per cluster)
  const size_t n_sc = k.n_sc, NP = dpk::npacked(k.U), groups = std::max(c->Cl, 1);
  const size_t bytes[3] = {n_sc * groups * NP * 8, n_sc * groups * k.K * k.U * 8, n_sc * groups * 4};
  void **ptrs[3] = {(void **)&c->G, (void **)&c->z, (void **)&c->beta};
  ncclWindow_t *wins[3] = {&c->win_g, &c->win_z, &c->win_b};
  for (int i = 0; i < 3; ++i) {
    const size_t b = (bytes[i] + NCCL_WIN_REQUIRED_ALIGNMENT - 1) / NCCL_WIN_REQUIRED_ALIGNMENT * NCCL_WIN_REQUIRED_ALIGNMENT;
    NK(ncclMemAlloc(ptrs[i], b));
    CK(cudaMemset(*ptrs[i], 0, b));
    NK(ncclCommWindowRegister(c->comm, *ptrs[i], b, wins[i], NCCL_WIN_COLL_SYMMETRIC));
  }
  ncclDevCommRequirements reqs = {};
  reqs.lsaBarrierCount = (int)(n_sc / k.world);
  c->devcomm = new ncclDevComm;
  NK(ncclDevCommCreate(c->comm, &reqs, c->devcomm));
  int lsa_size = c->devcomm->lsaSize;
  if (lsa_size != k.world)
    return fail(DP_ERR_UNSUPPORTED, "DP_PD_NVLINK: %d of %d ranks are load/store-accessible (NVLink)", lsa_size, k.world);
  c->lsa = true;
  return DP_OK;
}

void lsa_teardown(dp_ctx *c) {
  if (c->devcomm) {
    ncclDevCommDestroy(c->comm, c->devcomm);
    delete c->devcomm;
    c->devcomm = nullptr;
  }
  ncclWindow_t wins[3] = {c->win_g, c->win_z, c->win_b};
  void *ptrs[3] = {c->G, c->z, c->beta};
  for (int i = 0; i < 3; ++i) {
    if (wins[i]) ncclCommWindowDeregister(c->comm, wins[i]);
    if (ptrs[i]) ncclMemFree(ptrs[i]);
  }
  c->win_g = c->win_z = c->win_b = nullptr;
  c->G = c->z = nullptr;
  c->beta = nullptr;
  c->lsa = false;
}

template <int KS>
static int launch_solve_lsa_t(dp_ctx *c, const Args &a, int sc0, cudaStream_t st) {
  const size_t sm = (size_t)dpk::smw_smem_elems(a.K, KS, 4) * sizeof(float2);
  auto kern = dpk::solve_lsa_kernel<KS>;
  CK(set_smem(kern, sm));
  dpk::LsaArgs x;
  x.dc = *c->devcomm;
  x.wg = c->win_g;
  x.wz = c->win_z;
  x.wb = c->win_b;
  x.sc0 = sc0;
  LaunchScope ls(c, DP_KERNEL_SOLVE, st);
  CK(launch_pdl(kern, dim3(a.n_sc), dim3(dpk::SMW_THREADS), sm, st, a, x));
  return DP_OK;
}
// a: n_sc = this rank's block, zout / beta at the block inside the windows; sc0 = first subcarrier
int launch_solve_lsa(dp_ctx *c, const Args &a, int sc0, cudaStream_t st) {
  // whitening in symbol chunks of at most 8 (register budget at 9 CTAs per SM, as solve_mw)
  switch (kc_of(a.K)) {
    case 7: return launch_solve_lsa_t<7>(c, a, sc0, st);
    case 8: return launch_solve_lsa_t<8>(c, a, sc0, st);
    case 14: return launch_solve_lsa_t<7>(c, a, sc0, st);
    default: return launch_solve_lsa_t<8>(c, a, sc0, st);
  }
}

}  // namespace dpi
