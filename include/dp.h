/*
 * dp.h — C-ABI of libdp.so: B200-native decentralized Wiener-filter (WF)
 * precoding, the data-parallel hot path of arXiv 1804.10987
 * ("Feedforward Architectures for Decentralized Precoding in Massive MU-MIMO
 * Systems", Li, Jeon, Cavallaro, Studer).
 *
 * Citations: P:L = PAPER.md line L (LaTeX source); equation numbers follow
 * the paper's LaTeX numbering.
 *
 * The calls follow the paper's problem statement
 *     x   = P  (s, H,   N0, rho^2)       (P:87-91,  centralized)
 *     x_c = P_c(s, H_c, N0, rho^2)       (Eq. 8, per cluster c)
 * evaluated for every OFDM subcarrier w and every OFDM symbol k of a frame
 * (N_sc independent narrowband systems, channel constant over K).
 *
 * Method (both precoders, per subcarrier):
 *   PD-WF (Sec. III-B):  G_c = H_c H_c^H ; G = sum_c G_c ;
 *       kappa = U N0/rho^2 (Eq. 5) ; A = G + kappa I_U ; Cholesky A = L L^H ;
 *       A^{-1} by forward/back substitution ;
 *       beta = sqrt(Es/rho^2 (tr A^{-1} - kappa ||A^{-1}||_F^2)) (Lemma 1, Eq. 6) ;
 *       z_k = A^{-1} s_k / beta ; x_{c,k} = H_c^H z_k.
 *   FD-WF (Sec. III-C):  per cluster, the same chain on H_c alone
 *       with rho_c^2 = rho^2/C and kappa_c = tau U N0/rho_c^2 (Eq. 9)
 *       (per-cluster rho_c^2 and tau_c through dp_set_clusters).
 *
 * ---------------------------------------------------------------- layouts
 * dp_c32 is an interleaved complex float (== cuComplex == torch.complex64).
 * Antennas are numbered b = 0..B-1; cluster c owns antennas [c*S, (c+1)*S),
 * S = B/C (equal split; dp_set_clusters sets unequal sizes B_c, cluster c
 * then starting at sum_{c' < c} B_c').  Rank r of `world` owns clusters
 * [r*C/world, (r+1)*C/world), i.e. the contiguous antenna block
 * [r*B/world, (r+1)*B/world) — "one GPU per cluster" with the
 * cluster count C decoupled from the GPU count.
 *   H_local  [n_sc][B/world][U]   H_local[w][b][u] = H^paper_{u, b0+b} of subcarrier w
 *                                 (transpose of the paper's U x B, NOT conjugated)
 *   s        [n_sc][K][U]         transmit symbols s_k of subcarrier w
 *   x_local  [n_sc][K][B/world]   precoded x_k restricted to this rank's antennas
 * Stacking the ranks' x_local along the last axis gives x[n_sc][K][B].
 *
 * ---------------------------------------------------------------- ownership
 * Pointers may be DEVICE pointers (the fast path; the caller owns them, the
 * call is asynchronous on `stream`) or HOST pointers (pinned or pageable; the
 * library stages them through context-owned device buffers with H2D / D2H
 * copies on `stream` and the call returns after the D2H copy completed;
 * with DP_FLAG_HOST_ASYNC at world == 1 it returns once the copies and kernels
 * are enqueued, see the flag).
 * All of H_local, s, x_local must be of the same kind.  `stream` is a
 * cudaStream_t passed as void* (NULL = legacy default stream).
 * The context owns every workspace (sized at dp_init; precode calls perform
 * no allocation on the device-pointer path and are CUDA-graph capturable when
 * world == 1) and, for world > 1, its own NCCL communicator.
 * A context is not thread-safe; distinct contexts are independent.
 *
 * ---------------------------------------------------------------- errors
 * Every call returns a dp_status code; dp_last_error() gives a thread-local
 * message for the last failing call.  Numerical failures (A not Hermitian
 * positive definite: Cholesky pivot <= 0 or non-finite, or beta radicand
 * <= 0 — e.g. N0 = 0 with a rank-deficient H_c, or non-finite input) are
 * detected on the device per (subcarrier, cluster); the affected outputs
 * are set to zero and counted.  They are reported by dp_status(), or
 * returned directly as DP_ERR_NUMERIC by the precode call when DP_FLAG_SYNC
 * is set (the call then synchronizes `stream`).
 */
#ifndef DP_H_
#define DP_H_

#if defined(DP_BUILD) && defined(__GNUC__)
#define DP_API __attribute__((visibility("default")))
#else
#define DP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* return codes */
#define DP_OK              0
#define DP_ERR_NUMERIC     1   /* A not HPD / beta undefined on >= 1 (subcarrier, cluster)      */
#define DP_ERR_INVALID     2   /* bad argument: NULL pointer, dims, N0 < 0, rho2 <= 0, ...      */
#define DP_ERR_CUDA        3   /* CUDA runtime error (message in dp_last_error)                 */
#define DP_ERR_NCCL        4   /* NCCL error                                                    */
#define DP_ERR_UNSUPPORTED 5   /* e.g. U not in {4,8,16,32}; a shape a kernel lacks (dp_last_error)  */

/* dp_config.flags */
#define DP_FLAG_SYNC        1  /* synchronize at the end of each precode call; return numeric errors */
#define DP_FLAG_UNFUSED     2  /* run the three-kernel path (a) Gram -> (b) solve+whiten -> (c) precode
                                  even where the single-pass fused kernel applies                      */
#define DP_FLAG_PROFILE     4  /* bracket every kernel launch with CUDA events (dp_profile_read)        */
#define DP_FLAG_FORCE_COMM  8  /* world == 1: still issue the NCCL collectives (tests the comm path);
                                  requires nccl_id                                                     */
#define DP_FLAG_HOST_ASYNC 32  /* host-pointer precode calls at world == 1 (the chunked H2D / kernels /
                                  D2H pipeline) return once the work is enqueued: x (and the scalars)
                                  are complete, and H, s, x may be reused by the host, only after
                                  `stream` has been synchronized.  Consecutive calls of the context then
                                  overlap: a call's H2D of chunk i waits only for the previous call's
                                  kernels on chunk i (not for the whole previous call), its kernels on
                                  chunk i for the previous D2H of chunk i; the H2D is not ordered after
                                  other work the caller queued on `stream`.  Device-pointer calls and
                                  world > 1 are unaffected.  A streaming mode for frame sequences
                                  (a new channel and symbol block every frame)            */
#define DP_FLAG_FP64       16  /* accuracy option (SURVEY.md §8(b) "DP_GRAM_FP64"): Gram,
                                  regularised solve, beta, whitening and precode accumulate in fp64
                                  (H, s, x stay complex64).  For square clusters (B_c = U) at high SNR
                                  or N0 = 0 (the ZF limit), where cond(G_c) of 1e4..1e9 puts the
                                  fp32 path above the 1e-4 bar.  FD needs B_c >= U (the B_c < U branch
                                  is well conditioned and stays fp32-only: DP_ERR_UNSUPPORTED); PD uses
                                  the allreduce exchange (ncclDouble) whatever pd_topology says;
                                  DP_FLAG_UNFUSED does not apply; prepare / apply: DP_ERR_UNSUPPORTED.
                                  Slower than the default path (fp64 FMAs run at half the fp32 rate
                                  and no tensor cores are used)                                       */

/* dp_config.pd_topology */
#define DP_PD_ALLREDUCE     0  /* allreduce packed G; every rank solves redundantly (default)          */
#define DP_PD_REDUCE_BCAST  1  /* paper's design: reduce G to rank 0, rank 0 solves
                                  and whitens, broadcast z                                             */
#define DP_PD_SCATTER_GATHER 2 /* reduce-scatter G over subcarrier blocks, each rank solves and whitens
                                  its n_sc/world subcarriers, all-gather z and beta (n_sc % world == 0)  */
#define DP_PD_NVLINK        3  /* DP_PD_SCATTER_GATHER's split with the exchange inside the whitening
                                  kernel: each rank sums its subcarriers' partial Grams straight from
                                  every peer's memory and stores z and beta into every peer's memory
                                  over NVLink load/store, with per-CTA cross-GPU barriers (NCCL 2.28
                                  device API: symmetric windows, LSA pointers and barriers; DESIGN.md
                                  §6).  U = 32, n_sc % world == 0, every rank load/store-accessible
                                  (dp_init: DP_ERR_UNSUPPORTED otherwise).  G, z and beta are then
                                  ncclMemAlloc'd symmetric windows                                    */

typedef struct { float re, im; } dp_c32;
typedef struct dp_ctx dp_ctx;                       /* opaque */

typedef struct {
    int n_sc;            /* subcarriers per frame, > 0                                  */
    int B;               /* BS antennas (all ranks), > 0                                        */
    int U;               /* UEs, 1 <= U <= 32                                                   */
    int K;               /* OFDM symbols per frame sharing one channel, 1..64           */
    int C;               /* antenna clusters, C % world == 0, B % world == 0.  B % C == 0 gives the
                            equal split B_c = B/C (any B_c >= 1: B_c < U takes the P:230 branch); otherwise FD / MRT
                            need dp_set_clusters first (unequal B_c)                     */
    int rank, world;     /* this process's rank and the number of GPUs (one process per GPU)    */
    int device;          /* CUDA device ordinal of this rank                                    */
    const void *nccl_id; /* 128-byte ncclUniqueId from dp_get_unique_id on rank 0, identical on
                            all ranks; NULL iff world == 1 (without DP_FLAG_FORCE_COMM)         */
    double Es;           /* average symbol energy of the constellation (reading R1), > 0 */
    double tau;          /* FD regularisation scale tau_c (Eq. 9; P:241 default 0.125), >= 0    */
    int pd_topology;     /* DP_PD_ALLREDUCE, DP_PD_REDUCE_BCAST, DP_PD_SCATTER_GATHER or DP_PD_NVLINK */
    int s_on_all_ranks;  /* 1: s is valid on every rank; 0: s is read on rank 0 only and
                            broadcast by the library ("s is the only signal that must be
                            broadcast")                                    */
    int flags;           /* DP_FLAG_*                                                           */
} dp_config;

/* scalar outputs readable after a precode call (dp_read_scalars `which`) */
#define DP_SCALAR_BETA   0  /* PD: beta^WF[n_sc] (Lemma 1).  FD: this rank's beta_c[n_sc][C/world] */
#define DP_SCALAR_RX     1  /* joint UE receive scale per subcarrier [n_sc]: PD beta^WF;
                               FD 1 / sum_c (1/beta_c) over ALL clusters (reading R9)              */
#define DP_SCALAR_POWER  2  /* sum_k ||x_k||^2 over ALL B antennas, per subcarrier [n_sc]
                               (check of the power constraint, Eq. 2)                     */

/* kernels reported by dp_profile_read (index into its arrays) */
#define DP_KERNEL_FUSED_FD      0   /* FD single pass: Gram + solve + whiten + precode per cluster     */
#define DP_KERNEL_GRAM          1   /* (a) batched Gram, packed Hermitian output                        */
#define DP_KERNEL_SOLVE         2   /* (b) regularise + Cholesky-type sweep + beta + whiten z           */
#define DP_KERNEL_PRECODE       3   /* (c) x_c = H_c^H z + power partials + per-subcarrier scalars      */
#define DP_KERNEL_FINISH        4   /* FD per-subcarrier scalar combination                             */
#define DP_KERNEL_FUSED_PD      5   /* PD single pass at world 1 (U < 32): Gram over all B antennas +
                                       solve + whiten + precode per subcarrier                          */
#define DP_NUM_KERNELS          6

/* exchange ledger kinds (dp_comm_ledger index): float payload elements this rank hands to */
#define DP_COMM_GRAM     0  /* PD: allreduce / reduce of the packed Hermitian Gram     */
#define DP_COMM_S_BCAST  1  /* broadcast of s from rank 0 (FD P:166; PD allreduce topo) */
#define DP_COMM_Z_BCAST  2  /* PD paper topology: broadcast of z and beta from rank 0           */
#define DP_COMM_SCALARS  3  /* allreduce of the [n_sc][2] per-subcarrier scalars (rx scale, power)    */
#define DP_NUM_COMM      4

/* Fill `out128` with a fresh ncclUniqueId (call on rank 0 only, then share the
 * 128 bytes with every rank, e.g. through torch.distributed). */
DP_API int dp_get_unique_id(void *out128);

/* Validate `cfg`, select `cfg->device`, allocate all workspace, and (world > 1)
 * create the NCCL communicator (collective: every rank must call it).
 * On success *out is a new context; on failure *out is NULL. */
DP_API int dp_init(const dp_config *cfg, dp_ctx **out);

/* PD-WF frame (Sec. III-B): x_local = H_local^H A^{-1} s / beta^WF for every
 * subcarrier and symbol, with A = sum over ALL clusters (all ranks) of
 * G_c + kappa I, kappa = U N0 / rho2.  Collective when world > 1.
 * N0 >= 0 (noise variance per complex entry), rho2 > 0 (power budget, Eq. 2). */
DP_API int dp_precode_pd(dp_ctx *ctx, const dp_c32 *H_local, const dp_c32 *s,
                  double N0, double rho2, dp_c32 *x_local, void *stream);

/* FD-WF frame (Sec. III-C): for every local cluster c, x_c = Q_c s / beta_c with
 * rho_c^2 = rho2 / C, kappa_c = tau U N0 / rho_c^2 (Eq. 9) and
 *   Q_c = H_c^H (H_c H_c^H + kappa_c I_U)^{-1}        if B_c >= U
 *   Q_c = (H_c^H H_c + kappa_c I_{B_c})^{-1} H_c^H    if B_c <  U (any 1 <= B_c < U;
 *         defined at N0 = 0 when H_c has full column rank)
 * beta_c^2 = Es tr(Q_c^H Q_c) / rho_c^2.  Only s (and 2 n_sc scalars) cross ranks. */
DP_API int dp_precode_fd(dp_ctx *ctx, const dp_c32 *H_local, const dp_c32 *s,
                  double N0, double rho2, dp_c32 *x_local, void *stream);

/* Unequal clusters, per-cluster power and tau ("B_c = w_c B", P:215 with its footnote,
 * Eq. 9 "tau_c").  Host arrays over ALL C clusters (global order), copied:
 *   B_c[C]    cluster sizes, sum = B; each rank's clusters (c in [rank C/world, (rank+1) C/world))
 *             must hold B/world antennas; B_c < U takes the small-cluster branch (any size);
 *             NULL = the equal split B/C;
 *   power[C]  shares w_c = rho_c^2 / rho2 > 0 with sum_c w_c = 1 (within 1e-9); NULL = 1/C each;
 *   tau[C]    tau_c >= 0; NULL = cfg.tau for every cluster.
 * Applies to dp_precode_fd and dp_precode_mrt (kappa_c = tau_c U N0 / rho_c^2, beta_c^2 =
 * Es tr(Q_c^H Q_c) / rho_c^2); PD does not depend on the partition.  The equal split with
 * equal shares and cfg.tau restores the default path.  DP_FLAG_UNFUSED, dp_prepare_fd and
 * dp_apply after dp_prepare_fd return DP_ERR_UNSUPPORTED while clusters are unequal.
 * Cluster c of a rank starts at local antenna row sum_{c' < c, same rank} B_c'.  The rank's
 * clusters run as maximal runs of equal (B_c, w_c, tau_c), one launch each (at most 64 runs).
 * Errors: DP_ERR_INVALID (sums, signs, NULL ctx), DP_ERR_UNSUPPORTED (sizes the kernels lack). */
DP_API int dp_set_clusters(dp_ctx *ctx, const int *B_c, const double *power, const double *tau);

/* Fully-distributed MRT (the baseline of Fig. 2): per cluster the
 * matched filter x_c = H_c^H s / beta_c with beta_c = sqrt(Es ||H_c||_F^2 / rho_c^2),
 * rho_c^2 = rho2 / C (Eq. 5 applied to the cluster).  N0 is accepted and ignored.
 * Same layouts, ownership and errors as dp_precode_fd.  DP_SCALAR_BETA then holds the effective
 * per-cluster scale beta_c U / ||H_c||_F^2 and DP_SCALAR_RX = 1 / sum_c (||H_c||_F^2 / (U beta_c)):
 * the joint UE scaling with the cluster array gain (H_c H_c^H ~ ||H_c||_F^2 / U I; R24). */
DP_API int dp_precode_mrt(dp_ctx *ctx, const dp_c32 *H_local, const dp_c32 *s,
                  double N0, double rho2, dp_c32 *x_local, void *stream);

/* Copy scalar output `which` (DP_SCALAR_*) of the last precode call into
 * `dst` (device or host float array of the documented length), ordered on
 * `stream`; a host `dst` is complete when the call returns. */
DP_API int dp_read_scalars(dp_ctx *ctx, int which, float *dst, void *stream);

/* Synchronize the context's work and report the number of (subcarrier,
 * cluster) problems whose regularised Gram was not HPD since the last call
 * (then reset it).  Returns DP_ERR_NUMERIC if that number is > 0. */
DP_API int dp_status(dp_ctx *ctx, int *n_bad);

/* Kernel-level profile (requires DP_FLAG_PROFILE): per DP_KERNEL_* the summed
 * device milliseconds and launch counts since the last reset.  Synchronizes. */
DP_API int dp_profile_read(dp_ctx *ctx, double *ms /*[DP_NUM_KERNELS]*/,
                    long long *launches /*[DP_NUM_KERNELS]*/, int reset);

/* Total kernels launched by this context since dp_init (all kinds). */
DP_API long long dp_launch_count(dp_ctx *ctx);

/* The context's communicator: *nranks = ranks of its NCCL communicator (0 when the context has
 * none: world == 1 without DP_FLAG_FORCE_COMM), *nccl_version = the linked NCCL's version code
 * (ncclGetVersion, e.g. 22809).  Either pointer may be NULL.  DP_ERR_INVALID for a NULL ctx. */
DP_API int dp_comm_info(dp_ctx *ctx, int *nranks, int *nccl_version);

/* Destroy the communicator and free all workspace.  Does not touch caller
 * buffers or streams.  NULL is accepted. */
DP_API int dp_finalize(dp_ctx *ctx);

/* Exchange ledger: floats[DP_NUM_COMM] = payload elements (fp32) this
 * rank passed to each kind of collective since the last reset (reset != 0 zeroes them).
 * Host-side counters: exact and free; compared with the paper's per-link closed forms in
 * paper_1804_10987_b200/ledger.py. */
DP_API int dp_comm_ledger(dp_ctx *ctx, long long *floats /*[DP_NUM_COMM]*/, int reset);

/* Thread-local message describing the last error ("" if none). */
DP_API const char *dp_last_error(void);

/* --------------------------------------------------------------------------
 * Test-only step exports (per-step parity).  Device pointers.
 * dp_debug_gram:  G_packed[n_sc][groups][U(U+1)/2] = upper triangle (u <= v,
 *   row-major) of sum_{b in group} h_b h_b^H, groups = C/world clusters
 *   (per_cluster = 1) or 1 (all local antennas).
 * dp_debug_solve: from G_packed [n_sc][groups][U(U+1)/2] and s: beta[n_sc][groups]
 *   and z[n_sc][groups][K][U] = (G + kappa I)^{-1} s_k / beta, with
 *   beta = sqrt(Es/rho_x2 (tr A^{-1} - kappa ||A^{-1}||_F^2)).
 * -------------------------------------------------------------------------- */
DP_API int dp_debug_gram(dp_ctx *ctx, const dp_c32 *H_local, int per_cluster, dp_c32 *G_packed, void *stream);
DP_API int dp_debug_solve(dp_ctx *ctx, const dp_c32 *G_packed, int groups, const dp_c32 *s,
                   double kappa, double rho_x2, float *beta, dp_c32 *z, void *stream);

/* --------------------------------------------------------------------------
 * Prepare / apply split.  The whitening matrix depends only on
 * the channel, so it is computed once per channel realisation and applied to
 * every OFDM symbol (A^{-1} and beta computed once, reused for
 * the K symbols).  Device pointers only; asynchronous on `stream`.
 * dp_prepare_pd / dp_prepare_fd: Gram (+ cross-rank sum for PD, collective when
 *   world > 1; every rank solves) -> A = G + kappa I -> W = A^{-1}/beta (Lemma 1),
 *   cached in the context as packed Hermitian W per (subcarrier, group) with beta.
 *   N0, rho2 as in dp_precode_*.  FD with B_c < U: DP_ERR_UNSUPPORTED (fused only).
 * dp_apply: x_local = H_local^H W s for Ka in [1, K] symbols s [n_sc][Ka][U]
 *   (z = W s, then the precode of the prepared mode); x_local [n_sc][Ka][B/world].
 *   dp_read_scalars afterwards gives beta, rx and the power of these Ka symbols.
 *   Equal (up to rounding order) to dp_precode_* on the same H, s, N0, rho2.
 *   DP_ERR_INVALID without a preceding prepare; any dp_precode_* call discards
 *   the prepared state (shared workspace).
 * -------------------------------------------------------------------------- */
DP_API int dp_prepare_pd(dp_ctx *ctx, const dp_c32 *H_local, double N0, double rho2, void *stream);
DP_API int dp_prepare_fd(dp_ctx *ctx, const dp_c32 *H_local, double N0, double rho2, void *stream);
DP_API int dp_apply(dp_ctx *ctx, const dp_c32 *H_local, const dp_c32 *s, int Ka, dp_c32 *x_local, void *stream);
/* Prepare from a Gram the caller already holds (uplink/downlink reuse of H_c H_c^H):
 * fd = 0: G_packed [n_sc][U(U+1)/2] = this rank's sum over its clusters (summed across ranks here);
 * fd = 1: G_packed [n_sc][C/world][U(U+1)/2] per local cluster; packed upper triangle, row-major
 * (u <= v), the layout of dp_debug_gram.  Then dp_apply as after dp_prepare_pd / dp_prepare_fd. */
DP_API int dp_prepare_from_gram(dp_ctx *ctx, int fd, const dp_c32 *G_packed, double N0, double rho2, void *stream);

/* --------------------------------------------------------------------------
 * Uncoded-BER harness (Sec. IV-D "Simulation Results", P:236-242,
 * Fig. 2).  Not part of the precoder: draws the paper's synthetic frames on the
 * device and scores precoded outputs at the UEs.  Device pointers, asynchronous
 * on `stream`; DP_ERR_INVALID for NULL pointers, dims <= 0, U > 32, B > 256,
 * K > 16, M not in {4, 16, 64, 256}, N0 < 0.
 *
 * dp_synth_frame: one frame from Philox4x32-10 keyed by `seed`, counter
 *   (index, stream, frame) — every value is a pure function of (seed, frame, index):
 *     H     [n_sc][B][U]   i.i.d. CN(0, 1) Rayleigh (layout as H_local)
 *     idx   [n_sc][K][U]   uniform M-QAM symbol indices (uint8), index =
 *                          (Gray label I << log2(M)/2) | Gray label Q
 *     s     [n_sc][K][U]   square Gray QAM points scaled to Es = 1
 *     noise [n_sc][K][U]   i.i.d. CN(0, N0); may be NULL (not drawn)
 * dp_receive_count: s_hat[sc][k][u] = rx[sc] (sum_b H[sc][b][u] x[sc][k][b]
 *   + noise[sc][k][u]) — Eq. (1) with the joint UE scaling (rx from
 *   dp_read_scalars(DP_SCALAR_RX)); per-axis nearest-level decisions; adds the
 *   number of bit errors against idx to *errors (a device counter the caller
 *   zeroes).  noise may be NULL (noiseless).
 * -------------------------------------------------------------------------- */
DP_API int dp_synth_frame(unsigned long long seed, unsigned long long frame, int n_sc, int B, int U, int K,
                          int M, double N0, dp_c32 *H, dp_c32 *s, unsigned char *idx, dp_c32 *noise,
                          void *stream);
DP_API int dp_receive_count(int n_sc, int B, int U, int K, int M, const dp_c32 *H, const dp_c32 *x,
                            const dp_c32 *noise, const float *rx, const unsigned char *idx,
                            unsigned long long *errors, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* DP_H_ */
