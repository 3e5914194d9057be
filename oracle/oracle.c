/*
 * oracle.c — fp64 CPU ORACLE for the decentralized Wiener-filter precoders of
 * arXiv 1804.10987 (Li, Jeon, Cavallaro, Studer).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (libdp.so + paper_1804_10987_b200/) never links, imports or
 * calls it, and shares no code, header, table or constant with it.
 *
 * Plain, slow, obviously-correct loops in double-precision complex arithmetic
 * (C99 `double complex`), one function per step of the paper.  No blocking, no
 * fusion, no reordering beyond what the paper's formulas state.  The only
 * parallelism is an OpenMP loop over independent OFDM subcarriers (P:264-266:
 * "Each OFDM subcarrier corresponds to an independent narrowband block-fading
 * downlink system"), which does not change any arithmetic.
 *
 * Citations: P:L = /root/reference/PAPER.md line L (LaTeX source); equation
 * numbers follow the paper's LaTeX numbering.
 *
 * Data layout (reading R2): the channel is passed as
 *     Ht[sc][b][u] = H^paper_{u,b}      (transpose, NOT conjugate transpose)
 * i.e. per subcarrier a B x U row-major array whose row b is antenna b.
 * Symbols s[sc][k][u], precoded output x[sc][k][b].
 *
 * Return codes: 0 ok, 1 numerical (matrix not Hermitian positive definite:
 * Cholesky pivot <= 0 or non-finite, or singular Gauss-Jordan pivot),
 * 2 invalid argument.
 *
 * Parity pins: every function here is pinned by tests/test_oracle.py (closed
 * forms, worked examples, identities, brute force); the one exception is
 * `oracle_rx_scale_fd` (reading R9, the paper is silent), marked
 * "parity unpinned" below and in DESIGN.md.
 */
#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;

#define OK 0
#define ERR_NUMERIC 1
#define ERR_ARG 2

/* ------------------------------------------------------------------------ */
/* Gram matrix G = H H^H  ("G_c = H_c H_c^H"; "G = H H^H").       */
/* With Ht[b][u] = H_{u,b}:  G[u][v] = sum_b H_{u,b} conj(H_{v,b})            */
/*                                   = sum_b Ht[b][u] conj(Ht[b][v]).          */
/* ------------------------------------------------------------------------ */
int oracle_gram(const cplx *Ht, int nb, int U, cplx *G)
{
    if (!Ht || !G || nb <= 0 || U <= 0) return ERR_ARG;
    for (int u = 0; u < U; ++u)
        for (int v = 0; v < U; ++v) {
            cplx acc = 0;
            for (int b = 0; b < nb; ++b)
                acc += Ht[(size_t)b * U + u] * conj(Ht[(size_t)b * U + v]);
            G[u * U + v] = acc;
        }
    return OK;
}

/* ------------------------------------------------------------------------ */
/* Cholesky factorisation A = L L^H of a Hermitian positive-definite matrix   */
/* (P:285 names "Cholesky decomposition"; A = G + kappa I is HPD for kappa>0).*/
/* Textbook column algorithm:                                                 */
/*   L[j][j] = sqrt(A[j][j] - sum_{m<j} |L[j][m]|^2)                          */
/*   L[i][j] = (A[i][j] - sum_{m<j} L[i][m] conj(L[j][m])) / L[j][j],  i > j  */
/* Only the lower triangle of A is read.  Returns ERR_NUMERIC when a pivot is */
/* not a finite positive number.                                              */
/* ------------------------------------------------------------------------ */
int oracle_cholesky(const cplx *A, int U, cplx *L)
{
    if (!A || !L || U <= 0) return ERR_ARG;
    for (int i = 0; i < U * U; ++i) L[i] = 0;
    for (int j = 0; j < U; ++j) {
        double d = creal(A[j * U + j]);
        for (int m = 0; m < j; ++m) {
            cplx l = L[j * U + m];
            d -= creal(l * conj(l));
        }
        if (!(d > 0.0) || !isfinite(d)) return ERR_NUMERIC;
        double ljj = sqrt(d);
        L[j * U + j] = ljj;
        for (int i = j + 1; i < U; ++i) {
            cplx acc = A[i * U + j];
            for (int m = 0; m < j; ++m) acc -= L[i * U + m] * conj(L[j * U + m]);
            L[i * U + j] = acc / ljj;
        }
    }
    return OK;
}

/* ------------------------------------------------------------------------ */
/* A^{-1} for HPD A via Cholesky, then forward and backward substitution      */
/* ("Cholesky decomposition, followed by ... forward and backward  */
/* substitution operations to obtain A^{-1}").  Column j of A^{-1} solves      */
/* L y = e_j (forward), L^H x = y (backward).                                 */
/* ------------------------------------------------------------------------ */
int oracle_hpd_inverse(const cplx *A, int U, cplx *Ainv)
{
    if (!A || !Ainv || U <= 0) return ERR_ARG;
    cplx *L = malloc(sizeof(cplx) * U * U);
    cplx *y = malloc(sizeof(cplx) * U);
    if (!L || !y) { free(L); free(y); return ERR_ARG; }
    int rc = oracle_cholesky(A, U, L);
    if (rc == OK) {
        for (int j = 0; j < U; ++j) {
            for (int i = 0; i < U; ++i) {           /* forward: L y = e_j */
                cplx acc = (i == j) ? 1.0 : 0.0;
                for (int m = 0; m < i; ++m) acc -= L[i * U + m] * y[m];
                y[i] = acc / L[i * U + i];
            }
            for (int i = U - 1; i >= 0; --i) {      /* backward: L^H x = y */
                cplx acc = y[i];
                for (int m = i + 1; m < U; ++m) acc -= conj(L[m * U + i]) * Ainv[m * U + j];
                Ainv[i * U + j] = acc / conj(L[i * U + i]);
            }
        }
    }
    free(L);
    free(y);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* Inverse of a general square matrix by Gauss-Jordan elimination with        */
/* partial pivoting.  Used ONLY for the B x B Theorem-1 route (Eq. 4) and the */
/* B_c < U branch of FD, so that the U x U Cholesky route is      */
/* checked against an independent algorithm.                                  */
/* ------------------------------------------------------------------------ */
int oracle_gauss_jordan_inverse(const cplx *M, int n, cplx *Minv)
{
    if (!M || !Minv || n <= 0) return ERR_ARG;
    cplx *a = malloc(sizeof(cplx) * n * n);
    if (!a) return ERR_ARG;
    memcpy(a, M, sizeof(cplx) * n * n);
    for (int i = 0; i < n * n; ++i) Minv[i] = 0;
    for (int i = 0; i < n; ++i) Minv[i * n + i] = 1;
    int rc = OK;
    for (int col = 0; col < n && rc == OK; ++col) {
        int piv = col;
        for (int r = col + 1; r < n; ++r)
            if (cabs(a[r * n + col]) > cabs(a[piv * n + col])) piv = r;
        cplx p = a[piv * n + col];
        if (!(cabs(p) > 0.0) || !isfinite(cabs(p))) { rc = ERR_NUMERIC; break; }
        if (piv != col)
            for (int c = 0; c < n; ++c) {
                cplx t = a[col * n + c]; a[col * n + c] = a[piv * n + c]; a[piv * n + c] = t;
                t = Minv[col * n + c]; Minv[col * n + c] = Minv[piv * n + c]; Minv[piv * n + c] = t;
            }
        for (int c = 0; c < n; ++c) { a[col * n + c] /= p; Minv[col * n + c] /= p; }
        for (int r = 0; r < n; ++r) {
            if (r == col) continue;
            cplx f = a[r * n + col];
            if (f == 0) continue;
            for (int c = 0; c < n; ++c) {
                a[r * n + c] -= f * a[col * n + c];
                Minv[r * n + c] -= f * Minv[col * n + c];
            }
        }
    }
    free(a);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* Lemma 1, Eq. (6):                                              */
/*   beta = sqrt( Es/rho2 * ( tr(A^{-1}) - kappa * ||A^{-1}||_F^2 ) )         */
/* Returns NaN when the radicand is not a finite positive number.             */
/* ------------------------------------------------------------------------ */
double oracle_beta_lemma1(const cplx *Ainv, int U, double kappa, double Es, double rho2)
{
    double tr = 0.0, fro = 0.0;
    for (int u = 0; u < U; ++u) tr += creal(Ainv[u * U + u]);
    for (int i = 0; i < U * U; ++i) fro += creal(Ainv[i] * conj(Ainv[i]));
    double r = Es / rho2 * (tr - kappa * fro);
    if (!(r > 0.0) || !isfinite(r)) return NAN;
    return sqrt(r);
}

/* ------------------------------------------------------------------------ */
/* Theorem 1, the plain B x B definition, one narrowband system:  */
/*   kappa = U N0 / rho2                                   (Eq. 5)            */
/*   Q = (H^H H + kappa I_B)^{-1} H^H                      (Eq. 4), B x U     */
/*   beta = sqrt( tr(Q^H Q) Es / rho2 )                    (Eq. 5)            */
/* Outputs Q[b][u] (B x U row-major) and beta.                               */
/* ------------------------------------------------------------------------ */
int oracle_wf_theorem1(const cplx *Ht, int B, int U, double N0, double rho2, double Es,
                       cplx *Q, double *beta)
{
    if (!Ht || !Q || !beta || B <= 0 || U <= 0 || !(rho2 > 0) || !(Es > 0) || N0 < 0) return ERR_ARG;
    double kappa = U * N0 / rho2;
    cplx *M = malloc(sizeof(cplx) * B * B);
    cplx *Minv = malloc(sizeof(cplx) * B * B);
    if (!M || !Minv) { free(M); free(Minv); return ERR_ARG; }
    /* (H^H H)[a][b] = sum_u conj(H_{u,a}) H_{u,b} = sum_u conj(Ht[a][u]) Ht[b][u] */
    for (int a = 0; a < B; ++a)
        for (int b = 0; b < B; ++b) {
            cplx acc = (a == b) ? kappa : 0.0;
            for (int u = 0; u < U; ++u) acc += conj(Ht[(size_t)a * U + u]) * Ht[(size_t)b * U + u];
            M[a * B + b] = acc;
        }
    int rc = oracle_gauss_jordan_inverse(M, B, Minv);
    if (rc == OK) {
        /* Q[a][u] = sum_b Minv[a][b] (H^H)_{b,u} = sum_b Minv[a][b] conj(Ht[b][u]) */
        double fro = 0.0;
        for (int a = 0; a < B; ++a)
            for (int u = 0; u < U; ++u) {
                cplx acc = 0;
                for (int b = 0; b < B; ++b) acc += Minv[a * B + b] * conj(Ht[(size_t)b * U + u]);
                Q[(size_t)a * U + u] = acc;
                fro += creal(acc * conj(acc));
            }
        double r = fro * Es / rho2;
        if (!(r > 0.0) || !isfinite(r)) rc = ERR_NUMERIC;
        *beta = sqrt(r);
    }
    free(M);
    free(Minv);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* Centralized WF precoder over an OFDM frame (Theorem 1, applied  */
/* per subcarrier):  x_k = Q s_k / beta  for k = 1..K.             */
/*   H  [n_sc][B][U], s [n_sc][K][U]  ->  x [n_sc][K][B], beta [n_sc]         */
/* ------------------------------------------------------------------------ */
int oracle_wf(const cplx *H, int n_sc, int B, int U, int K, const cplx *s,
              double N0, double rho2, double Es, cplx *x, double *beta)
{
    if (!H || !s || !x || !beta || n_sc <= 0 || B <= 0 || U <= 0 || K <= 0) return ERR_ARG;
    int rc = OK;
#pragma omp parallel for schedule(dynamic) reduction(max : rc)
    for (int w = 0; w < n_sc; ++w) {
        cplx *Q = malloc(sizeof(cplx) * B * U);
        double bw = NAN;
        int r = oracle_wf_theorem1(H + (size_t)w * B * U, B, U, N0, rho2, Es, Q, &bw);
        beta[w] = bw;
        for (int k = 0; k < K; ++k) {
            const cplx *sk = s + ((size_t)w * K + k) * U;
            cplx *xk = x + ((size_t)w * K + k) * B;
            for (int b = 0; b < B; ++b) {
                cplx acc = 0;
                for (int u = 0; u < U; ++u) acc += Q[(size_t)b * U + u] * sk[u];
                xk[b] = (r == OK) ? acc / bw : 0.0;
            }
        }
        free(Q);
        if (r > rc) rc = r;
    }
    return rc;
}

/* ------------------------------------------------------------------------ */
/* PD-WF (Sec. III-B), step by step, per subcarrier w:             */
/*   1. each cluster c:  G_c = H_c H_c^H                 */
/*   2. adder tree:      G = sum_c G_c, ascending c   (reading R15)    */
/*   3. whitening node:  kappa = U N0/rho2 (Eq. 5), A = G + kappa I_U */
/*                       A^{-1} by Cholesky + fwd/back substitution   */
/*                       beta by Lemma 1, Eq. (6)             */
/*                       z_k = A^{-1} s_k / beta             */
/*   4. each cluster c:  x_{c,k} = H_c^H z_k                 */
/* Cluster c owns antennas [c*B/C, (c+1)*B/C) (equal split, reading R14).     */
/* Outputs x [n_sc][K][B], beta [n_sc], optional z [n_sc][K][U] (may be NULL). */
/* A subcarrier whose A is not HPD gets x = 0, beta = NaN, and rc = 1.        */
/* ------------------------------------------------------------------------ */
int oracle_pd(const cplx *H, int n_sc, int B, int U, int K, int C, const cplx *s,
              double N0, double rho2, double Es, cplx *x, double *beta, cplx *z_out)
{
    if (!H || !s || !x || !beta || n_sc <= 0 || B <= 0 || U <= 0 || K <= 0 || C <= 0 || B % C)
        return ERR_ARG;
    if (N0 < 0 || !(rho2 > 0) || !(Es > 0)) return ERR_ARG;
    const int S = B / C;
    const double kappa = U * N0 / rho2;
    int rc = OK;
#pragma omp parallel for schedule(dynamic) reduction(max : rc)
    for (int w = 0; w < n_sc; ++w) {
        const cplx *Hw = H + (size_t)w * B * U;
        cplx *Gc = malloc(sizeof(cplx) * U * U);
        cplx *A = malloc(sizeof(cplx) * U * U);
        cplx *Ainv = malloc(sizeof(cplx) * U * U);
        cplx *z = malloc(sizeof(cplx) * U);
        /* steps 1-2 */
        for (int i = 0; i < U * U; ++i) A[i] = 0;
        for (int c = 0; c < C; ++c) {
            oracle_gram(Hw + (size_t)c * S * U, S, U, Gc);
            for (int i = 0; i < U * U; ++i) A[i] += Gc[i];
        }
        /* step 3 */
        for (int u = 0; u < U; ++u) A[u * U + u] += kappa;
        int r = oracle_hpd_inverse(A, U, Ainv);
        double bw = (r == OK) ? oracle_beta_lemma1(Ainv, U, kappa, Es, rho2) : NAN;
        if (r == OK && !isfinite(bw)) r = ERR_NUMERIC;
        beta[w] = bw;
        for (int k = 0; k < K; ++k) {
            const cplx *sk = s + ((size_t)w * K + k) * U;
            for (int u = 0; u < U; ++u) {
                cplx acc = 0;
                for (int v = 0; v < U; ++v) acc += Ainv[u * U + v] * sk[v];
                z[u] = (r == OK) ? acc / bw : 0.0;
            }
            if (z_out)
                for (int u = 0; u < U; ++u) z_out[((size_t)w * K + k) * U + u] = z[u];
            /* step 4: x_c = H_c^H z, i.e. x[b] = sum_u conj(H_{u,b}) z_u */
            cplx *xk = x + ((size_t)w * K + k) * B;
            for (int c = 0; c < C; ++c)
                for (int b = c * S; b < (c + 1) * S; ++b) {
                    cplx acc = 0;
                    for (int u = 0; u < U; ++u) acc += conj(Hw[(size_t)b * U + u]) * z[u];
                    xk[b] = acc;
                }
        }
        free(Gc); free(A); free(Ainv); free(z);
        if (r > rc) rc = r;
    }
    return rc;
}

/* ------------------------------------------------------------------------ */
/* FD-WF (Sec. III-C), step by step, per subcarrier w, cluster c:  */
/*   rho_c^2 = rho2 / C               */
/*   kappa_c = tau * U * N0 / rho_c^2                   (Eq. 9)    */
/*   Q_c = H_c^H (H_c H_c^H + kappa_c I_U)^{-1}         if B_c >= U   */
/*       = (H_c^H H_c + kappa_c I_{B_c})^{-1} H_c^H     if B_c <  U   */
/*   beta_c = sqrt( tr(Q_c^H Q_c) Es / rho_c^2 )               */
/*   x_{c,k} = Q_c s_k / beta_c               */
/* Outputs x [n_sc][K][B] and beta_c [n_sc][C].                               */
/* ------------------------------------------------------------------------ */
static int fd_cluster_Q(const cplx *Hc, int S, int U, double kappa_c, cplx *Q /*[S][U]*/)
{
    int rc;
    if (S >= U) {
        cplx *A = malloc(sizeof(cplx) * U * U);
        cplx *Ainv = malloc(sizeof(cplx) * U * U);
        oracle_gram(Hc, S, U, A);
        for (int u = 0; u < U; ++u) A[u * U + u] += kappa_c;
        rc = oracle_hpd_inverse(A, U, Ainv);
        /* Q[b][u] = sum_v (H_c^H)_{b,v} Ainv[v][u] = sum_v conj(Hc[b][v]) Ainv[v][u] */
        for (int b = 0; b < S; ++b)
            for (int u = 0; u < U; ++u) {
                cplx acc = 0;
                for (int v = 0; v < U; ++v) acc += conj(Hc[(size_t)b * U + v]) * Ainv[v * U + u];
                Q[(size_t)b * U + u] = acc;
            }
        free(A); free(Ainv);
    } else {
        cplx *M = malloc(sizeof(cplx) * S * S);
        cplx *Minv = malloc(sizeof(cplx) * S * S);
        for (int a = 0; a < S; ++a)
            for (int b = 0; b < S; ++b) {
                cplx acc = (a == b) ? kappa_c : 0.0;
                for (int u = 0; u < U; ++u) acc += conj(Hc[(size_t)a * U + u]) * Hc[(size_t)b * U + u];
                M[a * S + b] = acc;
            }
        rc = oracle_gauss_jordan_inverse(M, S, Minv);
        for (int a = 0; a < S; ++a)
            for (int u = 0; u < U; ++u) {
                cplx acc = 0;
                for (int b = 0; b < S; ++b) acc += Minv[a * S + b] * conj(Hc[(size_t)b * U + u]);
                Q[(size_t)a * U + u] = acc;
            }
        free(M); free(Minv);
    }
    return rc;
}

int oracle_fd(const cplx *H, int n_sc, int B, int U, int K, int C, const cplx *s,
              double N0, double rho2, double Es, double tau, cplx *x, double *beta_c)
{
    if (!H || !s || !x || !beta_c || n_sc <= 0 || B <= 0 || U <= 0 || K <= 0 || C <= 0 || B % C)
        return ERR_ARG;
    if (N0 < 0 || !(rho2 > 0) || !(Es > 0) || tau < 0) return ERR_ARG;
    const int S = B / C;
    const double rho_c2 = rho2 / C;
    const double kappa_c = tau * U * N0 / rho_c2;
    int rc = OK;
#pragma omp parallel for schedule(dynamic) reduction(max : rc)
    for (int w = 0; w < n_sc; ++w) {
        const cplx *Hw = H + (size_t)w * B * U;
        cplx *Q = malloc(sizeof(cplx) * S * U);
        for (int c = 0; c < C; ++c) {
            const cplx *Hc = Hw + (size_t)c * S * U;
            int r = fd_cluster_Q(Hc, S, U, kappa_c, Q);
            double fro = 0.0;
            for (int i = 0; i < S * U; ++i) fro += creal(Q[i] * conj(Q[i]));
            double rr = fro * Es / rho_c2;
            double bc = (r == OK && rr > 0.0 && isfinite(rr)) ? sqrt(rr) : NAN;
            if (r == OK && !isfinite(bc)) r = ERR_NUMERIC;
            beta_c[(size_t)w * C + c] = bc;
            for (int k = 0; k < K; ++k) {
                const cplx *sk = s + ((size_t)w * K + k) * U;
                cplx *xk = x + ((size_t)w * K + k) * B + (size_t)c * S;
                for (int b = 0; b < S; ++b) {
                    cplx acc = 0;
                    for (int u = 0; u < U; ++u) acc += Q[(size_t)b * U + u] * sk[u];
                    xk[b] = (r == OK) ? acc / bc : 0.0;
                }
            }
            if (r > rc) rc = r;
        }
        free(Q);
    }
    return rc;
}

/* ------------------------------------------------------------------------ */
/* FD-WF with unequal clusters: the same per-cluster precoder  */
/* as oracle_fd with the partition and the power split of the paper's        */
/* general statement instead of the equal one:                               */
/*   B_c = w_c B, sum_c B_c = B, cluster c = antennas sum_{c'<c} B_c' ...    */
/*                                                                     */
/*   rho_c^2 given, sum_c rho_c^2 = rho^2        */
/*   kappa_c = tau_c U N0 / rho_c^2                        (Eq. 9)     */
/*   Q_c by the branch of P:227-233 for each B_c; beta_c and x_c as in P:217. */
/* rho2_c[C] and tau_c[C] are per cluster; beta_c out [n_sc][C].             */
/* ------------------------------------------------------------------------ */
int oracle_fd_var(const cplx *H, int n_sc, int B, int U, int K, int C, const int *B_c,
                  const double *rho2_c, const double *tau_c, const cplx *s, double N0, double Es,
                  cplx *x, double *beta_c)
{
    if (!H || !s || !x || !beta_c || !B_c || !rho2_c || !tau_c || n_sc <= 0 || B <= 0 || U <= 0 ||
        K <= 0 || C <= 0 || N0 < 0 || !(Es > 0))
        return ERR_ARG;
    int tot = 0, Smax = 0;
    for (int c = 0; c < C; ++c) {
        if (B_c[c] <= 0 || !(rho2_c[c] > 0) || tau_c[c] < 0) return ERR_ARG;
        tot += B_c[c];
        if (B_c[c] > Smax) Smax = B_c[c];
    }
    if (tot != B) return ERR_ARG;
    int rc = OK;
#pragma omp parallel for schedule(dynamic) reduction(max : rc)
    for (int w = 0; w < n_sc; ++w) {
        const cplx *Hw = H + (size_t)w * B * U;
        cplx *Q = malloc(sizeof(cplx) * Smax * U);
        int off = 0;
        for (int c = 0; c < C; ++c) {
            const int S = B_c[c];
            const cplx *Hc = Hw + (size_t)off * U;
            const double kappa_c = tau_c[c] * U * N0 / rho2_c[c];
            int r = fd_cluster_Q(Hc, S, U, kappa_c, Q);
            double fro = 0.0;
            for (int i = 0; i < S * U; ++i) fro += creal(Q[i] * conj(Q[i]));
            double rr = fro * Es / rho2_c[c];
            double bc = (r == OK && rr > 0.0 && isfinite(rr)) ? sqrt(rr) : NAN;
            if (r == OK && !isfinite(bc)) r = ERR_NUMERIC;
            beta_c[(size_t)w * C + c] = bc;
            for (int k = 0; k < K; ++k) {
                const cplx *sk = s + ((size_t)w * K + k) * U;
                cplx *xk = x + ((size_t)w * K + k) * B + off;
                for (int b = 0; b < S; ++b) {
                    cplx acc = 0;
                    for (int u = 0; u < U; ++u) acc += Q[(size_t)b * U + u] * sk[u];
                    xk[b] = (r == OK) ? acc / bc : 0.0;
                }
            }
            if (r > rc) rc = r;
            off += S;
        }
        free(Q);
    }
    return rc;
}

/* Fully-distributed MRT with unequal clusters: Q_c = H_c^H, beta_c =        */
/* sqrt(Es ||H_c||_F^2 / rho_c^2) per cluster of size B_c.    */
int oracle_mrt_fd_var(const cplx *H, int n_sc, int B, int U, int K, int C, const int *B_c,
                      const double *rho2_c, const cplx *s, double Es, cplx *x, double *beta_c)
{
    if (!H || !s || !x || !beta_c || !B_c || !rho2_c || n_sc <= 0 || B <= 0 || U <= 0 || K <= 0 ||
        C <= 0 || !(Es > 0))
        return ERR_ARG;
    int tot = 0;
    for (int c = 0; c < C; ++c) {
        if (B_c[c] <= 0 || !(rho2_c[c] > 0)) return ERR_ARG;
        tot += B_c[c];
    }
    if (tot != B) return ERR_ARG;
    for (int w = 0; w < n_sc; ++w) {
        const cplx *Hw = H + (size_t)w * B * U;
        int off = 0;
        for (int c = 0; c < C; ++c) {
            const int S = B_c[c];
            const cplx *Hc = Hw + (size_t)off * U;
            double fro = 0.0;
            for (int i = 0; i < S * U; ++i) fro += creal(Hc[i] * conj(Hc[i]));
            const double bc = sqrt(Es * fro / rho2_c[c]);
            beta_c[(size_t)w * C + c] = bc;
            for (int k = 0; k < K; ++k) {
                const cplx *sk = s + ((size_t)w * K + k) * U;
                cplx *xk = x + ((size_t)w * K + k) * B + off;
                for (int b = 0; b < S; ++b) {
                    cplx acc = 0;
                    for (int u = 0; u < U; ++u) acc += conj(Hc[(size_t)b * U + u]) * sk[u];
                    xk[b] = bc > 0.0 ? acc / bc : 0.0;
                }
            }
            off += S;
        }
    }
    return OK;
}

/* ------------------------------------------------------------------------ */
/* Fully-distributed MRT, the baseline of Fig. 2: per   */
/* cluster the matched filter Q_c = H_c^H with the per-cluster power split    */
/* rho_c^2 = rho^2 / C and the normalisation of Eq. (5) applied to    */
/* the cluster, beta_c = sqrt(Es tr(Q_c^H Q_c) / rho_c^2)                    */
/* = sqrt(Es ||H_c||_F^2 / rho_c^2); x_c = Q_c s / beta_c.                   */
/* ------------------------------------------------------------------------ */
int oracle_mrt_fd(const cplx *H, int n_sc, int B, int U, int K, int C, const cplx *s,
                  double rho2, double Es, cplx *x, double *beta_c)
{
    if (!H || !s || !x || !beta_c || n_sc <= 0 || B <= 0 || U <= 0 || K <= 0 || C <= 0 || B % C)
        return ERR_ARG;
    if (!(rho2 > 0) || !(Es > 0)) return ERR_ARG;
    const int S = B / C;
    const double rho_c2 = rho2 / C;
    for (int w = 0; w < n_sc; ++w) {
        const cplx *Hw = H + (size_t)w * B * U;
        for (int c = 0; c < C; ++c) {
            const cplx *Hc = Hw + (size_t)c * S * U;
            double fro = 0.0;                                   /* tr(Q_c^H Q_c) = ||H_c||_F^2 */
            for (int i = 0; i < S * U; ++i) fro += creal(Hc[i] * conj(Hc[i]));
            const double bc = sqrt(Es * fro / rho_c2);
            beta_c[(size_t)w * C + c] = bc;
            for (int k = 0; k < K; ++k) {
                const cplx *sk = s + ((size_t)w * K + k) * U;
                cplx *xk = x + ((size_t)w * K + k) * B + (size_t)c * S;
                for (int b = 0; b < S; ++b) {                   /* (H_c^H s)_b = sum_u conj(H^paper_{u,b}) s_u */
                    cplx acc = 0;
                    for (int u = 0; u < U; ++u) acc += conj(Hc[(size_t)b * U + u]) * sk[u];
                    xk[b] = bc > 0.0 ? acc / bc : 0.0;
                }
            }
        }
    }
    return OK;
}

/* ------------------------------------------------------------------------ */
/* FD receive scale (reading R9 — parity unpinned: the paper does not state   */
/* which scalar a UE applies under FD-WF).  Each cluster's precoder is        */
/* designed for joint scaling by beta_c; in the ZF limit              */
/* H_c Q_c = I, so y = sum_c s / beta_c and the matching scalar is            */
/*     beta_rx = 1 / sum_c (1 / beta_c).                                      */
/* ------------------------------------------------------------------------ */
int oracle_rx_scale_fd(const double *beta_c, int n_sc, int C, double *beta_rx)
{
    if (!beta_c || !beta_rx || n_sc <= 0 || C <= 0) return ERR_ARG;
    for (int w = 0; w < n_sc; ++w) {
        double acc = 0.0;
        for (int c = 0; c < C; ++c) acc += 1.0 / beta_c[(size_t)w * C + c];
        beta_rx[w] = 1.0 / acc;
    }
    return OK;
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}
