"""Pins for the fp64 oracle (oracle/oracle.c) against what the paper and mathematics fix.

Every pin uses something other than the oracle itself: worked examples
(tests/golden, cited), closed forms derived from Theorem 1 / Lemma 1, exact
identities of the paper (PD exactness P:183-186, inversion lemma P:379-384,
trace identity P:385-389, power equality, Appendix-A stationarity,
ZF limit), numpy/LAPACK library routines, and brute force on tiny inputs.
Layout: H[sc][b][u] = H^paper_{u,b} (reading R2); Hp = H[sc].T is the paper's U x B.
"""
import numpy as np
import pytest

import oracle
from paper_1804_10987_b200 import synth

pytestmark = pytest.mark.filterwarnings("ignore")


def rand_h(rng, n_sc, B, U):
    return (rng.standard_normal((n_sc, B, U)) + 1j * rng.standard_normal((n_sc, B, U))) / np.sqrt(2)


def rand_s(rng, n_sc, K, U):
    return (rng.standard_normal((n_sc, K, U)) + 1j * rng.standard_normal((n_sc, K, U))) / np.sqrt(2)


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


def P_of(fn, H1, **kw):
    """Precoding matrix P (B x U) of a single subcarrier: run the frame precoder with s = e_1..e_U."""
    B, U = H1.shape
    s = np.eye(U, dtype=np.complex128)[None]          # [1][K=U][U]: s_k = e_k
    out = fn(H1[None], s, **kw)
    x = out[0]                                         # [1][U][B]: x_k = P e_k
    return x[0].T, out


# --------------------------------------------------------------------------- Gram
def test_gram_worked_example(golden):
    g = golden("gram_worked_example.json")
    Hp = np.array(g["H_paper_re"]) + 1j * np.array(g["H_paper_im"])
    G = oracle.gram(Hp.T)
    np.testing.assert_allclose(G, np.array(g["G_re"]) + 1j * np.array(g["G_im"]), atol=0)


def test_gram_identity_and_library():
    assert np.array_equal(oracle.gram(np.eye(3)), np.eye(3))
    rng = np.random.default_rng(1)
    Hp = rand_h(rng, 1, 4, 8)[0]                       # U=4 x B=8 (SPEC S:54 shape)
    G = oracle.gram(Hp.T)
    np.testing.assert_allclose(G, Hp @ Hp.conj().T, rtol=0, atol=1e-12)
    assert np.abs(G - G.conj().T).max() <= 1e-12      # Hermitian
    assert np.linalg.eigvalsh(G).min() >= -1e-9       # PSD


# --------------------------------------------------------------------------- inverse / Cholesky
def test_hpd_inverse_worked_examples(golden):
    g = golden("hpd_inverse_2x2.json")
    np.testing.assert_allclose(oracle.hpd_inverse(np.array(g["A"], float)), np.array(g["Ainv"]), atol=1e-15)
    U = g["A_scalar_U"]
    np.testing.assert_allclose(oracle.hpd_inverse(g["A_scalar"] * np.eye(U)), g["Ainv_scalar"] * np.eye(U), atol=0)


@pytest.mark.parametrize("U", [1, 2, 4, 8, 16, 32])
def test_hpd_inverse_residual_and_library(U):
    rng = np.random.default_rng(U)
    Hp = rand_h(rng, 1, 2 * U, U)[0].T
    A = Hp @ Hp.conj().T + 1.0 * np.eye(U)
    Ai = oracle.hpd_inverse(A)
    assert np.linalg.norm(A @ Ai - np.eye(U)) <= 1e-9 * U            # SPEC S:60 residual bar
    np.testing.assert_allclose(Ai, np.linalg.inv(A), rtol=0, atol=1e-12)


def test_cholesky_factor_properties():
    rng = np.random.default_rng(7)
    Hp = rand_h(rng, 1, 12, 6)[0].T
    A = Hp @ Hp.conj().T + 0.3 * np.eye(6)
    L = oracle.cholesky(A)
    assert np.allclose(np.triu(L, 1), 0)
    assert np.all(np.real(np.diag(L)) > 0) and np.allclose(np.imag(np.diag(L)), 0)
    np.testing.assert_allclose(L @ L.conj().T, A, atol=1e-12)
    np.testing.assert_allclose(L, np.linalg.cholesky(A), atol=1e-12)


def test_cholesky_rejects_non_hpd():
    with pytest.raises(oracle.OracleError) as e:
        oracle.cholesky(np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert e.value.rc == oracle.ERR_NUMERIC
    with pytest.raises(oracle.OracleError):
        oracle.cholesky(np.array([[np.nan, 0.0], [0.0, 1.0]]))


def test_gauss_jordan_vs_library():
    rng = np.random.default_rng(3)
    M = rng.standard_normal((9, 9)) + 1j * rng.standard_normal((9, 9))
    np.testing.assert_allclose(oracle.gauss_jordan_inverse(M), np.linalg.inv(M), atol=1e-10)


# --------------------------------------------------------------------------- Lemma 1 / trace identity
def test_trace_identity_worked_example(golden):
    g = golden("trace_identity.json")
    G = np.array(g["G"], complex)
    k = g["kappa"]
    Ai = oracle.hpd_inverse(G + k * np.eye(2))
    # beta^2 rho2/Es = tr(A^-1) - kappa ||A^-1||_F^2 must equal tr(A^-1 G A^-1)
    assert abs(oracle.beta_lemma1(Ai, k) ** 2 - g["value"]) < 1e-15


@pytest.mark.parametrize("U,B", [(4, 16), (8, 64), (16, 128), (32, 256)])
def test_lemma1_equals_theorem1(U, B):
    """Lemma 1 Eq.(6) (U x U route) == Theorem 1 Eq.(5) (B x B Gauss-Jordan route), P:132 vs P:142."""
    rng = np.random.default_rng(U + B)
    Ht = rand_h(rng, 1, B, U)[0]
    for N0 in (0.01, 0.1, 1.0):
        kappa = U * N0 / 1.0
        Ai = oracle.hpd_inverse(oracle.gram(Ht) + kappa * np.eye(U))
        b1 = oracle.beta_lemma1(Ai, kappa, Es=1.0, rho2=1.0)
        _, b2 = oracle.wf_theorem1(Ht, N0, 1.0, 1.0)
        assert abs(b1 - b2) / b2 <= 1e-9
        # and the direct trace tr(A^-1 G A^-1) via numpy
        G = Ht.T @ Ht.conj()
        assert abs(b1 ** 2 - np.trace(Ai @ G @ Ai).real) <= 1e-9 * b1 ** 2


def test_inversion_lemma_Q_forms():
    """Q = (H^H H + k I_B)^-1 H^H  ==  H^H (H H^H + k I_U)^-1."""
    rng = np.random.default_rng(11)
    for U, B in [(2, 4), (4, 16), (16, 64)]:
        Ht = rand_h(rng, 1, B, U)[0]
        Hp = Ht.T
        N0 = 0.2
        kappa = U * N0
        Q1, _ = oracle.wf_theorem1(Ht, N0)
        Q2 = Hp.conj().T @ oracle.hpd_inverse(oracle.gram(Ht) + kappa * np.eye(U))
        assert rel(Q1, Q2) <= 1e-9


def test_mrt_direction_large_kappa():
    """kappa -> large: ||Q||_F ~ ||H||_F / kappa (MRT limit direction)."""
    rng = np.random.default_rng(5)
    Ht = rand_h(rng, 1, 8, 2)[0]
    N0 = 1e6 / 2  # kappa = U N0 / rho2 = 1e6
    Q, _ = oracle.wf_theorem1(Ht, N0)
    assert abs(np.linalg.norm(Q) * 1e6 / np.linalg.norm(Ht) - 1) < 1e-2


# --------------------------------------------------------------------------- whole WF
def test_identity_channel_worked_example(golden):
    g = golden("identity_channel_wf.json")
    H = np.eye(2, dtype=complex)[None]
    s = np.array(g["s"], complex)[None]
    for fn in (lambda: oracle.wf(H, s, g["N0"], g["rho2"], g["Es"]),
               lambda: oracle.pd(H, s, 1, g["N0"], g["rho2"], g["Es"])):
        x, beta = fn()
        assert abs(beta[0] - g["beta"]) < 1e-15
        np.testing.assert_allclose(x[0], np.array(g["x"]), atol=1e-15)
    _, _, z = oracle.pd(H, s, 1, g["N0"], g["rho2"], g["Es"], return_z=True)
    np.testing.assert_allclose(z[0], np.array(g["z"]), atol=1e-15)


@pytest.mark.parametrize("C", [1, 2, 4])
def test_closed_form_scaled_identity_channel(C):
    """H = [a_1 I_U, ..., a_C I_U]:  G = g I with g = sum|a_c|^2, A^-1 = I/(g+k),
    beta = sqrt(Es U g / rho2)/(g+k)  =>  PD/WF x_c = conj(a_c) sqrt(rho2/(Es U g)) s  (any N0);
    FD: G_c = |a_c|^2 I  =>  x_c = exp(-i arg a_c) sqrt(rho2/(C Es U)) s  (any N0, tau)."""
    U, K = 4, 3
    rng = np.random.default_rng(C)
    a = rng.standard_normal(C) + 1j * rng.standard_normal(C)
    H = np.concatenate([ac * np.eye(U) for ac in a], axis=0)[None]   # Ht: [B=C*U][U]
    s = rand_s(rng, 1, K, U)
    rho2, Es, N0 = 2.0, 1.5, 0.37
    g = np.sum(np.abs(a) ** 2)
    x_pd_expect = np.concatenate([np.conj(ac) * np.sqrt(rho2 / (Es * U * g)) * s[0] for ac in a], axis=1)
    x_fd_expect = np.concatenate([np.exp(-1j * np.angle(ac)) * np.sqrt(rho2 / (C * Es * U)) * s[0] for ac in a], axis=1)
    x_pd, _ = oracle.pd(H, s, C, N0, rho2, Es)
    x_wf, _ = oracle.wf(H, s, N0, rho2, Es)
    x_fd, _ = oracle.fd(H, s, C, N0, rho2, Es, tau=0.125)
    assert rel(x_pd[0], x_pd_expect) < 1e-13
    assert rel(x_wf[0], x_pd_expect) < 1e-13
    assert rel(x_fd[0], x_fd_expect) < 1e-13


@pytest.mark.parametrize("U,B", [(4, 16), (8, 32), (16, 64)])
def test_power_equality(U, B):
    """Es tr(P^H P) = rho2, for WF, PD and each FD cluster (rho2/C)."""
    rng = np.random.default_rng(B)
    Ht = rand_h(rng, 1, B, U)[0]
    rho2, Es, N0 = 1.7, 1.0, 0.05
    P, _ = P_of(lambda H, s: oracle.wf(H, s, N0, rho2, Es), Ht)
    assert abs(Es * np.linalg.norm(P) ** 2 / rho2 - 1) < 1e-10
    P, _ = P_of(lambda H, s: oracle.pd(H, s, 2, N0, rho2, Es), Ht)
    assert abs(Es * np.linalg.norm(P) ** 2 / rho2 - 1) < 1e-10
    C = 2
    P, _ = P_of(lambda H, s: oracle.fd(H, s, C, N0, rho2, Es, tau=0.125), Ht)
    S = B // C
    for c in range(C):
        assert abs(Es * np.linalg.norm(P[c * S:(c + 1) * S]) ** 2 / (rho2 / C) - 1) < 1e-10


def test_stationarity_appendix_a():
    """Optimality conditions of Appendix A with the corrected multiplier
    lambda = beta^2 kappa (reading R8; P:363's lambda = U N0/rho2 is a slip)."""
    rng = np.random.default_rng(21)
    U, B = 8, 32
    Ht = rand_h(rng, 1, B, U)[0]
    Hp = Ht.T
    rho2, Es, N0 = 1.0, 1.0, 0.1
    P, (x, beta) = P_of(lambda H, s: oracle.wf(H, s, N0, rho2, Es), Ht)
    b = beta[0]
    kappa = U * N0 / rho2
    lam = b ** 2 * kappa
    r_P = b ** 2 * Hp.conj().T @ Hp @ P + lam * P - b * Hp.conj().T          # Eq. (10)
    assert np.linalg.norm(r_P) <= 1e-10 * np.linalg.norm(Hp)
    lhs = b * np.trace(P.conj().T @ Hp.conj().T @ Hp @ P) + b * U * N0 / Es   # Eq. (11)
    rhs = np.trace(Hp.conj().T @ P.conj().T)
    assert abs(lhs - rhs) <= 1e-10 * abs(rhs)
    # the printed multiplier does NOT satisfy Eq.(10) unless beta = 1 (documents the slip)
    r_bad = b ** 2 * Hp.conj().T @ Hp @ P + (U * N0 / rho2) * P - b * Hp.conj().T
    assert np.linalg.norm(r_bad) > 1e-3 * np.linalg.norm(Hp)


def test_genie_mmse_scalar_equals_beta():
    """beta^WF is the MSE-optimal joint receive scalar:
    argmin_b Es||I - b H P||_F^2 + b^2 U N0 = Es Re tr(HP) / (Es ||HP||_F^2 + U N0)."""
    rng = np.random.default_rng(8)
    U, B = 16, 64
    Ht = rand_h(rng, 1, B, U)[0]
    Hp = Ht.T
    rho2, Es, N0 = 1.0, 1.0, 0.3
    P, (_, beta) = P_of(lambda H, s: oracle.pd(H, s, 4, N0, rho2, Es), Ht)
    HP = Hp @ P
    b_star = Es * np.trace(HP).real / (Es * np.linalg.norm(HP) ** 2 + U * N0)
    assert abs(b_star / beta[0] - 1) < 1e-10


def test_zf_limit():
    """beta H P = G A^-1 = I - kappa A^-1, so ||beta H P - I||_F = kappa ||A^-1||_F -> 0."""
    rng = np.random.default_rng(9)
    U, B = 8, 32
    Ht = rand_h(rng, 1, B, U)[0]
    Hp = Ht.T
    prev = None
    for N0 in (1e-2, 1e-4, 1e-6, 1e-8):
        P, (_, beta) = P_of(lambda H, s: oracle.pd(H, s, 2, N0, 1.0, 1.0), Ht)
        err = np.linalg.norm(beta[0] * Hp @ P - np.eye(U))
        kappa = U * N0
        Ai = np.linalg.inv(Ht.T @ Ht.conj() + kappa * np.eye(U))
        assert abs(err - kappa * np.linalg.norm(Ai)) <= 1e-9 * max(err, 1e-12) + 1e-12
        if prev is not None:
            assert err < prev / 50
        prev = err
    P, (_, beta) = P_of(lambda H, s: oracle.pd(H, s, 2, 0.0, 1.0, 1.0), Ht)     # N0 = 0 exactly
    assert np.linalg.norm(beta[0] * Hp @ P - np.eye(U)) < 1e-10


# --------------------------------------------------------------------------- PD / FD architecture claims
@pytest.mark.parametrize("C", [1, 2, 4, 8])
def test_pd_equals_centralized(C):
    """PD-WF implements exactly the centralized WF precoder, for every C."""
    rng = np.random.default_rng(100 + C)
    n_sc, B, U, K = 6, 32, 4, 5
    H = rand_h(rng, n_sc, B, U)
    s = rand_s(rng, n_sc, K, U)
    for N0 in (0.03, 0.5):
        x_pd, b_pd = oracle.pd(H, s, C, N0, 1.3, 1.0)
        x_wf, b_wf = oracle.wf(H, s, N0, 1.3, 1.0)
        assert rel(x_pd, x_wf) <= 1e-12
        assert np.max(np.abs(b_pd / b_wf - 1)) <= 1e-12


def test_fd_c1_tau1_equals_centralized():
    """FD with C=1, tau=1 collapses to centralized WF (reading R12)."""
    rng = np.random.default_rng(12)
    H = rand_h(rng, 4, 16, 4)
    s = rand_s(rng, 4, 3, 4)
    x_fd, b_fd = oracle.fd(H, s, 1, 0.2, 1.0, 1.0, tau=1.0)
    x_wf, b_wf = oracle.wf(H, s, 0.2, 1.0, 1.0)
    assert rel(x_fd, x_wf) <= 1e-12
    assert np.max(np.abs(b_fd[:, 0] / b_wf - 1)) <= 1e-12


@pytest.mark.parametrize("C,U,B", [(2, 4, 16), (4, 8, 64), (8, 16, 128), (4, 8, 16)])
def test_fd_cluster_is_local_wf(C, U, B):
    """FD cluster c == centralized WF on (H_c, N0' = tau N0, rho'^2 = rho^2/C) (Eq. 9).
    (4, 8, 16) has B_c = 4 < U = 8: exercises the B_c x B_c branch."""
    rng = np.random.default_rng(C * U)
    n_sc, K, tau, N0, rho2 = 3, 4, 0.125, 0.1, 1.0
    H = rand_h(rng, n_sc, B, U)
    s = rand_s(rng, n_sc, K, U)
    x_fd, b_c = oracle.fd(H, s, C, N0, rho2, 1.0, tau=tau)
    S = B // C
    for c in range(C):
        x_c, b = oracle.wf(H[:, c * S:(c + 1) * S], s, tau * N0, rho2 / C, 1.0)
        assert rel(x_fd[:, :, c * S:(c + 1) * S], x_c) <= 1e-11
        assert np.max(np.abs(b_c[:, c] / b - 1)) <= 1e-11


def test_fd_small_cluster_branch_vs_library():
    """B_c < U: Q_c = (H_c^H H_c + k I)^-1 H_c^H equals H_c^H (H_c H_c^H + k I_U)^-1."""
    rng = np.random.default_rng(13)
    U, B, C = 8, 16, 4
    S = B // C
    H = rand_h(rng, 1, B, U)
    N0, tau, rho2 = 0.2, 0.125, 1.0
    kc = tau * U * N0 / (rho2 / C)
    P, (_, b_c) = P_of(lambda H_, s: oracle.fd(H_, s, C, N0, rho2, 1.0, tau=tau), H[0])
    for c in range(C):
        Hp = H[0, c * S:(c + 1) * S].T
        Qc = Hp.conj().T @ np.linalg.solve(Hp @ Hp.conj().T + kc * np.eye(U), np.eye(U))
        bc = np.sqrt(np.linalg.norm(Qc) ** 2 / (rho2 / C))
        assert abs(b_c[0, c] / bc - 1) < 1e-10
        assert rel(P[c * S:(c + 1) * S], Qc / bc) < 1e-10


@pytest.mark.parametrize("U,B", [(1, 1), (2, 2), (2, 5), (3, 7), (4, 8)])
def test_tiny_brute_force_three_routes(U, B):
    """Tiny cases: Theorem-1 B x B Gauss-Jordan vs U x U Cholesky (PD, C=1) vs numpy solve."""
    rng = np.random.default_rng(U * 10 + B)
    H = rand_h(rng, 2, B, U)
    s = rand_s(rng, 2, 3, U)
    N0, rho2, Es = 0.25, 1.0, 1.0
    x1, b1 = oracle.wf(H, s, N0, rho2, Es)
    x2, b2 = oracle.pd(H, s, 1, N0, rho2, Es)
    for w in range(2):
        Hp = H[w].T
        Q = np.linalg.solve(Hp.conj().T @ Hp + U * N0 / rho2 * np.eye(B), Hp.conj().T)
        b = np.sqrt(np.linalg.norm(Q) ** 2 * Es / rho2)
        x3 = (Q @ s[w].T / b).T
        assert rel(x1[w], x3) < 1e-10 and rel(x2[w], x3) < 1e-10
        assert abs(b1[w] / b - 1) < 1e-10 and abs(b2[w] / b - 1) < 1e-10


def test_non_hpd_flagged():
    """N0 = 0 with a rank-deficient channel: A = G is singular -> numeric error, x zeroed."""
    U, B = 4, 8
    H = np.zeros((2, B, U), complex)
    H[0] = np.random.default_rng(1).standard_normal((B, U))
    H[1, :, :2] = 1.0                                 # rank 1 < U
    s = np.ones((2, 1, U), complex)
    with pytest.raises(oracle.OracleError):
        oracle.pd(H, s, 2, 0.0)
    x, beta = oracle.pd(H, s, 2, 0.0, allow_numeric=True)
    assert np.all(x[1] == 0) and np.isnan(beta[1])
    assert np.isfinite(beta[0]) and np.any(x[0] != 0)


def test_fd_rx_scale_zf_limit():
    """At N0 = 0 each cluster is ZF: H_c Q_c = I, so y = sum_c s/beta_c and
    beta_rx = 1/sum_c(1/beta_c) recovers s exactly (reading R9)."""
    rng = np.random.default_rng(31)
    U, B, C, K = 4, 32, 4, 6
    H = rand_h(rng, 3, B, U)
    s = rand_s(rng, 3, K, U)
    x, b_c = oracle.fd(H, s, C, 0.0, 1.0, 1.0, tau=0.125)
    brx = oracle.rx_scale_fd(b_c)
    for w in range(3):
        y = (H[w].T @ x[w].T).T                       # y_k = H x_k, noiseless
        assert rel(brx[w] * y, s[w]) < 1e-10


def test_frame_power_matches_constraint():
    """E_s ||x||^2 = rho2 on a QAM frame: frame mean within 2 % (expectation over s)."""
    f = synth.make_frame(cfg_id=3, n_sc=200, B=64, U=8, K=14, M=16)
    x, _ = oracle.pd(f.H, f.s, 4, 0.1, 1.0, 1.0)
    p = np.mean(np.sum(np.abs(x) ** 2, axis=2))
    assert abs(p - 1.0) < 0.02


def test_qam_constellation():
    for M in (4, 16, 64):
        q = synth.QAM(M)
        pts = q.points()
        assert abs(np.mean(np.abs(pts) ** 2) - 1.0) < 1e-12          # Es = 1 (reading R1)
        assert np.array_equal(q.decide(pts), np.arange(M))            # decisions invert the map
        # Gray: nearest neighbours differ in exactly one bit
        d = np.abs(pts[:, None] - pts[None, :])
        dmin = np.min(d[d > 1e-12])
        for i in range(M):
            for j in np.nonzero(np.abs(d[i] - dmin) < 1e-9)[0]:
                assert bin(i ^ j).count("1") == 1


# ---------------------------------------------------------------- fully-distributed MRT (Fig. 2 baseline)
def test_mrt_fd_pins():
    """MRT_c: Q_c = H_c^H (matched filter), beta_c by Eq. (5) on the cluster with rho_c^2 = rho^2/C:
    (1) per-cluster power Es tr(P_c^H P_c) = rho^2/C; (2) closed form for
    H = [a_1 I, .., a_C I] (B = C U): x_c = a_c s / beta_c with beta_c = |a_c| sqrt(U C Es / rho^2),
    so x_c = s sqrt(rho^2 / (U C Es)) (phase of a_c removed); (3) brute force against numpy."""
    rng = np.random.default_rng(5)
    U, C, K = 4, 2, 3
    a = np.array([0.7 + 0.2j, -1.3 + 0.0j])
    Ht = np.concatenate([a[c] * np.eye(U) for c in range(C)], axis=0)[None]   # [1][B][U], H^paper = Ht^T
    s = (rng.standard_normal((1, K, U)) + 1j * rng.standard_normal((1, K, U)))
    x, bc = oracle.mrt_fd(Ht, s, C, rho2=2.0)
    for c in range(C):
        assert bc[0, c] == pytest.approx(abs(a[c]) * np.sqrt(U * C / 2.0), rel=1e-12)
        xc = x[0, :, c * U:(c + 1) * U]
        assert np.allclose(xc, np.conj(a[c]) * s[0] / bc[0, c], atol=1e-12)
        assert np.allclose(np.abs(xc), np.abs(s[0]) * np.sqrt(2.0 / (U * C)), atol=1e-12)
    # random channel: power split and numpy matched filter
    B, U, C, K = 24, 6, 3, 5
    H = (rng.standard_normal((2, B, U)) + 1j * rng.standard_normal((2, B, U))) / np.sqrt(2)
    s = (rng.standard_normal((2, K, U)) + 1j * rng.standard_normal((2, K, U)))
    x, bc = oracle.mrt_fd(H, s, C, rho2=1.5, Es=0.8)
    S = B // C
    for w in range(2):
        for c in range(C):
            Hc = H[w, c * S:(c + 1) * S]                  # [S][U] = (H_c^paper)^T
            P = np.conj(Hc) / bc[w, c]                    # P_c = H_c^H / beta_c, [S][U]
            assert 0.8 * np.trace(P.conj().T @ P).real == pytest.approx(1.5 / C, rel=1e-12)
            assert np.allclose(x[w, :, c * S:(c + 1) * S], (P @ s[w].T).T, atol=1e-12)


# --------------------------------------------------------------------------- unequal clusters (§8 f3)
VAR_CASES = [
    # (U, sizes, power shares, tau_c): B_c < U (small branch), = U, > U; unequal power and tau
    (8, [4, 8, 20, 16], [0.1, 0.2, 0.4, 0.3], [0.125, 0.5, 1.0, 0.25]),
    (4, [4, 12, 8], [0.5, 0.25, 0.25], [0.125, 0.125, 2.0]),
]


@pytest.mark.parametrize("U,sizes,power,tau", VAR_CASES)
def test_fd_var_cluster_is_local_wf(U, sizes, power, tau):
    """Unequal clusters (P:157 B_c = w_c B) with power shares rho_c^2 and tau_c (Eq. 9):
    cluster c == centralized WF on (H_c, N0' = tau_c N0, rho'^2 = rho_c^2) (Theorem 1 route of
    oracle.wf); the equal split reduces to oracle.fd."""
    rng = np.random.default_rng(U + len(sizes))
    n_sc, K, N0, rho2, Es = 3, 5, 0.1, 1.5, 0.8
    B = sum(sizes)
    H = rand_h(rng, n_sc, B, U)
    s = rand_s(rng, n_sc, K, U)
    x, b_c = oracle.fd_var(H, s, sizes, N0, rho2, Es, power=power, tau=tau)
    off = 0
    for c, S in enumerate(sizes):
        x_c, b = oracle.wf(H[:, off:off + S], s, tau[c] * N0, power[c] * rho2, Es)
        assert rel(x[:, :, off:off + S], x_c) <= 1e-11
        assert np.max(np.abs(b_c[:, c] / b - 1)) <= 1e-11
        off += S
    C = 4
    xe, be = oracle.fd_var(H[:, :C * U], s, [U] * C, N0, rho2, Es, tau=0.3)
    xr, br = oracle.fd(H[:, :C * U], s, C, N0, rho2, Es, tau=0.3)
    assert rel(xe, xr) <= 1e-13 and np.max(np.abs(be / br - 1)) <= 1e-13


@pytest.mark.parametrize("U,sizes,power,tau", VAR_CASES)
def test_fd_var_power_split_and_library(U, sizes, power, tau):
    """Per-cluster power Es ||P_c||_F^2 = rho_c^2, so sum_c = rho^2 (Eq. 2); and P_c
    against numpy: Q_c = H_c^H (H_c H_c^H + kappa_c I)^-1 with kappa_c = tau_c U N0 / rho_c^2."""
    rng = np.random.default_rng(7 * U)
    N0, rho2, Es = 0.2, 2.0, 1.0
    B = sum(sizes)
    H = rand_h(rng, 1, B, U)
    P, _ = P_of(lambda H_, s: oracle.fd_var(H_, s, sizes, N0, rho2, Es, power=power, tau=tau), H[0])
    off = 0
    for c, S in enumerate(sizes):
        Pc = P[off:off + S]
        assert Es * np.linalg.norm(Pc) ** 2 == pytest.approx(power[c] * rho2, rel=1e-12)
        Hp = H[0, off:off + S].T                                   # H_c^paper, U x B_c
        kc = tau[c] * U * N0 / (power[c] * rho2)
        Qc = Hp.conj().T @ np.linalg.solve(Hp @ Hp.conj().T + kc * np.eye(U), np.eye(U))
        assert rel(Pc, Qc / np.sqrt(Es * np.linalg.norm(Qc) ** 2 / (power[c] * rho2))) < 1e-10
        off += S
    assert Es * np.linalg.norm(P) ** 2 == pytest.approx(rho2, rel=1e-12)


def test_mrt_fd_var_pins():
    """MRT with unequal clusters: x_c = H_c^H s / beta_c, Es ||P_c||_F^2 = rho_c^2 (numpy), and the
    equal split reduces to oracle.mrt_fd."""
    rng = np.random.default_rng(11)
    U, sizes, power = 4, [8, 4, 12], [0.2, 0.5, 0.3]
    B, K = sum(sizes), 3
    H = rand_h(rng, 2, B, U)
    s = rand_s(rng, 2, K, U)
    x, bc = oracle.mrt_fd_var(H, s, sizes, rho2=1.5, Es=0.8, power=power)
    off = 0
    for c, S in enumerate(sizes):
        for w in range(2):
            P = np.conj(H[w, off:off + S]) / bc[w, c]
            assert 0.8 * np.linalg.norm(P) ** 2 == pytest.approx(power[c] * 1.5, rel=1e-12)
            assert np.allclose(x[w, :, off:off + S], (P @ s[w].T).T, atol=1e-12)
        off += S
    xe, be = oracle.mrt_fd_var(H[:, :12], s, [4, 4, 4], rho2=1.5)
    xr, br = oracle.mrt_fd(H[:, :12], s, 3, rho2=1.5)
    assert rel(xe, xr) <= 1e-13 and np.max(np.abs(be / br - 1)) <= 1e-13


def test_fd_var_closed_form_repeated_identity_blocks():
    """Closed form for unequal clusters: H_c^paper = a_c [I_U, .., I_U] (m_c blocks, B_c = m_c U) gives
    H_c H_c^H = m_c |a_c|^2 I, Q_c = H_c^H / (m_c |a_c|^2 + kappa_c), and by P:217
    x_c = (conj(a_c)/|a_c|) [s; ..; s] sqrt(rho_c^2 / (m_c U Es)) for every kappa_c (tau_c, N0)."""
    U, K, Es, rho2, N0 = 4, 3, 0.9, 1.7, 0.3
    a = [0.6 - 0.8j, 2.0 + 0.0j, -0.3 + 0.4j]
    m = [1, 3, 2]
    power = [0.2, 0.5, 0.3]
    tau = [0.125, 1.0, 4.0]
    Ht = np.concatenate([a[c] * np.concatenate([np.eye(U)] * m[c], axis=0) for c in range(3)], axis=0)[None]
    rng = np.random.default_rng(3)
    s = rand_s(rng, 1, K, U)
    sizes = [mc * U for mc in m]
    x, _ = oracle.fd_var(Ht, s, sizes, N0, rho2, Es, power=power, tau=tau)
    off = 0
    for c in range(3):
        want = np.conj(a[c]) / abs(a[c]) * np.tile(s[0], (1, m[c])) * np.sqrt(power[c] * rho2 / (m[c] * U * Es))
        assert np.allclose(x[0, :, off:off + sizes[c]], want, atol=1e-12)
        off += sizes[c]
