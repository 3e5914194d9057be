"""fp64 CPU oracle for the decentralized WF precoders (arXiv 1804.10987).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` / ``--oracle-seconds`` legs and the N > 1
sampled parity check of ``bench.py`` may import this package.  The product (``paper_1804_10987_b200``, ``libdp.so``) never imports,
links or calls it and shares no code with it.

Thin ctypes wrapper around ``oracle.c`` (plain C99 double-complex loops).  The
wrapper only marshals numpy arrays; every arithmetic step lives in oracle.c and
cites the paper passage it follows.  Layouts (reading R2):
``H[sc][b][u]`` (= H^paper_{u,b}), ``s[sc][k][u]``, ``x[sc][k][b]``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, ERR_NUMERIC, ERR_ARG = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc (plain -O2, OpenMP over subcarriers)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-std=c99", "-O2", "-fPIC", "-shared", "-fopenmp", _SRC, "-o", _LIB, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


_lib = None


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        I = ctypes.c_int
        D = ctypes.c_double
        lib.oracle_gram.argtypes = [P, I, I, P]
        lib.oracle_cholesky.argtypes = [P, I, P]
        lib.oracle_hpd_inverse.argtypes = [P, I, P]
        lib.oracle_gauss_jordan_inverse.argtypes = [P, I, P]
        lib.oracle_beta_lemma1.argtypes = [P, I, D, D, D]
        lib.oracle_beta_lemma1.restype = D
        lib.oracle_wf_theorem1.argtypes = [P, I, I, D, D, D, P, P]
        lib.oracle_wf.argtypes = [P, I, I, I, I, P, D, D, D, P, P]
        lib.oracle_pd.argtypes = [P, I, I, I, I, I, P, D, D, D, P, P, P]
        lib.oracle_fd.argtypes = [P, I, I, I, I, I, P, D, D, D, D, P, P]
        lib.oracle_rx_scale_fd.argtypes = [P, I, I, P]
        lib.oracle_mrt_fd.argtypes = [P, I, I, I, I, I, P, D, D, P, P]
        lib.oracle_fd_var.argtypes = [P, I, I, I, I, I, P, P, P, P, D, D, P, P]
        lib.oracle_mrt_fd_var.argtypes = [P, I, I, I, I, I, P, P, P, D, P, P]
        lib.oracle_num_threads.restype = I
        _lib = lib
    return _lib


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), dtype=np.complex128)


def _p(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


class OracleError(RuntimeError):
    def __init__(self, rc: int, what: str):
        super().__init__(f"oracle {what} failed with rc={rc}")
        self.rc = rc


def _check(rc: int, what: str, allow_numeric: bool = False) -> None:
    if rc == OK or (allow_numeric and rc == ERR_NUMERIC):
        return
    raise OracleError(rc, what)


def num_threads() -> int:
    return int(_L().oracle_num_threads())


def gram(Ht) -> np.ndarray:
    """G = H H^H for one narrowband system given Ht[b][u]."""
    Ht = _c128(Ht)
    nb, U = Ht.shape
    G = np.empty((U, U), np.complex128)
    _check(_L().oracle_gram(_p(Ht), nb, U, _p(G)), "gram")
    return G


def cholesky(A) -> np.ndarray:
    A = _c128(A)
    U = A.shape[0]
    L = np.empty_like(A)
    _check(_L().oracle_cholesky(_p(A), U, _p(L)), "cholesky")
    return L


def hpd_inverse(A) -> np.ndarray:
    A = _c128(A)
    U = A.shape[0]
    Ai = np.empty_like(A)
    _check(_L().oracle_hpd_inverse(_p(A), U, _p(Ai)), "hpd_inverse")
    return Ai


def gauss_jordan_inverse(M) -> np.ndarray:
    M = _c128(M)
    n = M.shape[0]
    Mi = np.empty_like(M)
    _check(_L().oracle_gauss_jordan_inverse(_p(M), n, _p(Mi)), "gauss_jordan_inverse")
    return Mi


def beta_lemma1(Ainv, kappa: float, Es: float = 1.0, rho2: float = 1.0) -> float:
    Ainv = _c128(Ainv)
    return float(_L().oracle_beta_lemma1(_p(Ainv), Ainv.shape[0], kappa, Es, rho2))


def wf_theorem1(Ht, N0: float, rho2: float = 1.0, Es: float = 1.0):
    """Theorem 1 (Eqs. 4-5), B x B route.  Returns (Q[b][u], beta)."""
    Ht = _c128(Ht)
    B, U = Ht.shape
    Q = np.empty((B, U), np.complex128)
    beta = np.zeros(1, np.float64)
    _check(_L().oracle_wf_theorem1(_p(Ht), B, U, N0, rho2, Es, _p(Q), _p(beta)), "wf_theorem1")
    return Q, float(beta[0])


def wf(H, s, N0: float, rho2: float = 1.0, Es: float = 1.0):
    """Centralized WF over a frame (Theorem 1 per subcarrier).  Returns (x, beta)."""
    H, s = _c128(H), _c128(s)
    n_sc, B, U = H.shape
    K = s.shape[1]
    x = np.empty((n_sc, K, B), np.complex128)
    beta = np.empty(n_sc, np.float64)
    _check(_L().oracle_wf(_p(H), n_sc, B, U, K, _p(s), N0, rho2, Es, _p(x), _p(beta)), "wf")
    return x, beta


def pd(H, s, C: int, N0: float, rho2: float = 1.0, Es: float = 1.0, allow_numeric=False,
       return_z=False):
    """PD-WF (Sec. III-B).  Returns (x, beta[, z]) ; rc==1 allowed if allow_numeric."""
    H, s = _c128(H), _c128(s)
    n_sc, B, U = H.shape
    K = s.shape[1]
    x = np.empty((n_sc, K, B), np.complex128)
    beta = np.empty(n_sc, np.float64)
    z = np.empty((n_sc, K, U), np.complex128)
    rc = _L().oracle_pd(_p(H), n_sc, B, U, K, C, _p(s), N0, rho2, Es, _p(x), _p(beta), _p(z))
    _check(rc, "pd", allow_numeric)
    return (x, beta, z) if return_z else (x, beta)


def fd(H, s, C: int, N0: float, rho2: float = 1.0, Es: float = 1.0, tau: float = 0.125,
       allow_numeric=False):
    """FD-WF (Sec. III-C).  Returns (x, beta_c[n_sc][C])."""
    H, s = _c128(H), _c128(s)
    n_sc, B, U = H.shape
    K = s.shape[1]
    x = np.empty((n_sc, K, B), np.complex128)
    beta_c = np.empty((n_sc, C), np.float64)
    rc = _L().oracle_fd(_p(H), n_sc, B, U, K, C, _p(s), N0, rho2, Es, tau, _p(x), _p(beta_c))
    _check(rc, "fd", allow_numeric)
    return x, beta_c


def mrt_fd(H, s, C: int, rho2: float = 1.0, Es: float = 1.0):
    """Fully-distributed MRT (Fig. 2 baseline): x_c = H_c^H s / beta_c. Returns (x, beta_c[n_sc][C])."""
    H, s = _c128(H), _c128(s)
    n_sc, B, U = H.shape
    K = s.shape[1]
    x = np.empty((n_sc, K, B), np.complex128)
    beta_c = np.empty((n_sc, C), np.float64)
    _check(_L().oracle_mrt_fd(_p(H), n_sc, B, U, K, C, _p(s), rho2, Es, _p(x), _p(beta_c)), "mrt_fd")
    return x, beta_c


def _var_args(sizes, power, tau, C, rho2):
    B_c = np.ascontiguousarray(sizes, dtype=np.int32)
    w = np.full(C, 1.0 / C) if power is None else np.asarray(power, dtype=np.float64)
    rho2_c = np.ascontiguousarray(w * rho2, dtype=np.float64)
    t = np.ascontiguousarray(np.broadcast_to(np.asarray(tau, dtype=np.float64), (C,)))
    return B_c, rho2_c, t


def fd_var(H, s, sizes, N0: float, rho2: float = 1.0, Es: float = 1.0, power=None, tau=0.125,
           allow_numeric=False):
    """FD-WF with unequal clusters B_c, power shares rho_c^2 = power_c rho^2 (
    default 1/C) and per-cluster tau_c (Eq. 9; scalar or sequence).  Returns (x, beta_c[n_sc][C])."""
    H, s = _c128(H), _c128(s)
    n_sc, B, U = H.shape
    K = s.shape[1]
    C = len(sizes)
    B_c, rho2_c, t = _var_args(sizes, power, tau, C, rho2)
    x = np.empty((n_sc, K, B), np.complex128)
    beta_c = np.empty((n_sc, C), np.float64)
    rc = _L().oracle_fd_var(_p(H), n_sc, B, U, K, C, _p(B_c), _p(rho2_c), _p(t), _p(s), N0, Es, _p(x),
                            _p(beta_c))
    _check(rc, "fd_var", allow_numeric)
    return x, beta_c


def mrt_fd_var(H, s, sizes, rho2: float = 1.0, Es: float = 1.0, power=None):
    """Fully-distributed MRT with unequal clusters and power shares.  Returns (x, beta_c[n_sc][C])."""
    H, s = _c128(H), _c128(s)
    n_sc, B, U = H.shape
    K = s.shape[1]
    C = len(sizes)
    B_c, rho2_c, _ = _var_args(sizes, power, 0.0, C, rho2)
    x = np.empty((n_sc, K, B), np.complex128)
    beta_c = np.empty((n_sc, C), np.float64)
    _check(_L().oracle_mrt_fd_var(_p(H), n_sc, B, U, K, C, _p(B_c), _p(rho2_c), _p(s), Es, _p(x), _p(beta_c)),
           "mrt_fd_var")
    return x, beta_c


def rx_scale_fd(beta_c) -> np.ndarray:
    """beta_rx = 1/sum_c(1/beta_c) per subcarrier (reading R9; parity unpinned)."""
    beta_c = np.ascontiguousarray(beta_c, dtype=np.float64)
    n_sc, C = beta_c.shape
    out = np.empty(n_sc, np.float64)
    _check(_L().oracle_rx_scale_fd(_p(beta_c), n_sc, C, _p(out)), "rx_scale_fd")
    return out
