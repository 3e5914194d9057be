"""Unequal clusters, per-cluster power shares and tau_c ("B_c = w_c B",
P:213-215 with its footnote, Eq. 9 "tau_c"): dp_set_clusters + dp_precode_fd / dp_precode_mrt
against oracle.fd_var / oracle.mrt_fd_var, element by element, with the receive scale and the
power scalars; the equal split through dp_set_clusters is the default path bit for bit."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from paper_1804_10987_b200 import _lib as L
from paper_1804_10987_b200 import synth
from paper_1804_10987_b200.api import Precoder

from helpers import REL_TOL, rel_l2

pytestmark = pytest.mark.gpu

# (U, K, sizes, power shares or None, tau_c or None): runs that hit every FD kernel --
# fd_tc (B_c = U = 32; a run of 4 uses the tensor-core whitening, shorter runs the SIMT one),
# the SIMT fused kernel (B_c > U or U < 32), the small-cluster branch (B_c < U)
CASES = [
    (32, 14, [32, 32, 64, 32, 16, 80], [0.1, 0.2, 0.25, 0.15, 0.1, 0.2], [0.125, 0.125, 0.5, 1.0, 0.25, 0.125]),
    (32, 14, [32, 32, 32, 32, 64, 64], None, [0.125, 0.125, 0.125, 0.125, 0.3, 0.3]),
    (16, 14, [16, 48, 8, 32, 24], [0.3, 0.1, 0.2, 0.2, 0.2], None),
    (8, 7, [4, 8, 12, 40], [0.25, 0.25, 0.25, 0.25], [1.0, 0.125, 0.125, 2.0]),
    (4, 16, [4, 8, 4, 16], None, None),
]


def _frame(U, K, B, n_sc, seed):
    rng = np.random.default_rng(seed)
    H = synth.rayleigh(rng, n_sc, B, U)
    _, s = synth.QAM(64).draw(rng, (n_sc, K, U))
    return H.astype(np.complex64), s.astype(np.complex64)


def _run(pre, fn, H, s, N0, rho2, host=False):
    if host:
        Ht, st = torch.from_numpy(H).pin_memory(), torch.from_numpy(s).pin_memory()
    else:
        Ht, st = torch.from_numpy(H).cuda(), torch.from_numpy(s).cuda()
    x = fn(Ht, st, N0, rho2)
    out = (x.cpu().numpy(), pre.read_scalars("beta").cpu().numpy(), pre.read_scalars("rx").cpu().numpy(),
           pre.read_scalars("power").cpu().numpy())
    torch.cuda.synchronize()
    assert pre.status() == 0
    return out


@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("host", [False, True])
def test_fd_unequal_vs_oracle(case, host):
    U, K, sizes, power, tau = CASES[case]
    B, C, n_sc, N0, rho2 = sum(sizes), len(sizes), 37, 0.1, 1.3
    H, s = _frame(U, K, B, n_sc, 100 + case)
    with Precoder(n_sc, B, U, K, C, tau=0.125) as pre:
        pre.set_clusters(sizes, power, tau)
        x, beta, rx, pw = _run(pre, pre.precode_fd, H, s, N0, rho2, host)
    xr, br = oracle.fd_var(H, s, sizes, N0, rho2, power=power, tau=0.125 if tau is None else tau)
    assert rel_l2(x, xr) <= REL_TOL
    assert np.max(np.abs(beta.reshape(br.shape) / br - 1)) <= REL_TOL
    assert np.max(np.abs(rx / oracle.rx_scale_fd(br) - 1)) <= REL_TOL
    assert np.max(np.abs(pw / np.sum(np.abs(xr) ** 2, axis=(1, 2)) - 1)) <= REL_TOL


@pytest.mark.parametrize("case", [0, 2, 4])
def test_mrt_unequal_vs_oracle(case):
    U, K, sizes, power, _ = CASES[case]
    B, C, n_sc, rho2 = sum(sizes), len(sizes), 19, 0.7
    H, s = _frame(U, K, B, n_sc, 200 + case)
    with Precoder(n_sc, B, U, K, C) as pre:
        pre.set_clusters(sizes, power)
        x, beta, rx, pw = _run(pre, pre.precode_mrt, H, s, 0.0, rho2)
    xr, br = oracle.mrt_fd_var(H, s, sizes, rho2=rho2, power=power)
    assert rel_l2(x, xr) <= REL_TOL
    # reading R24: effective per-cluster scale beta_c / g_c, g_c = ||H_c||_F^2 / U
    bounds = np.cumsum([0] + sizes)
    g = np.stack([np.sum(np.abs(H[:, a:b].astype(np.complex128)) ** 2, axis=(1, 2)) / U
                  for a, b in zip(bounds[:-1], bounds[1:])], axis=1)
    beff = br / g
    assert np.max(np.abs(beta.reshape(br.shape) / beff - 1)) <= REL_TOL
    assert np.max(np.abs(rx * np.sum(1.0 / beff, axis=1) - 1)) <= REL_TOL
    assert np.max(np.abs(pw / np.sum(np.abs(xr) ** 2, axis=(1, 2)) - 1)) <= REL_TOL


def test_equal_split_is_default_path():
    """Setting the equal split, 1/C shares and the constructor's tau restores the default kernels:
    identical bytes to a context that never called dp_set_clusters."""
    U, K, B, C, n_sc = 32, 14, 256, 8, 23
    H, s = _frame(U, K, B, n_sc, 5)
    with Precoder(n_sc, B, U, K, C) as pre:
        x0, b0, r0, p0 = _run(pre, pre.precode_fd, H, s, 0.1, 1.0)
        pre.set_clusters([B // C] * C, [1.0 / C] * C, [0.125] * C)
        x1, b1, r1, p1 = _run(pre, pre.precode_fd, H, s, 0.1, 1.0)
        # and a genuinely unequal setting, then back
        pre.set_clusters([64, 32, 32, 32, 32, 32, 16, 16])
        pre.set_clusters(None)
        x2, *_ = _run(pre, pre.precode_fd, H, s, 0.1, 1.0)
    assert np.array_equal(x0, x1) and np.array_equal(b0, b1) and np.array_equal(r0, r1)
    assert np.array_equal(x0, x2)


def test_unequal_single_run_matches_oracle_fd():
    """One run of equal clusters with a non-default tau / power share for all of them: the var
    path (offsets, run scratch, var finish) against oracle.fd with that tau."""
    U, K, B, C, n_sc = 16, 14, 128, 4, 29
    H, s = _frame(U, K, B, n_sc, 8)
    with Precoder(n_sc, B, U, K, C, tau=0.125) as pre:
        pre.set_clusters(None, None, [0.6] * C)
        x, beta, rx, pw = _run(pre, pre.precode_fd, H, s, 0.2, 1.0)
    xr, br = oracle.fd(H, s, C, 0.2, 1.0, tau=0.6)
    assert rel_l2(x, xr) <= REL_TOL
    assert np.max(np.abs(beta.reshape(br.shape) / br - 1)) <= REL_TOL


def test_set_clusters_errors():
    U, K, B, C = 16, 14, 128, 4
    with Precoder(8, B, U, K, C) as pre:
        with pytest.raises(L.DpError) as e:
            pre.set_clusters([32, 32, 32, 16])                      # sum 112 != 128
        assert e.value.code == L.DP_ERR_INVALID
        pre.set_clusters([6, 26, 48, 48])                           # any B_c >= 1 (B_c < U: padded sub-group)
        with pytest.raises(L.DpError) as e:
            pre.set_clusters([0, 32, 48, 48])                       # B_c = 0
        assert e.value.code == L.DP_ERR_INVALID
        with pytest.raises(L.DpError) as e:
            pre.set_clusters(None, [0.5, 0.5, 0.5, 0.5])            # shares sum to 2
        assert e.value.code == L.DP_ERR_INVALID
        with pytest.raises(L.DpError) as e:
            pre.set_clusters(None, None, [0.1, -1.0, 0.1, 0.1])      # negative tau
        assert e.value.code == L.DP_ERR_INVALID
        pre.set_clusters([16, 48, 32, 32])
        H = torch.zeros((8, B, U), dtype=torch.complex64, device="cuda")
        with pytest.raises(L.DpError) as e:
            pre.prepare_fd(H, 0.1)
        assert e.value.code == L.DP_ERR_UNSUPPORTED


def test_cluster_count_not_dividing_B():
    """C does not divide B (B = 100, C = 3): FD needs the sizes (DP_ERR_INVALID before
    dp_set_clusters), then matches oracle.fd_var; PD does not depend on the partition and equals
    centralized WF."""
    U, K, B, C, n_sc, N0 = 16, 14, 100, 3, 21, 0.1
    sizes = [16, 36, 48]
    H, s = _frame(U, K, B, n_sc, 9)
    with Precoder(n_sc, B, U, K, C) as pre:
        Hd, sd = torch.from_numpy(H).cuda(), torch.from_numpy(s).cuda()
        with pytest.raises(L.DpError) as e:
            pre.precode_fd(Hd, sd, N0)
        assert e.value.code == L.DP_ERR_INVALID
        xp = pre.precode_pd(Hd, sd, N0).cpu().numpy()
        pre.set_clusters(sizes)
        x, beta, rx, pw = _run(pre, pre.precode_fd, H, s, N0, 1.0)
    xr, br = oracle.fd_var(H, s, sizes, N0)
    assert rel_l2(x, xr) <= REL_TOL
    assert np.max(np.abs(beta.reshape(br.shape) / br - 1)) <= REL_TOL
    xw, _ = oracle.wf(H, s, N0)
    assert rel_l2(xp, xw) <= REL_TOL
