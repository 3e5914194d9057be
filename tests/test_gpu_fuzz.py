"""Randomised GPU parity sweep over the supported shape space (U, C, cluster size incl. B_c < U,
K, n_sc incl. 1 and ragged, SNR), PD and FD against the fp64 oracle.  Seeded: the same cases every
run.  Square clusters (B_c = U) are kept at <= 15 dB on the fp32 path, where conditioning leaves margin
to the 1e-4 bar; test_random_shapes_fp64_high_snr covers 15-40 dB and N0 = 0 with
DP_FLAG_FP64."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from paper_1804_10987_b200 import synth
from paper_1804_10987_b200.api import Precoder

from helpers import REL_TOL, rel_l2

pytestmark = pytest.mark.gpu


def _case(seed: int):
    rng = np.random.default_rng(1000 + seed)
    U = int(rng.choice([4, 8, 16, 32]))
    C = int(rng.choice([1, 2, 4, 8]))
    sizes = [U, 2 * U, 4 * U] + [b for b in (2, 4, 6, 8, 16, 24) if b < U]
    S = int(rng.choice(sizes))
    if S * C > 256:
        C = max(1, 256 // S)
    K = int(rng.integers(1, 21))
    n_sc = int(rng.choice([1, 3, int(rng.integers(4, 41))]))
    snr = float(rng.uniform(0.0, 15.0 if S <= U else 25.0))
    M = int(rng.choice([4, 16, 64]))
    return U, C, S, K, n_sc, snr, M


@pytest.mark.parametrize("seed", range(48))
def test_random_shapes(seed):
    U, C, S, K, n_sc, snr, M = _case(seed)
    B = S * C
    f = synth.make_frame(50 + seed, n_sc, B, U, K, M)
    N0 = synth.n0_from_snr_db(snr)
    H = torch.from_numpy(f.H).cuda()
    s = torch.from_numpy(f.s).cuda()
    with Precoder(n_sc, B, U, K, C) as pre:
        x_pd = pre.precode_pd(H, s, N0, 1.0).cpu().numpy()
        x_fd = pre.precode_fd(H, s, N0, 1.0).cpu().numpy()
        rx_fd = pre.read_scalars("rx").cpu().numpy()
        assert pre.status() == 0
    xr_pd, _ = oracle.pd(f.H, f.s, C, N0)
    xr_fd, br = oracle.fd(f.H, f.s, C, N0, tau=0.125)
    case = dict(U=U, C=C, S=S, K=K, n_sc=n_sc, snr=round(snr, 1), M=M)
    assert rel_l2(x_pd, xr_pd) <= REL_TOL, (case, rel_l2(x_pd, xr_pd))
    assert rel_l2(x_fd, xr_fd) <= REL_TOL, (case, rel_l2(x_fd, xr_fd))
    assert np.max(np.abs(rx_fd / oracle.rx_scale_fd(br) - 1)) <= REL_TOL, case


def _var_case(seed: int):
    """Random unequal partition: sizes from the supported set, Dirichlet power shares,
    per-cluster tau_c; C need not divide B."""
    rng = np.random.default_rng(5000 + seed)
    U = int(rng.choice([4, 8, 16, 32]))
    allowed = [U, U + 8, 2 * U, 3 * U] + [b for b in (3, 4, 8, 12, 16, 20) if b < U]
    C = int(rng.integers(2, 9))
    sizes = [int(rng.choice(allowed)) for _ in range(C)]
    if rng.random() < 0.5:                            # long runs of equal clusters too
        sizes = sorted(sizes)
    power = rng.dirichlet(np.full(C, 2.0)).tolist()
    tau = [float(v) for v in rng.choice([0.125, 0.25, 0.5, 1.0], size=C)]
    K = int(rng.integers(1, 17))
    n_sc = int(rng.choice([1, int(rng.integers(2, 41)), int(rng.integers(2, 41))]))
    snr = float(rng.uniform(0.0, 15.0))
    return U, sizes, power, tau, K, n_sc, snr


@pytest.mark.parametrize("seed", range(24))
def test_random_unequal_clusters(seed):
    U, sizes, power, tau, K, n_sc, snr = _var_case(seed)
    B, C = sum(sizes), len(sizes)
    f = synth.make_frame(90 + seed, n_sc, B, U, K, 16)
    N0 = synth.n0_from_snr_db(snr)
    with Precoder(n_sc, B, U, K, C) as pre:
        pre.set_clusters(sizes, power, tau)
        x = pre.precode_fd(torch.from_numpy(f.H).cuda(), torch.from_numpy(f.s).cuda(), N0, 1.0).cpu().numpy()
        rx = pre.read_scalars("rx").cpu().numpy()
        assert pre.status() == 0
    xr, br = oracle.fd_var(f.H, f.s, sizes, N0, power=power, tau=tau)
    case = dict(U=U, sizes=sizes, K=K, n_sc=n_sc, snr=round(snr, 1))
    assert rel_l2(x, xr) <= REL_TOL, (case, rel_l2(x, xr))
    assert np.max(np.abs(rx / oracle.rx_scale_fd(br) - 1)) <= REL_TOL, case


def _f64_case(seed: int):
    """B_c >= U (the branch DP_FLAG_FP64 covers), SNR up to 40 dB or N0 = 0, square clusters
    (B_c = U) with probability 1/2: the high-SNR envelope the fp32 fuzz above stays out of."""
    rng = np.random.default_rng(7000 + seed)
    U = int(rng.choice([4, 8, 16, 32]))
    S = U if rng.random() < 0.5 else int(rng.choice([2 * U, 4 * U]))
    C = int(rng.choice([1, 2, 4, 8]))
    if S * C > 256:
        C = max(1, 256 // S)
    K = int(rng.integers(1, 21))
    n_sc = int(rng.choice([1, 3, int(rng.integers(4, 41))]))
    snr = None if rng.random() < 0.25 else float(rng.uniform(15.0, 40.0))
    return U, C, S, K, n_sc, snr


@pytest.mark.parametrize("seed", range(24))
def test_random_shapes_fp64_high_snr(seed):
    from paper_1804_10987_b200 import _lib as L
    U, C, S, K, n_sc, snr = _f64_case(seed)
    B = S * C
    f = synth.make_frame(150 + seed, n_sc, B, U, K, 16)
    N0 = 0.0 if snr is None else synth.n0_from_snr_db(snr)
    H = torch.from_numpy(f.H).cuda()
    s = torch.from_numpy(f.s).cuda()
    with Precoder(n_sc, B, U, K, C, flags=L.DP_FLAG_FP64) as pre:
        x_pd = pre.precode_pd(H, s, N0, 1.0).cpu().numpy()
        x_fd = pre.precode_fd(H, s, N0, 1.0).cpu().numpy()
        rx_fd = pre.read_scalars("rx").cpu().numpy()
        assert pre.status() == 0
    xr_pd, _ = oracle.pd(f.H, f.s, C, N0)
    xr_fd, br = oracle.fd(f.H, f.s, C, N0, tau=0.125)
    case = dict(U=U, C=C, S=S, K=K, n_sc=n_sc, snr=snr)
    assert rel_l2(x_pd, xr_pd) <= REL_TOL, (case, rel_l2(x_pd, xr_pd))
    assert rel_l2(x_fd, xr_fd) <= REL_TOL, (case, rel_l2(x_fd, xr_fd))
    assert np.max(np.abs(rx_fd / oracle.rx_scale_fd(br) - 1)) <= REL_TOL, case
