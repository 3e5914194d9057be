"""Device-side BER harness: the GPU frame generator and
the GPU receiver / bit counter, checked against host computations on the same bytes
(oracle precoders, numpy receiver, synth.QAM decisions)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from paper_1804_10987_b200 import synth

from helpers import DECISION_MARGIN, receive, rel_l2

pytestmark = pytest.mark.gpu


def _popcount(a: np.ndarray) -> np.ndarray:
    a = a.astype(np.int64)
    c = np.zeros_like(a)
    while np.any(a):
        c += a & 1
        a >>= 1
    return c


@pytest.mark.parametrize("M", [4, 16, 64])
def test_synth_frame_distribution_and_mapping(M):
    from paper_1804_10987_b200.ber import synth_frame
    n_sc, B, U, K, N0 = 64, 128, 16, 14, 0.25
    H, s, idx, n = synth_frame(3, n_sc, B, U, K, M, N0)
    H2, s2, idx2, n2 = synth_frame(3, n_sc, B, U, K, M, N0)
    H3, *_ = synth_frame(4, n_sc, B, U, K, M, N0)
    torch.cuda.synchronize()
    # reproducible per (seed, frame), different across frames
    assert torch.equal(H, H2) and torch.equal(s, s2) and torch.equal(idx, idx2) and torch.equal(n, n2)
    assert not torch.equal(H, H3)
    H, s, idx, n = (t.cpu().numpy() for t in (H, s, idx, n))
    qam = synth.QAM(M)
    # symbols are the Gray QAM points of their indices (the host constellation, Es = 1)
    assert np.max(np.abs(s - qam.points()[idx.astype(np.int64)])) <= 1e-6
    # statistics: CN(0, 1) channel, CN(0, N0) noise, uniform indices
    assert abs(np.mean(np.abs(H) ** 2) - 1.0) < 0.01
    assert abs(np.mean(H)) < 0.01
    assert abs(np.mean(H.real ** 2) - 0.5) < 0.01 and abs(np.mean(H.real * H.imag)) < 0.01
    assert abs(np.mean(np.abs(n) ** 2) / N0 - 1.0) < 0.03
    cnt = np.bincount(idx.ravel(), minlength=M)
    assert cnt.min() > 0.8 * idx.size / M and cnt.max() < 1.2 * idx.size / M
    assert abs(np.mean(np.abs(s) ** 2) - 1.0) < 0.05


@pytest.mark.parametrize("mode", ["pd", "fd"])
def test_receive_count_matches_host(mode):
    """GPU bit-error count of one frame == the host receiver on the same H, x, noise,
    scale, up to symbols within DECISION_MARGIN of a boundary (reading R11); and the
    GPU-precoded frame agrees with the oracle (relative L2 <= 1e-4)."""
    from paper_1804_10987_b200.api import Precoder
    from paper_1804_10987_b200.ber import receive_count, synth_frame
    n_sc, B, U, K, M, C, snr = 24, 128, 16, 14, 64, 4, 12.0
    N0 = synth.n0_from_snr_db(snr)
    H, s, idx, n = synth_frame(7, n_sc, B, U, K, M, N0)
    with Precoder(n_sc, B, U, K, C) as pre:
        x = (pre.precode_pd if mode == "pd" else pre.precode_fd)(H, s, N0, 1.0)
        rx = pre.read_scalars("rx")
        err = torch.zeros(1, dtype=torch.int64, device="cuda")
        receive_count(H, x, n, rx, idx, M, err)
        torch.cuda.synchronize()
    Hh, sh, ih, nh, xh, rxh = (t.cpu().numpy() for t in (H, s, idx, n, x, rx))
    # host receiver on the GPU's own precoded output
    qam = synth.QAM(M)
    shat = receive(Hh, xh, nh, rxh)
    dec = qam.decide(shat)
    inside = qam.margin(shat) < DECISION_MARGIN
    bits_host = _popcount(dec ^ ih.astype(np.int64))
    lo = int(bits_host[~inside].sum())
    hi = lo + qam.bits * int(inside.sum())
    assert lo <= int(err.item()) <= hi, (int(err.item()), lo, hi)
    assert lo > 0                                   # 12 dB, 64-QAM: errors do occur
    # and the precoder itself against the fp64 oracle on these device-drawn inputs
    if mode == "pd":
        xr, _ = oracle.pd(Hh, sh, C, N0)
    else:
        xr, _ = oracle.fd(Hh, sh, C, N0, tau=0.125)
    assert rel_l2(xh, xr) <= 1e-4


def test_noiseless_wf_recovers_symbols():
    """PD (= centralized WF) at N0 -> 0 without noise is the ZF precoder: beta H P = I
    (P:37), so every symbol is recovered and the GPU count is zero."""
    from paper_1804_10987_b200.api import Precoder
    from paper_1804_10987_b200.ber import receive_count, synth_frame
    H, s, idx, _ = synth_frame(1, 32, 64, 8, 14, 64, 0.0, noise=False)
    with Precoder(32, 64, 8, 14, 4) as pre:
        x = pre.precode_pd(H, s, 1e-7, 1.0)
        rx = pre.read_scalars("rx")
        err = torch.zeros(1, dtype=torch.int64, device="cuda")
        receive_count(H, x, None, rx, idx, 64, err)
        torch.cuda.synchronize()
    assert int(err.item()) == 0


def test_pd_ber_independent_of_cluster_count():
    """PD-WF equals centralized WF for every C: identical inputs give the same
    error count for C = 1, 2, 4, 8 (up to near-boundary symbols), while FD differs."""
    from paper_1804_10987_b200.ber import BerRun
    run = BerRun(n_sc=64, B=128, U=16, K=14, M=64)
    pd = [run.point("pd", C, 10.0, frames=2)[0] for C in (1, 2, 4, 8)]
    fd8, bits = run.point("fd", 8, 10.0, frames=2)
    run.close()
    assert max(pd) - min(pd) <= 0.01 * max(pd) + 8, pd
    assert fd8 > pd[0]          # FD at B_c = 16 loses against WF (Fig. 2)
    assert 0 < pd[0] < bits
