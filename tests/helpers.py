"""Shared test helpers: parity metrics and the test-side receiver (reading R11)."""
from __future__ import annotations

import numpy as np

from paper_1804_10987_b200 import synth

REL_TOL = 1e-4          # north_star: relative L2 error <= 1e-4 (fp32 vs fp64)
DECISION_MARGIN = 1e-4  # reading R11: symbols within this distance of a boundary are excluded


def rel_l2(a, b) -> float:
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def receive(H, x, noise, rx_scale):
    """s_hat[sc][k][u] = beta_rx[sc] (sum_b H_{u,b} x_k[b] + n_k[u])  (Eq. 1, joint UE scaling P:106-114).
    H[sc][b][u] (paper H^T), x[sc][k][b]."""
    H = np.asarray(H, np.complex128)
    x = np.asarray(x, np.complex128)
    y = np.einsum("wbu,wkb->wku", H, x) + noise
    return np.asarray(rx_scale, np.float64)[:, None, None] * y


def decision_parity(qam: synth.QAM, H, x_gpu, rx_gpu, x_ref, rx_ref, noise):
    """Compare per-UE hard decisions of the GPU and oracle outputs under the same channel and noise.
    Returns (n_mismatch_outside_margin, n_inside_margin, n_total)."""
    s_ref = receive(H, x_ref, noise, rx_ref)
    s_gpu = receive(H, x_gpu, noise, rx_gpu)
    d_ref = qam.decide(s_ref)
    d_gpu = qam.decide(s_gpu)
    inside = qam.margin(s_ref) < DECISION_MARGIN
    mism = (d_ref != d_gpu) & ~inside
    return int(mism.sum()), int(inside.sum()), int(d_ref.size)
