"""Device-side uncoded-BER harness (Fig. 2).

    from paper_1804_10987_b200.ber import BerRun
    run = BerRun(n_sc=1200, B=128, U=16, K=14, M=64)
    errs, bits = run.point(mode="fd", C=4, snr_db=10.0, frames=100)

Every frame is drawn on the GPU (dp_synth_frame: Philox4x32-10 keyed by the seed,
counter = (index, stream, frame)), precoded by libdp (dp_precode_pd / _fd), received
and scored on the GPU (dp_receive_count).  This module only marshals tensors; the
generator, the precoders, the receiver and the bit counting are CUDA kernels.
"""
from __future__ import annotations

import math

import torch

from . import _lib as L
from .api import Precoder

SEED = 180410987


def synth_frame(frame: int, n_sc: int, B: int, U: int, K: int, M: int, N0: float, seed: int = SEED,
                noise: bool = True, stream=None):
    """(H, s, idx, noise) on the current CUDA device, drawn by dp_synth_frame."""
    dev = torch.device("cuda", torch.cuda.current_device())
    H = torch.empty((n_sc, B, U), dtype=torch.complex64, device=dev)
    s = torch.empty((n_sc, K, U), dtype=torch.complex64, device=dev)
    idx = torch.empty((n_sc, K, U), dtype=torch.uint8, device=dev)
    n = torch.empty((n_sc, K, U), dtype=torch.complex64, device=dev) if noise else None
    st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    L.check(L.dp_synth_frame(seed, frame, n_sc, B, U, K, M, N0, H.data_ptr(), s.data_ptr(), idx.data_ptr(),
                             n.data_ptr() if n is not None else None, st), "dp_synth_frame")
    return H, s, idx, n


def receive_count(H, x, noise, rx, idx, M: int, errors: torch.Tensor, stream=None) -> None:
    """errors (uint64 device counter) += bit errors of s_hat = rx (H^T x + n) vs idx."""
    n_sc, B, U = H.shape
    K = x.shape[1]
    st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    L.check(L.dp_receive_count(n_sc, B, U, K, M, H.data_ptr(), x.data_ptr(),
                               noise.data_ptr() if noise is not None else None, rx.data_ptr(), idx.data_ptr(),
                               errors.data_ptr(), st), "dp_receive_count")


class BerRun:
    """BER points for one antenna configuration (B, U) and frame shape (n_sc, K, M)."""

    def __init__(self, n_sc: int, B: int, U: int, K: int, M: int, tau: float = 0.125, seed: int = SEED):
        self.n_sc, self.B, self.U, self.K, self.M, self.tau, self.seed = n_sc, B, U, K, M, tau, seed
        self._pre = {}

    def _precoder(self, C: int) -> Precoder:
        if C not in self._pre:
            self._pre[C] = Precoder(self.n_sc, self.B, self.U, self.K, C, tau=self.tau)
        return self._pre[C]

    def point(self, mode: str, C: int, snr_db: float, frames: int, frame0: int = 0, sizes=None, power=None,
              taus=None):
        """Bit errors and bits for `frames` frames; mode "pd" (= centralized WF), "fd",
        "mrt" (fully-distributed MRT, the Fig. 2 baseline) or "zf" (centralized zero-forcing, the
        N0 -> 0 limit of WF: the PD precoder evaluated at N0 = 0, received at the point's N0).  sizes / power / taus: an unequal
        partition for FD / MRT (dp_set_clusters; None = equal split, 1/C, the run's tau)."""
        N0 = 10.0 ** (-snr_db / 10.0)       # rho^2 = Es = 1 (reading R10)
        pre = self._precoder(C)
        pre.set_clusters(sizes, power, taus)
        errors = torch.zeros(1, dtype=torch.int64, device="cuda")
        rx = torch.empty(self.n_sc, dtype=torch.float32, device="cuda")
        for f in range(frame0, frame0 + frames):
            H, s, idx, n = synth_frame(f, self.n_sc, self.B, self.U, self.K, self.M, N0, seed=self.seed)
            if mode == "zf":
                x = pre.precode_pd(H, s, 0.0, 1.0)
            else:
                x = {"pd": pre.precode_pd, "fd": pre.precode_fd, "mrt": pre.precode_mrt}[mode](H, s, N0, 1.0)
            L.check(L.dp_read_scalars(pre.ctx, L.DP_SCALAR_RX, rx.data_ptr(),
                                      torch.cuda.current_stream().cuda_stream), "dp_read_scalars")
            receive_count(H, x, n, rx, idx, self.M, errors)
        bits = frames * self.n_sc * self.K * self.U * int(math.log2(self.M))
        return int(errors.item()), bits

    def close(self):
        for p in self._pre.values():
            p.close()
        self._pre.clear()
