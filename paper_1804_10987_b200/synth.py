"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the precoder's arithmetic: it only draws the
channel and the transmit symbols the paper's experiments use, and maps QAM
decisions for the test-side receiver.  Both the oracle (tests) and the CUDA
path consume exactly the complex64 bytes produced here.

* Channel: i.i.d. Rayleigh fading, entries CN(0, 1) (re, im each variance 1/2),
  independent across subcarriers, constant over the K OFDM symbols
  (P:86 perfect CSI, "Rayleigh fading", P:264-266 OFDM; reading R16).
  Layout H[sc][b][u] = H^paper_{u,b} (reading R2).
* Symbols: uniform i.i.d. square Gray-mapped QAM, normalised to Es = 1
  (P:91 s in O^U, P:237 64-QAM; readings R1, R17).  Layout s[sc][k][u].
* SNR: SNR = rho^2 / N0 with rho^2 = Es = 1, so N0 = 10^(-SNR/10) (reading R10).
* Seeds: numpy PCG64(SeedSequence([180410987, cfg_id, frame])).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SEED_BASE = 180410987


def rng_for(cfg_id: int, frame: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([SEED_BASE, cfg_id, frame])))


def rayleigh(rng: np.random.Generator, n_sc: int, B: int, U: int) -> np.ndarray:
    """H[sc][b][u] ~ CN(0,1) i.i.d., complex64."""
    re = rng.standard_normal((n_sc, B, U), dtype=np.float32)
    im = rng.standard_normal((n_sc, B, U), dtype=np.float32)
    h = np.empty((n_sc, B, U), np.complex64)
    h.real = re * np.float32(np.sqrt(0.5))
    h.imag = im * np.float32(np.sqrt(0.5))
    return h


def _gray(n: np.ndarray) -> np.ndarray:
    return n ^ (n >> 1)


@dataclass(frozen=True)
class QAM:
    """Square Gray-mapped M-QAM scaled to unit average energy (Es = 1)."""

    M: int

    @property
    def bits(self) -> int:
        return int(np.log2(self.M))

    @property
    def m_axis(self) -> int:
        return int(round(np.sqrt(self.M)))

    @property
    def scale(self) -> float:
        # average energy of the unscaled grid {±1, ±3, ..} x {±1, ±3, ..} is 2(M-1)/3
        return float(np.sqrt(3.0 / (2.0 * (self.M - 1))))

    def points(self) -> np.ndarray:
        """Constellation indexed by symbol index i = (iI << bits/2) | iQ (Gray per axis)."""
        m = self.m_axis
        lev = (2 * np.arange(m) - (m - 1)).astype(np.float64)  # level index -> amplitude
        # Gray label g sits at level position p with gray(p) == g
        pos_of_label = np.empty(m, np.int64)
        pos_of_label[_gray(np.arange(m))] = np.arange(m)
        i = np.arange(self.M)
        gi, gq = i >> (self.bits // 2), i & (m - 1)
        return (lev[pos_of_label[gi]] + 1j * lev[pos_of_label[gq]]) * self.scale

    def draw(self, rng: np.random.Generator, shape) -> tuple[np.ndarray, np.ndarray]:
        """Uniform i.i.d. symbol indices and their complex64 symbols."""
        idx = rng.integers(0, self.M, size=shape, dtype=np.int64)
        return idx, self.points()[idx].astype(np.complex64)

    def decide(self, shat: np.ndarray) -> np.ndarray:
        """Nearest-point decision, per axis (square QAM), ties -> lower level."""
        m = self.m_axis
        gray = _gray(np.arange(m))

        def axis(v):
            p = np.floor((v / self.scale + (m - 1)) / 2.0 + 0.5 - 1e-12)
            p = np.clip(p, 0, m - 1).astype(np.int64)
            return gray[p]

        return (axis(np.real(shat)) << (self.bits // 2)) | axis(np.imag(shat))

    def margin(self, shat: np.ndarray) -> np.ndarray:
        """Distance of each soft value to the nearest decision boundary (inner boundaries only)."""
        m = self.m_axis

        def axis(v):
            t = v / self.scale  # unscaled units; boundaries at even integers within range
            bnd = np.clip(2.0 * np.round(t / 2.0), -(m - 2), m - 2)
            return np.abs(t - bnd) * self.scale

        return np.minimum(axis(np.real(shat)), axis(np.imag(shat)))


def n0_from_snr_db(snr_db: float, rho2: float = 1.0) -> float:
    """N0 = rho^2 / 10^(SNR/10) (reading R10)."""
    return float(rho2 / (10.0 ** (snr_db / 10.0)))


@dataclass
class Frame:
    H: np.ndarray      # [n_sc][B][U] complex64
    s: np.ndarray      # [n_sc][K][U] complex64
    idx: np.ndarray    # [n_sc][K][U] symbol indices
    qam: QAM


def make_frame(cfg_id: int, n_sc: int, B: int, U: int, K: int, M: int, frame: int = 0) -> Frame:
    rng = rng_for(cfg_id, frame)
    H = rayleigh(rng, n_sc, B, U)
    qam = QAM(M)
    idx, s = qam.draw(rng, (n_sc, K, U))
    return Frame(H=H, s=s, idx=idx, qam=qam)


def noise(rng: np.random.Generator, shape, N0: float) -> np.ndarray:
    """CN(0, N0) i.i.d., complex128 (test-side receiver only)."""
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) * np.sqrt(N0 / 2.0)
