"""Workload configurations (BASELINE.json `configs`).

Pure data: dimensions and modulation only, no arithmetic of the method.
"""
from __future__ import annotations

from dataclasses import dataclass, asdict


@dataclass(frozen=True)
class Config:
    cfg_id: int
    name: str
    n_sc: int   # OFDM subcarriers
    B: int      # BS antennas
    U: int      # single-antenna UEs
    C: int      # antenna clusters, B_c = B / C
    K: int      # OFDM symbols per frame sharing one channel
    M: int      # QAM order
    snr_db: float = 10.0   # reading R10: throughput configs run at 10 dB
    tau: float = 0.125     # P:241 "tau_c = 0.125 performs well"

    @property
    def S(self) -> int:
        return self.B // self.C

    @property
    def bits_per_frame(self) -> int:
        # reading R19: bits = N_sc * K * U * log2(M)
        return self.n_sc * self.K * self.U * (self.M.bit_length() - 1)

    def as_dict(self):
        d = asdict(self)
        d["S"] = self.S
        return d


CONFIGS = {
    1: Config(1, "cfg1_B16_U4_C2", n_sc=64, B=16, U=4, C=2, K=1, M=4),
    2: Config(2, "cfg2_B64_U8_C4", n_sc=1200, B=64, U=8, C=4, K=14, M=16),
    3: Config(3, "cfg3_B128_U16_C8", n_sc=1200, B=128, U=16, C=8, K=14, M=16),
    # reading R20: K for config 4 is unstated; K = 14 as configs 2-3
    4: Config(4, "cfg4_B256_U32_C8", n_sc=1200, B=256, U=32, C=8, K=14, M=64),
}

# Paper-aligned points (Fig. 2): U=16, N_sc=1200, K=7, 64-QAM.
PAPER_POINTS = {
    "fig2a": Config(101, "fig2a_B256_C2", 1200, 256, 16, 2, 7, 64),
    "fig2b": Config(102, "fig2b_B256_C4", 1200, 256, 16, 4, 7, 64),
    "fig2c": Config(103, "fig2c_B256_C8", 1200, 256, 16, 8, 7, 64),
    "fig2d": Config(104, "fig2d_B64_C2", 1200, 64, 16, 2, 7, 64),
    "fig2e": Config(105, "fig2e_B128_C4", 1200, 128, 16, 4, 7, 64),
}
