"""PD kernel times at n_sc = 1184 (= 148 x 8: every persistent CTA gets the same number of
subcarriers) vs 1200 (16 CTAs get a 9th): does the item-granular split cost time?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1804_10987_b200 import _lib as L  # noqa: E402
from paper_1804_10987_b200.api import Precoder  # noqa: E402

for n_sc in (1184, 1200, 1332):
    H = torch.randn((n_sc, 256, 32), dtype=torch.complex64, device="cuda")
    s = torch.randn((n_sc, 14, 32), dtype=torch.complex64, device="cuda")
    x = torch.empty((n_sc, 14, 256), dtype=torch.complex64, device="cuda")
    with Precoder(n_sc, 256, 32, 14, 8, flags=L.DP_FLAG_PROFILE) as pre:
        for _ in range(5):
            pre.precode_pd(H, s, 0.1, out=x)
        torch.cuda.synchronize()
        pre.profile(reset=True)
        for _ in range(20):
            pre.precode_pd(H, s, 0.1, out=x)
        torch.cuda.synchronize()
        p = pre.profile(reset=True)
    print(n_sc, {k: round(1e3 * v["ms"] / max(v["launches"], 1), 2) for k, v in p.items() if v["launches"]},
          "per 1200 sc:", {k: round(1e3 * v["ms"] / max(v["launches"], 1) * 1200 / n_sc, 2) for k, v in p.items() if v["launches"]})
