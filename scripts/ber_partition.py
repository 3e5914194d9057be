"""Uncoded BER of FD-WF under unequal cluster sizes and power splits (P:157,
P:213-215 and its footnote: unequal per-cluster power "did not provide significant performance
advantages in massive MU-MIMO").  B = 256, U = 16, C = 8, 64-QAM, 1200 x 14 per frame, frames drawn
and scored on the GPU (paper_1804_10987_b200.ber).

    python scripts/ber_partition.py [--frames F] [--snr=0:20:2] [--out PATH]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1804_10987_b200.ber import BerRun  # noqa: E402

B, U, C = 256, 16, 8
UNEQ = [64, 64, 32, 32, 16, 16, 16, 16]
VARIANTS = {
    "equal sizes, equal power (paper)": (None, None),
    "equal sizes, power 1.5/C on half, 0.5/C on half": (None, [1.5 / C] * 4 + [0.5 / C] * 4),
    "unequal sizes, equal power 1/C": (UNEQ, None),
    "unequal sizes, power prop. to B_c": (UNEQ, [b / B for b in UNEQ]),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=20)
    ap.add_argument("--snr", default="0:20:2")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    lo, hi, step = (float(v) for v in args.snr.split(":"))
    snrs = [lo + i * step for i in range(int(round((hi - lo) / step)) + 1)]
    run = BerRun(1200, B, U, 14, 64, tau=0.125)
    rows, t0 = [], time.time()
    for snr in snrs:
        for name, (sizes, power) in VARIANTS.items():
            e, bits = run.point("fd", C, snr, args.frames, sizes=sizes, power=power)
            row = {"variant": name, "sizes": sizes or [B // C] * C, "power": power or [1.0 / C] * C,
                   "snr_db": snr, "errors": e, "bits": bits, "ber": e / bits, "frames": args.frames}
            rows.append(row)
            print(json.dumps(row), flush=True)
    torch.cuda.synchronize()
    run.close()
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"meta": {"what": "FD-WF uncoded BER vs partition / power split", "B": B, "U": U, "C": C,
                                "tau": 0.125, "seconds": time.time() - t0}, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
