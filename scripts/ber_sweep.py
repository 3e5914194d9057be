"""Uncoded BER sweep on the GPU (BASELINE.json configs[4] / SURVEY.md §8 f1; Fig. 2).

    python scripts/ber_sweep.py [--frames F] [--snr=-5:25:1] [--B 128] [--U 16] [--C 1,2,4,8] [--out PATH]

Config 5: B = 128, U = 16, C in {1, 2, 4, 8}, 64-QAM, 1200 subcarriers x 14 OFDM
symbols per frame, SNR -5..25 dB; FD-WF (tau = 0.125) vs PD-WF, which equals
centralized WF for every C and is therefore run once (C = 1).  Frames are
drawn on the device (dp_synth_frame), precoded by libdp and scored on the device
(dp_receive_count).  Prints one JSON line per point and writes the table to --out.
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=20)
    ap.add_argument("--snr", default="-5:25:1")
    ap.add_argument("--B", type=int, default=128)
    ap.add_argument("--U", type=int, default=16)
    ap.add_argument("--C", default="1,2,4,8")
    ap.add_argument("--n_sc", type=int, default=1200)
    ap.add_argument("--K", type=int, default=14)
    ap.add_argument("--M", type=int, default=64)
    ap.add_argument("--tau", default="0.125", help="FD regularisation tau_c (Eq. 9); comma list = tau sweep")
    ap.add_argument("--no-pd", action="store_true", help="FD points only")
    ap.add_argument("--mrt", action="store_true", help="add fully-distributed MRT (Fig. 2 baseline) at every C")
    ap.add_argument("--zf", action="store_true", help="add centralized zero-forcing (WF in the N0 -> 0 limit, P:37)")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    lo, hi, step = (float(v) for v in args.snr.split(":"))
    snrs = [lo + i * step for i in range(int(round((hi - lo) / step)) + 1)]
    Cs = [int(c) for c in args.C.split(",")]
    taus = [float(t) for t in args.tau.split(",")]
    runs = {t: BerRun(args.n_sc, args.B, args.U, args.K, args.M, tau=t) for t in taus}
    rows = []
    t0 = time.time()
    for snr in snrs:
        pts = ([] if args.no_pd else [("pd", 1, taus[0])]) + [("fd", c, t) for t in taus for c in Cs] + \
              ([("mrt", c, taus[0]) for c in Cs] if args.mrt else []) + ([("zf", 1, taus[0])] if args.zf else [])
        for mode, C, tau in pts:
            e, bits = runs[tau].point(mode, C, snr, args.frames)
            row = {"mode": {"pd": "WF(=PD)", "fd": "FD", "mrt": "MRT", "zf": "ZF"}[mode], "C": C, "B": args.B, "U": args.U,
                   "snr_db": snr, "errors": e, "bits": bits, "ber": e / bits, "frames": args.frames}
            if mode == "fd":
                row["tau"] = tau
            rows.append(row)
            print(json.dumps(row), flush=True)
    torch.cuda.synchronize()
    for r in runs.values():
        r.close()
    meta = {"what": "uncoded BER, Rayleigh, GPU-drawn frames (Philox), libdp precoders", "seconds": time.time() - t0,
            "n_sc": args.n_sc, "K": args.K, "M": args.M, "tau": taus}
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"meta": meta, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
