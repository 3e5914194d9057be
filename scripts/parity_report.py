"""Print the CUDA-vs-oracle error envelope for every config, mode and SNR (GPU box).

    python scripts/parity_report.py [--n-sc 64] [--out profiles/parity_rXX.json]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
from helpers import decision_parity, rel_l2  # noqa: E402
from paper_1804_10987_b200 import CONFIGS, PAPER_POINTS, synth  # noqa: E402
from paper_1804_10987_b200 import _lib as L  # noqa: E402
from paper_1804_10987_b200.api import Precoder  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-sc", type=int, default=64)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rows = []
    cfgs = [CONFIGS[i] for i in (1, 2, 3, 4)] + [PAPER_POINTS["fig2a"], PAPER_POINTS["fig2c"]]
    for cfg in cfgs:
        n = min(args.n_sc, cfg.n_sc)
        f = synth.make_frame(cfg.cfg_id, n, cfg.B, cfg.U, cfg.K, cfg.M, frame=3)
        for snr in (-5.0, 10.0, 25.0, 40.0):
            N0 = synth.n0_from_snr_db(snr)
            for mode in ("pd", "fd"):
                for unfused in (False, True):
                    with Precoder(n, cfg.B, cfg.U, cfg.K, cfg.C, tau=cfg.tau,
                                  flags=L.DP_FLAG_UNFUSED if unfused else 0) as pre:
                        H = torch.from_numpy(f.H).cuda()
                        s = torch.from_numpy(f.s).cuda()
                        x = (pre.precode_pd if mode == "pd" else pre.precode_fd)(H, s, N0, 1.0).cpu().numpy()
                        rx = pre.read_scalars("rx").cpu().numpy()
                        beta = pre.read_scalars("beta").cpu().numpy()
                        nbad = pre.status()
                    if mode == "pd":
                        xr, br = oracle.pd(f.H, f.s, cfg.C, N0)
                        rxr = br
                    else:
                        xr, br = oracle.fd(f.H, f.s, cfg.C, N0, tau=cfg.tau)
                        rxr = oracle.rx_scale_fd(br)
                    noise = synth.noise(synth.rng_for(cfg.cfg_id, 11), (n, cfg.K, cfg.U), N0)
                    mism, inside, tot = decision_parity(f.qam, f.H, x, rx, xr, rxr, noise)
                    row = dict(cfg=cfg.name, snr_db=snr, mode=mode, path="unfused" if unfused else "fused",
                               rel_l2=rel_l2(x, xr),
                               beta_max_rel=float(np.max(np.abs(beta.reshape(br.shape) / br - 1))),
                               decisions_mismatch=mism, inside_margin=inside, symbols=tot, nbad=nbad)
                    rows.append(row)
                    print(f"{cfg.name:20s} {snr:6.1f} dB {mode} {row['path']:8s} relL2={row['rel_l2']:.2e} "
                          f"beta={row['beta_max_rel']:.2e} mism={mism} inside={inside}/{tot} bad={nbad}", flush=True)
    if args.out:
        with open(args.out, "w") as fo:
            json.dump(rows, fo, indent=1)


if __name__ == "__main__":
    main()
