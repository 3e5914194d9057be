"""Compare FD outputs of the tensor-core FD kernel vs the SIMT fused kernel per
(subcarrier, cluster) problem: python scripts/debug_fdtc.py [n_sc] (runs both arms
as subprocesses; the kernel choice is read from DP_NO_TC_FD once per process)."""
import os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
n = int(sys.argv[1]) if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else 8
if "--child" in sys.argv:
    sys.path.insert(0, ROOT)
    import torch
    from paper_1804_10987_b200 import CONFIGS, synth
    from paper_1804_10987_b200.api import Precoder
    cfg = CONFIGS[4]
    f = synth.make_frame(cfg.cfg_id, n, cfg.B, cfg.U, cfg.K, cfg.M)
    with Precoder(n, cfg.B, cfg.U, cfg.K, cfg.C) as pre:
        x = pre.precode_fd(torch.from_numpy(f.H).cuda(), torch.from_numpy(f.s).cuda(), synth.n0_from_snr_db(10.0), 1.0)
        beta = pre.read_scalars("beta").cpu().numpy() if hasattr(pre, "read_scalars") else None
        np.save(sys.argv[-1], x.cpu().numpy())
        if beta is not None:
            np.save(sys.argv[-1] + ".beta.npy", beta)
    sys.exit(0)
outs = []
for tag, env in (("tc", {}), ("simt", {"DP_NO_TC_FD": "1"})):
    path = f"/tmp/fd_{tag}.npy"
    subprocess.check_call([sys.executable, __file__, str(n), "--child", path], env={**os.environ, **env})
    outs.append(np.load(path))
a, b = outs
print("shapes", a.shape)
for sc in range(n):
    errs = []
    for c in range(8):
        xa, xb = a[sc, :, 32 * c:32 * c + 32], b[sc, :, 32 * c:32 * c + 32]
        errs.append(np.linalg.norm(xa - xb) / max(np.linalg.norm(xb), 1e-30))
    print(sc, " ".join(f"{e:.1e}" for e in errs))
