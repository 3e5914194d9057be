"""Host enqueue rate of dp_precode_* calls (how long the Python + C-ABI host side takes per
frame), to see whether small configs are host-bound.  python scripts/host_rate.py --config 2"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1804_10987_b200 import CONFIGS, synth  # noqa: E402
from paper_1804_10987_b200.api import Precoder  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--n", type=int, default=200)
args = ap.parse_args()
cfg = CONFIGS[args.config]
f = synth.make_frame(cfg.cfg_id, cfg.n_sc, cfg.B, cfg.U, cfg.K, cfg.M)
H = torch.from_numpy(f.H).cuda()
s = torch.from_numpy(f.s).cuda()
x = torch.empty((cfg.n_sc, cfg.K, cfg.B), dtype=torch.complex64, device="cuda")
with Precoder(cfg.n_sc, cfg.B, cfg.U, cfg.K, cfg.C, tau=cfg.tau) as pre:
    for _ in range(20):
        pre.precode_pd(H, s, 0.1, out=x)
        pre.precode_fd(H, s, 0.1, out=x)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.n):
        pre.precode_pd(H, s, 0.1, out=x)
        pre.precode_fd(H, s, 0.1, out=x)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
print(f"cfg{args.config}: host enqueue {1e6 * (t1 - t0) / args.n:.1f} us per PD+FD step, "
      f"wall incl. drain {1e6 * (t2 - t0) / args.n:.1f} us per step")

# the same frames through the raw C-ABI (pointers and stream precomputed): what the Python
# wrapper costs on top of the library's own host path
from paper_1804_10987_b200 import _lib as L  # noqa: E402

with Precoder(cfg.n_sc, cfg.B, cfg.U, cfg.K, cfg.C, tau=cfg.tau) as pre:
    st = torch.cuda.current_stream().cuda_stream
    hp, sp, xp = H.data_ptr(), s.data_ptr(), x.data_ptr()
    lib = L.lib()
    for _ in range(20):
        lib.dp_precode_pd(pre.ctx, hp, sp, 0.1, 1.0, xp, st)
        lib.dp_precode_fd(pre.ctx, hp, sp, 0.1, 1.0, xp, st)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.n):
        lib.dp_precode_pd(pre.ctx, hp, sp, 0.1, 1.0, xp, st)
        lib.dp_precode_fd(pre.ctx, hp, sp, 0.1, 1.0, xp, st)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
print(f"cfg{args.config}: raw C-ABI host enqueue {1e6 * (t1 - t0) / args.n:.1f} us per PD+FD step")
