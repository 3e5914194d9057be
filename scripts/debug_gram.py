import sys, os, numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle
from paper_1804_10987_b200 import CONFIGS, synth
from paper_1804_10987_b200.api import Precoder
cfg = CONFIGS[4]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
f = synth.make_frame(cfg.cfg_id, n, cfg.B, cfg.U, cfg.K, cfg.M)
iu = np.triu_indices(cfg.U)
with Precoder(n, cfg.B, cfg.U, cfg.K, cfg.C) as pre:
    H = torch.from_numpy(f.H).cuda()
    Gs = pre.debug_gram(H, False).cpu().numpy()
    Gc = pre.debug_gram(H, True).cpu().numpy()
for w in range(n):
    G = oracle.gram(f.H[w])
    e = np.linalg.norm(Gs[w, 0] - G[iu]) / np.linalg.norm(G[iu])
    ec = max(np.linalg.norm(Gc[w, c] - oracle.gram(f.H[w, 32*c:32*c+32])[iu]) / np.linalg.norm(oracle.gram(f.H[w, 32*c:32*c+32])[iu]) for c in range(8))
    print(w, f"sum relerr {e:.3e}  per-cluster max relerr {ec:.3e}")
    if w == 0:
        print("gpu", Gs[0, 0, :4], "\nref", G[iu][:4])
G0 = oracle.gram(f.H[0, 0:32])
Gfull = np.zeros((32, 32), complex)
Gfull[iu] = Gc[0, 0]
print("diag gpu", np.real(np.diag(Gfull))[:6], "\ndiag ref", np.real(np.diag(G0))[:6])
print("row0 gpu", Gfull[0, :4], "\nrow0 ref", G0[0, :4])
print("row20 gpu", Gfull[20, 20:24], "\nrow20 ref", G0[20, 20:24])
