"""Validate the tcgen05 helper conventions (scripts/tc_probe.py, GPU box)."""
import ctypes, os, subprocess, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
so = os.path.join(ROOT, "paper_1804_10987_b200", "libtcprobe.so")
lib = ctypes.CDLL(so)
torch.manual_seed(0)
for K in (8, 32, 256):
    A = torch.randn(64, K, device="cuda")
    B = torch.randn(64, K, device="cuda")
    ref = (A.double() @ B.double().T).float()
    for mode in (0,):
        D = torch.zeros(2 * 64 * 64, device="cuda")
        rc = lib.tc_probe(ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()), ctypes.c_void_p(D.data_ptr()), K, mode)
        D0 = D[:4096].view(64, 64)
        err = ((D0 - ref).norm() / ref.norm()).item()
        print(f"K={K} mode={mode} rc={rc} relerr={err:.3e} hi-lanes-norm={D[4096:].norm().item():.3e}", flush=True)
