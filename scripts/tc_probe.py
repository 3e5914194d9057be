"""Validate the tcgen05 helper conventions (scripts/tc_probe.py, GPU box)."""
import ctypes, os, subprocess, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
so = os.path.join(ROOT, "paper_1804_10987_b200", "libtcprobe.so")
lib = ctypes.CDLL(so)
torch.manual_seed(0)
for K in ((8, 32, 256) if len(sys.argv) == 1 else ()):
    A = torch.randn(64, K, device="cuda")
    B = torch.randn(64, K, device="cuda")
    ref = (A.double() @ B.double().T).float()
    for mode in (0,):
        D = torch.zeros(2 * 64 * 64, device="cuda")
        rc = lib.tc_probe(ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()), ctypes.c_void_p(D.data_ptr()), K, mode)
        D0 = D[:4096].view(64, 64)
        err = ((D0 - ref).norm() / ref.norm()).item()
        print(f"K={K} mode={mode} rc={rc} relerr={err:.3e} hi-lanes-norm={D[4096:].norm().item():.3e}", flush=True)
# MN-major SW128 probe (fd_tc.cuh's Gram operand); each mode in its own process
if len(sys.argv) > 2 and sys.argv[1] == "p2":
    sw, lt, lbo, sbo = (int(v) for v in sys.argv[2:6])
    loff = int(sys.argv[6]) if len(sys.argv) > 6 else 0
    X = torch.arange(2048, device="cuda", dtype=torch.float32).view(32, 64)
    dump = torch.zeros(2048, device="cuda")
    D = torch.zeros(128 * 64, device="cuda")
    rc = lib.mn_probe2(ctypes.c_void_p(X.data_ptr()), ctypes.c_void_p(dump.data_ptr()), ctypes.c_void_p(D.data_ptr()), sw, lt, lbo, sbo, loff)
    dm = dump.cpu().numpy().astype(int)
    if sw == 4 and lt == 1 and lbo == 4096:
        print("smem layout: position -> (row, col) for box 0, first 4 rows x 32 floats:")
        for r in range(6):
            print(" ", [(v // 64, v % 64) for v in dm[r * 32:(r + 1) * 32:4]])
    Xr = torch.randn(32, 64, device="cuda")
    rc = lib.mn_probe2(ctypes.c_void_p(Xr.data_ptr()), ctypes.c_void_p(dump.data_ptr()), ctypes.c_void_p(D.data_ptr()), sw, lt, lbo, sbo, loff)
    ref = (Xr.double().T @ Xr.double()).float()
    Dl = D.view(128, 64)
    D0 = torch.cat([Dl[32 * q + loff:32 * q + loff + 16] for q in range(4)])
    print("lane-block norms", [round(Dl[16 * i:16 * i + 16].norm().item(), 1) for i in range(8)])
    err = ((D0 - ref).norm() / ref.norm()).item()
    print(f"P2 loff={loff} sw={sw} lt={lt} lbo={lbo} sbo={sbo} rc={rc} relerr={err:.3e} norm={D0.norm().item():.3e}", flush=True)
    sys.exit(0)
if len(sys.argv) > 1:
    mode = int(sys.argv[1])
    X = torch.randn(32, 64, device="cuda")
    ref = (X.double().T @ X.double()).float()
    D = torch.zeros(128 * 64, device="cuda")
    rc = lib.mn_probe(ctypes.c_void_p(X.data_ptr()), ctypes.c_void_p(D.data_ptr()), mode)
    print(f"MN mode={mode} rc={rc}", flush=True)
    Dl = D.view(128, 64)
    print("lane norms", [round(Dl[32 * q + h * 16:32 * q + h * 16 + 16].norm().item(), 1) for q in range(4) for h in range(2)])
    D0 = torch.cat([Dl[32 * q:32 * q + 16] for q in range(4)])
    err = ((D0 - ref).norm() / ref.norm()).item()
    print(f"MN mode={mode} relerr={err:.3e} norm={D0.norm().item():.3e} ref={ref.norm().item():.3e}", flush=True)
    print(D0[:2, :6].cpu().numpy(), "\n", ref[:2, :6].cpu().numpy())
    sys.exit(0)
for args in (["4", "1", "4096", "512", "0"], ["4", "1", "4096", "512", "16"]):
    subprocess.run([sys.executable, __file__, "p2"] + args)
