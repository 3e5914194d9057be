"""K-major tf32 UMMA with the SWIZZLE_128B_BASE32B layout (scripts/kmaj32_probe.cu); GPU box.
Each configuration in its own process (a bad descriptor may fault the context)."""
import ctypes, os, subprocess, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
so = os.path.join(ROOT, "scripts", "libkprobe.so")
if len(sys.argv) == 1:
    for swz, lt, lbo, sbo in [(1, 2, 16, 1024), (0, 1, 16, 1024), (0, 1, 16, 512), (0, 1, 1024, 512), (0, 1, 512, 1024)]:
        r = subprocess.run([sys.executable, __file__, str(swz), str(lt), str(lbo), str(sbo)], capture_output=True, text=True, timeout=120)
        print(r.stdout.strip() or r.stderr.strip()[-300:], flush=True)
    sys.exit(0)
swz, lt, lbo, sbo = (int(v) for v in sys.argv[1:5])
lib = ctypes.CDLL(so)
torch.manual_seed(0)
X = torch.randn(128, 32, device="cuda")
Y = torch.randn(32, 32, device="cuda")
ref = (X.double() @ Y.double().T).float()
D = torch.zeros(128, 32, device="cuda")
rc = lib.kprobe(ctypes.c_void_p(X.data_ptr()), ctypes.c_void_p(Y.data_ptr()), ctypes.c_void_p(D.data_ptr()), swz, lt, lbo, sbo)
err = ((D - ref).norm() / ref.norm()).item()
print(f"swz={'SW128' if swz else 'ATOM32B'} layout_type={lt} lbo={lbo} sbo={sbo} rc={rc} relerr={err:.3e}")
