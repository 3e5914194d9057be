import ctypes, os, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_1804_10987_b200", "libtmaprobe.so"))
torch.manual_seed(0)
R = 512
A = torch.randn(R, 64, device="cuda")
B = torch.randn(64, 32, device="cuda")
Bt = (B.view(torch.int32) & 0xFFFFE000).view(torch.float32)    # exactly tf32
for row0, col0 in ((0, 0), (128, 32), (384, 0)):
    for split in (0, 1):
        D = torch.zeros(128, 64, device="cuda")
        rc = lib.tma_probe(ctypes.c_void_p(A.data_ptr()), R, ctypes.c_void_p(Bt.data_ptr()), ctypes.c_void_p(D.data_ptr()), row0, col0, split)
        ref = (A[row0:row0 + 128, col0:col0 + 32].double() @ Bt.double().T)
        print(f"row0={row0} col0={col0} split={split} rc={rc} relerr={((D.double() - ref).norm() / ref.norm()).item():.3e}", flush=True)
