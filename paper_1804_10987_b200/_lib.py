"""ctypes binding of libdp.so — the C-ABI declared in include/dp.h.

Names match the C entry points.  This module only marshals arguments; every
step of the precoders runs in the CUDA kernels of libdp.so.  There is no
fallback: if libdp.so is missing or cannot be loaded, importing fails loudly.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DP_LIB_PATH") or os.path.join(_HERE, "libdp.so")   # override: A/B experiments

DP_OK, DP_ERR_NUMERIC, DP_ERR_INVALID, DP_ERR_CUDA, DP_ERR_NCCL, DP_ERR_UNSUPPORTED = range(6)
DP_FLAG_SYNC, DP_FLAG_UNFUSED, DP_FLAG_PROFILE, DP_FLAG_FORCE_COMM, DP_FLAG_FP64, DP_FLAG_HOST_ASYNC = 1, 2, 4, 8, 16, 32
DP_PD_ALLREDUCE, DP_PD_REDUCE_BCAST, DP_PD_SCATTER_GATHER, DP_PD_NVLINK = 0, 1, 2, 3
DP_SCALAR_BETA, DP_SCALAR_RX, DP_SCALAR_POWER = 0, 1, 2
COMM_KINDS = ["gram", "s_bcast", "z_bcast", "scalars"]   # DP_COMM_* order
DP_NUM_COMM = len(COMM_KINDS)
KERNEL_NAMES = ["fused_fd", "gram", "solve", "precode", "finish", "fused_pd"]
DP_NUM_KERNELS = len(KERNEL_NAMES)

# every symbol include/dp.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "dp_get_unique_id", "dp_init", "dp_precode_pd", "dp_precode_fd", "dp_read_scalars",
    "dp_status", "dp_profile_read", "dp_launch_count", "dp_finalize", "dp_last_error",
    "dp_debug_gram", "dp_debug_solve", "dp_synth_frame", "dp_receive_count",
    "dp_prepare_pd", "dp_prepare_fd", "dp_apply", "dp_comm_ledger", "dp_precode_mrt", "dp_prepare_from_gram",
    "dp_set_clusters", "dp_comm_info",
]


class DpConfig(ctypes.Structure):
    _fields_ = [
        ("n_sc", ctypes.c_int), ("B", ctypes.c_int), ("U", ctypes.c_int), ("K", ctypes.c_int),
        ("C", ctypes.c_int), ("rank", ctypes.c_int), ("world", ctypes.c_int), ("device", ctypes.c_int),
        ("nccl_id", ctypes.c_void_p), ("Es", ctypes.c_double), ("tau", ctypes.c_double),
        ("pd_topology", ctypes.c_int), ("s_on_all_ranks", ctypes.c_int), ("flags", ctypes.c_int),
    ]


class DpError(RuntimeError):
    def __init__(self, code: int, where: str, msg: str):
        super().__init__(f"{where} failed (code {code}): {msg}")
        self.code = code


_lib = None


def lib() -> ctypes.CDLL:
    """Load libdp.so (raises OSError/ImportError if it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    P, I, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
    L.dp_get_unique_id.argtypes = [P]
    L.dp_init.argtypes = [ctypes.POINTER(DpConfig), ctypes.POINTER(P)]
    for f in (L.dp_precode_pd, L.dp_precode_fd, L.dp_precode_mrt):
        f.argtypes = [P, P, P, D, D, P, P]
    L.dp_read_scalars.argtypes = [P, I, P, P]
    L.dp_status.argtypes = [P, ctypes.POINTER(I)]
    L.dp_profile_read.argtypes = [P, P, P, I]
    L.dp_launch_count.argtypes = [P]
    L.dp_launch_count.restype = ctypes.c_longlong
    L.dp_finalize.argtypes = [P]
    L.dp_last_error.restype = ctypes.c_char_p
    L.dp_debug_gram.argtypes = [P, P, I, P, P]
    L.dp_debug_solve.argtypes = [P, P, I, P, D, D, P, P, P]
    L.dp_comm_ledger.argtypes = [P, P, I]
    L.dp_prepare_pd.argtypes = [P, P, D, D, P]
    L.dp_prepare_fd.argtypes = [P, P, D, D, P]
    L.dp_apply.argtypes = [P, P, P, I, P, P]
    L.dp_prepare_from_gram.argtypes = [P, I, P, D, D, P]
    L.dp_set_clusters.argtypes = [P, P, P, P]
    L.dp_comm_info.argtypes = [P, P, P]
    U64 = ctypes.c_ulonglong
    L.dp_synth_frame.argtypes = [U64, U64, I, I, I, I, I, D, P, P, P, P, P]
    L.dp_receive_count.argtypes = [I, I, I, I, I, P, P, P, P, P, P, P]
    for name in EXPORTS:
        getattr(L, name).restype = getattr(L, name).restype if name in ("dp_launch_count", "dp_last_error") else I
    _lib = L
    return L


def check(rc: int, where: str) -> int:
    if rc != DP_OK:
        raise DpError(rc, where, lib().dp_last_error().decode(errors="replace"))
    return rc


# ---------------------------------------------------------------- same-name wrappers
def dp_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(lib().dp_get_unique_id(buf), "dp_get_unique_id")
    return buf.raw


def dp_init(cfg: DpConfig) -> ctypes.c_void_p:
    ctx = ctypes.c_void_p()
    check(lib().dp_init(ctypes.byref(cfg), ctypes.byref(ctx)), "dp_init")
    return ctx


def dp_precode_pd(ctx, H_ptr: int, s_ptr: int, N0: float, rho2: float, x_ptr: int, stream: int) -> int:
    return lib().dp_precode_pd(ctx, H_ptr, s_ptr, float(N0), float(rho2), x_ptr, stream)


def dp_precode_fd(ctx, H_ptr: int, s_ptr: int, N0: float, rho2: float, x_ptr: int, stream: int) -> int:
    return lib().dp_precode_fd(ctx, H_ptr, s_ptr, float(N0), float(rho2), x_ptr, stream)


def dp_precode_mrt(ctx, H_ptr: int, s_ptr: int, N0: float, rho2: float, x_ptr: int, stream: int) -> int:
    return lib().dp_precode_mrt(ctx, H_ptr, s_ptr, float(N0), float(rho2), x_ptr, stream)


def dp_set_clusters(ctx, B_c=None, power=None, tau=None, C=None) -> int:
    """Sequences of C cluster sizes / power shares / tau values (None = the default).  The C side
    reads exactly C entries of each array, so when C is given every sequence must have length C."""
    def arr(ct, v):
        if v is None:
            return None
        if C is not None and len(v) != C:
            raise ValueError(f"dp_set_clusters: got {len(v)} entries, need C={C}")
        return (ct * len(v))(*v)
    return lib().dp_set_clusters(ctx, arr(ctypes.c_int, B_c), arr(ctypes.c_double, power), arr(ctypes.c_double, tau))


def dp_read_scalars(ctx, which: int, dst_ptr: int, stream: int) -> int:
    return lib().dp_read_scalars(ctx, which, dst_ptr, stream)


def dp_status(ctx) -> tuple[int, int]:
    nb = ctypes.c_int(0)
    rc = lib().dp_status(ctx, ctypes.byref(nb))
    return rc, nb.value


def dp_profile_read(ctx, reset: bool = False):
    ms = (ctypes.c_double * DP_NUM_KERNELS)()
    n = (ctypes.c_longlong * DP_NUM_KERNELS)()
    check(lib().dp_profile_read(ctx, ms, n, int(reset)), "dp_profile_read")
    return list(ms), list(n)


def dp_launch_count(ctx) -> int:
    return int(lib().dp_launch_count(ctx))


def dp_comm_info(ctx) -> tuple[int, int]:
    """(ranks of the context's NCCL communicator or 0, linked NCCL version code)."""
    n, v = ctypes.c_int(0), ctypes.c_int(0)
    check(lib().dp_comm_info(ctx, ctypes.byref(n), ctypes.byref(v)), "dp_comm_info")
    return n.value, v.value


def dp_finalize(ctx) -> int:
    return lib().dp_finalize(ctx)


def dp_last_error() -> str:
    return lib().dp_last_error().decode(errors="replace")


def dp_debug_gram(ctx, H_ptr: int, per_cluster: bool, G_ptr: int, stream: int) -> int:
    return lib().dp_debug_gram(ctx, H_ptr, int(per_cluster), G_ptr, stream)


def dp_debug_solve(ctx, G_ptr: int, groups: int, s_ptr: int, kappa: float, rho_x2: float,
                   beta_ptr: int, z_ptr: int, stream: int) -> int:
    return lib().dp_debug_solve(ctx, G_ptr, groups, s_ptr, float(kappa), float(rho_x2), beta_ptr, z_ptr, stream)


def dp_synth_frame(seed: int, frame: int, n_sc: int, B: int, U: int, K: int, M: int, N0: float,
                   H_ptr: int, s_ptr: int, idx_ptr: int, noise_ptr: int, stream: int) -> int:
    return lib().dp_synth_frame(seed, frame, n_sc, B, U, K, M, float(N0), H_ptr, s_ptr, idx_ptr, noise_ptr, stream)


def dp_receive_count(n_sc: int, B: int, U: int, K: int, M: int, H_ptr: int, x_ptr: int, noise_ptr: int,
                     rx_ptr: int, idx_ptr: int, errors_ptr: int, stream: int) -> int:
    return lib().dp_receive_count(n_sc, B, U, K, M, H_ptr, x_ptr, noise_ptr, rx_ptr, idx_ptr, errors_ptr, stream)


def dp_prepare_pd(ctx, H_ptr: int, N0: float, rho2: float, stream: int) -> int:
    return lib().dp_prepare_pd(ctx, H_ptr, float(N0), float(rho2), stream)


def dp_prepare_fd(ctx, H_ptr: int, N0: float, rho2: float, stream: int) -> int:
    return lib().dp_prepare_fd(ctx, H_ptr, float(N0), float(rho2), stream)


def dp_apply(ctx, H_ptr: int, s_ptr: int, Ka: int, x_ptr: int, stream: int) -> int:
    return lib().dp_apply(ctx, H_ptr, s_ptr, Ka, x_ptr, stream)


def dp_comm_ledger(ctx, reset: bool = False) -> dict:
    out = (ctypes.c_longlong * DP_NUM_COMM)()
    check(lib().dp_comm_ledger(ctx, out, int(reset)), "dp_comm_ledger")
    return {k: int(out[i]) for i, k in enumerate(COMM_KINDS)}


def dp_prepare_from_gram(ctx, fd: bool, G_ptr: int, N0: float, rho2: float, stream: int) -> int:
    return lib().dp_prepare_from_gram(ctx, int(fd), G_ptr, float(N0), float(rho2), stream)
