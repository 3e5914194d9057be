"""Torch-facing wrapper of libdp.so: the public API a user of the method calls.

    pre = Precoder(n_sc=1200, B=256, U=32, K=14, C=8)
    x = pre.precode_pd(H, s, N0, rho2)     # PD-WF, Sec. III-B
    x = pre.precode_fd(H, s, N0, rho2)     # FD-WF, Sec. III-C

Tensors: H_local [n_sc][B/world][U], s [n_sc][K][U], x_local [n_sc][K][B/world],
complex64, contiguous (layouts in include/dp.h).  CUDA tensors run
asynchronously on the current torch stream; CPU tensors (pinned for speed) go
through the library's host staging path (H2D, compute, D2H inside the call).
PyTorch provides memory and streams only: every arithmetic step runs in the
CUDA kernels of libdp.so.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib as L


def _ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


class Precoder:
    def __init__(self, n_sc: int, B: int, U: int, K: int, C: int, *, rank: int = 0, world: int = 1,
                 device: int | None = None, Es: float = 1.0, tau: float = 0.125,
                 pd_topology: str = "allreduce", s_on_all_ranks: bool = True, flags: int = 0,
                 nccl_id: bytes | None = None):
        if device is None:
            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        self.n_sc, self.B, self.U, self.K, self.C = n_sc, B, U, K, C
        self.rank, self.world, self.device = rank, world, device
        self.Bl = B // world
        self.Cl = C // world
        self._id_buf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        cfg = L.DpConfig(n_sc=n_sc, B=B, U=U, K=K, C=C, rank=rank, world=world, device=device,
                         nccl_id=ctypes.cast(self._id_buf, ctypes.c_void_p) if self._id_buf is not None else None,
                         Es=Es, tau=tau,
                         pd_topology={"allreduce": L.DP_PD_ALLREDUCE, "reduce_bcast": L.DP_PD_REDUCE_BCAST,
                                      "scatter_gather": L.DP_PD_SCATTER_GATHER,
                                      "nvlink": L.DP_PD_NVLINK}[pd_topology],
                         s_on_all_ranks=int(s_on_all_ranks), flags=flags)
        self.cfg = cfg
        self.ctx = L.dp_init(cfg)
        self._last = None
        self._raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)

    # ------------------------------------------------------------ helpers
    def _check_io(self, H, s, x):
        want_H = (self.n_sc, self.Bl, self.U)
        want_s = (self.n_sc, self.K, self.U)
        want_x = (self.n_sc, self.K, self.Bl)
        for name, t, shape in (("H", H, want_H), ("s", s, want_s), ("x", x, want_x)):
            if t is None:
                continue
            if t.dtype != torch.complex64:
                raise TypeError(f"{name} must be complex64, got {t.dtype}")
            if tuple(t.shape) != shape:
                raise ValueError(f"{name} must have shape {shape}, got {tuple(t.shape)}")
            if not t.is_contiguous():
                raise ValueError(f"{name} must be contiguous")

    def _stream(self, stream):
        if stream is not None:
            return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        if self._raw_stream is not None:
            return self._raw_stream(self.device)          # torch's current stream, no Stream object
        if torch.cuda.is_available():
            return torch.cuda.current_stream(self.device).cuda_stream
        return 0

    def _alloc_x(self, H):
        return torch.empty((self.n_sc, self.K, self.Bl), dtype=torch.complex64, device=H.device,
                           pin_memory=(H.device.type == "cpu" and H.is_pinned()))

    def _run(self, fn, name, H, s, N0, rho2, out, stream):
        x = out if out is not None else self._alloc_x(H)
        self._check_io(H, s, x)
        sp = _ptr(s) if s is not None else None
        L.check(fn(self.ctx, _ptr(H), sp, N0, rho2, _ptr(x), self._stream(stream)), name)
        self._last = name
        return x

    # ------------------------------------------------------------ public API
    def precode_pd(self, H, s, N0: float, rho2: float = 1.0, out=None, stream=None):
        """PD-WF (Sec. III-B): x_c = H_c^H A^{-1} s / beta for all subcarriers/symbols."""
        return self._run(L.dp_precode_pd, "dp_precode_pd", H, s, N0, rho2, out, stream)

    def precode_fd(self, H, s, N0: float, rho2: float = 1.0, out=None, stream=None):
        """FD-WF (Sec. III-C): per-cluster WF with rho_c^2 = rho^2/C, kappa_c = tau U N0/rho_c^2."""
        return self._run(L.dp_precode_fd, "dp_precode_fd", H, s, N0, rho2, out, stream)

    def set_clusters(self, sizes=None, power=None, tau=None):
        """Unequal clusters B_c = w_c B, power shares rho_c^2 / rho^2 (P:215 footnote) and
        per-cluster tau_c (Eq. 9) for precode_fd / precode_mrt; sequences over all C clusters,
        None = the default (equal split, 1/C, the constructor's tau).  include/dp.h dp_set_clusters."""
        L.check(L.dp_set_clusters(self.ctx, None if sizes is None else [int(v) for v in sizes],
                                  None if power is None else [float(v) for v in power],
                                  None if tau is None else [float(v) for v in tau], C=self.C), "dp_set_clusters")

    # ------------------------------------------------------------ prepare / apply
    def prepare_pd(self, H, N0: float, rho2: float = 1.0, stream=None):
        """Cache W = A^{-1}/beta^WF for this channel (PD); then apply() per batch of symbols."""
        self._check_io(H, None, None)
        L.check(L.dp_prepare_pd(self.ctx, _ptr(H), N0, rho2, self._stream(stream)), "dp_prepare_pd")
        self._prepared = "dp_precode_pd"

    def prepare_fd(self, H, N0: float, rho2: float = 1.0, stream=None):
        """Cache W_c = A_c^{-1}/beta_c per cluster (FD); then apply() per batch of symbols."""
        self._check_io(H, None, None)
        L.check(L.dp_prepare_fd(self.ctx, _ptr(H), N0, rho2, self._stream(stream)), "dp_prepare_fd")
        self._prepared = "dp_precode_fd"

    def prepare_from_gram(self, G, mode: str, N0: float, rho2: float = 1.0, stream=None):
        """Prepare from a Gram already computed (uplink reuse): G [n_sc][U(U+1)/2] (PD) or
        [n_sc][C/world][U(U+1)/2] (FD), packed upper triangle (the layout debug_gram returns)."""
        fd = mode == "fd"
        L.check(L.dp_prepare_from_gram(self.ctx, fd, _ptr(G.contiguous()), N0, rho2, self._stream(stream)),
                "dp_prepare_from_gram")
        self._prepared = "dp_precode_fd" if fd else "dp_precode_pd"

    def apply(self, H, s, out=None, stream=None):
        """x_local = H_local^H W s for s [n_sc][Ka][U], 1 <= Ka <= K (the prepared mode's W)."""
        Ka = s.shape[1] if s is not None else self.K
        x = out if out is not None else torch.empty((self.n_sc, Ka, self.Bl), dtype=torch.complex64, device=H.device)
        L.check(L.dp_apply(self.ctx, _ptr(H), _ptr(s) if s is not None else None, Ka, _ptr(x), self._stream(stream)),
                "dp_apply")
        self._last = getattr(self, "_prepared", None)
        return x

    def precode_mrt(self, H, s, N0: float = 0.0, rho2: float = 1.0, out=None, stream=None):
        """Fully-distributed MRT baseline (Fig. 2): x_c = H_c^H s / beta_c per cluster."""
        x = self._run(L.dp_precode_mrt, "dp_precode_mrt", H, s, N0, rho2, out, stream)
        self._last = "dp_precode_fd"                      # per-cluster scalars, like FD
        return x

    def read_scalars(self, which: str, device="cuda", stream=None) -> torch.Tensor:
        """'beta' (PD [n_sc]; FD local [n_sc][C/world]), 'rx' [n_sc], 'power' [n_sc]."""
        w = {"beta": L.DP_SCALAR_BETA, "rx": L.DP_SCALAR_RX, "power": L.DP_SCALAR_POWER}[which]
        if which == "beta" and self._last == "dp_precode_fd":
            shape = (self.n_sc, self.Cl)
        else:
            shape = (self.n_sc,)
        dev = torch.device(device)
        dst = torch.empty(shape, dtype=torch.float32, device=dev)
        L.check(L.dp_read_scalars(self.ctx, w, _ptr(dst), self._stream(stream)), "dp_read_scalars")
        return dst

    def status(self) -> int:
        rc, nb = L.dp_status(self.ctx)
        if rc not in (L.DP_OK, L.DP_ERR_NUMERIC):
            L.check(rc, "dp_status")
        return nb

    def profile(self, reset: bool = False) -> dict:
        ms, n = L.dp_profile_read(self.ctx, reset)
        return {k: {"ms": ms[i], "launches": n[i]} for i, k in enumerate(L.KERNEL_NAMES)}

    def comm_ledger(self, reset: bool = False) -> dict:
        """fp32 payload elements this rank handed to each collective kind (include/dp.h DP_COMM_*)."""
        return L.dp_comm_ledger(self.ctx, reset)

    def comm_info(self) -> dict:
        """{'nranks': ranks of the library's NCCL communicator (0: none), 'nccl_version': code}."""
        n, v = L.dp_comm_info(self.ctx)
        return {"nranks": n, "nccl_version": v}

    def launch_count(self) -> int:
        return L.dp_launch_count(self.ctx)

    # ------------------------------------------------------------ debug steps (tests)
    def debug_gram(self, H, per_cluster: bool, stream=None) -> torch.Tensor:
        groups = self.Cl if per_cluster else 1
        G = torch.empty((self.n_sc, groups, self.U * (self.U + 1) // 2), dtype=torch.complex64, device=H.device)
        L.check(L.dp_debug_gram(self.ctx, _ptr(H), per_cluster, _ptr(G), self._stream(stream)), "dp_debug_gram")
        return G

    def debug_solve(self, G, s, kappa: float, rho_x2: float, stream=None):
        groups = G.shape[1]
        beta = torch.empty((self.n_sc, groups), dtype=torch.float32, device=G.device)
        z = torch.empty((self.n_sc, groups, self.K, self.U), dtype=torch.complex64, device=G.device)
        L.check(L.dp_debug_solve(self.ctx, _ptr(G.contiguous()), groups, _ptr(s), kappa, rho_x2, _ptr(beta),
                                 _ptr(z), self._stream(stream)), "dp_debug_solve")
        return beta, z

    def close(self):
        if getattr(self, "ctx", None) is not None and self.ctx.value:
            L.dp_finalize(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
