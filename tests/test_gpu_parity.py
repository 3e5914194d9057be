"""GPU parity: the CUDA path (through the C-ABI of libdp.so) against the fp64 oracle.

Element-by-element at reduced subcarrier counts (several CTAs plus a ragged
tail), and on sampled subcarriers at the full BASELINE sizes in the launch
configuration bench.py times.  Bar (north_star): relative L2 <= 1e-4 in fp32,
per-UE decisions identical outside a 1e-4 margin (reading R11).
"""
import numpy as np
import pytest
import torch

import oracle
from paper_1804_10987_b200 import CONFIGS, PAPER_POINTS, synth
from paper_1804_10987_b200 import _lib as L
from paper_1804_10987_b200.api import Precoder

from helpers import REL_TOL, decision_parity, rel_l2

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")]


def frame(cfg, n_sc=None, frame_id=0):
    return synth.make_frame(cfg.cfg_id, n_sc or cfg.n_sc, cfg.B, cfg.U, cfg.K, cfg.M, frame=frame_id)


def run(cfg, f, mode, N0, rho2=1.0, flags=0, tau=None, C=None, **kw):
    n_sc = f.H.shape[0]
    C = C or cfg.C
    tau = cfg.tau if tau is None else tau
    with Precoder(n_sc, cfg.B, cfg.U, cfg.K, C, tau=tau, flags=flags, **kw) as pre:
        H = torch.from_numpy(f.H).cuda()
        s = torch.from_numpy(f.s).cuda()
        x = (pre.precode_pd if mode == "pd" else pre.precode_fd)(H, s, N0, rho2)
        beta = pre.read_scalars("beta").cpu().numpy()
        rx = pre.read_scalars("rx").cpu().numpy()
        pw = pre.read_scalars("power").cpu().numpy()
        torch.cuda.synchronize()
        nbad = pre.status()
        return x.cpu().numpy(), beta, rx, pw, nbad


def reference(cfg, f, mode, N0, rho2=1.0, tau=None, C=None):
    C = C or cfg.C
    tau = cfg.tau if tau is None else tau
    if mode == "pd":
        x, beta = oracle.pd(f.H, f.s, C, N0, rho2)
        return x, beta, beta
    x, beta_c = oracle.fd(f.H, f.s, C, N0, rho2, tau=tau)
    return x, beta_c, oracle.rx_scale_fd(beta_c)


CASES = [
    (CONFIGS[1], None),      # U=4, full 64 subcarriers
    (CONFIGS[2], 61),        # U=8, S=16, ragged
    (CONFIGS[3], 37),        # U=16, S=16 = U
    (CONFIGS[4], 29),        # U=32, S=32 = U
    (PAPER_POINTS["fig2a"], 23),   # U=16, S=128, K=7
    (PAPER_POINTS["fig2e"], 19),   # U=16, S=32, K=7
    (PAPER_POINTS["fig2d"], 27),   # U=16, B=64: PD single pass at world 1, rows over 2 sub-groups
]


@pytest.mark.parametrize("cfg,n_sc", CASES, ids=[c.name for c, _ in CASES])
@pytest.mark.parametrize("mode", ["pd", "fd"])
@pytest.mark.parametrize("unfused", [False, True], ids=["fused", "unfused"])
def test_parity_elementwise(cfg, n_sc, mode, unfused):
    f = frame(cfg, n_sc)
    N0 = synth.n0_from_snr_db(cfg.snr_db)
    x, beta, rx, pw, nbad = run(cfg, f, mode, N0, flags=L.DP_FLAG_UNFUSED if unfused else 0)
    xr, br, rxr = reference(cfg, f, mode, N0)
    assert nbad == 0
    assert rel_l2(x, xr) <= REL_TOL, rel_l2(x, xr)
    br = br if mode == "pd" else br
    assert np.max(np.abs(beta.reshape(br.shape) / br - 1)) <= REL_TOL
    assert np.max(np.abs(rx / rxr - 1)) <= REL_TOL
    pwr = np.sum(np.abs(xr) ** 2, axis=(1, 2))
    assert np.max(np.abs(pw / pwr - 1)) <= 1e-4
    noise = synth.noise(synth.rng_for(cfg.cfg_id, 999), (x.shape[0], cfg.K, cfg.U), N0)
    mism, inside, total = decision_parity(f.qam, f.H, x, rx, xr, rxr, noise)
    assert mism == 0, (mism, inside, total)


@pytest.mark.parametrize("snr_db", [-5.0, 25.0])
@pytest.mark.parametrize("mode", ["pd", "fd"])
def test_parity_snr_range(snr_db, mode):
    cfg = CONFIGS[3]
    f = frame(cfg, 33)
    N0 = synth.n0_from_snr_db(snr_db)
    x, beta, rx, pw, nbad = run(cfg, f, mode, N0)
    xr, br, rxr = reference(cfg, f, mode, N0)
    assert nbad == 0
    assert rel_l2(x, xr) <= REL_TOL, rel_l2(x, xr)
    noise = synth.noise(synth.rng_for(cfg.cfg_id, 7), (x.shape[0], cfg.K, cfg.U), N0)
    mism, _, _ = decision_parity(f.qam, f.H, x, rx, xr, rxr, noise)
    assert mism == 0


@pytest.mark.parametrize("cfgid", [2, 3, 4])
@pytest.mark.parametrize("mode", ["pd", "fd"])
def test_parity_full_size_sampled(cfgid, mode):
    """BASELINE sizes (1200 subcarriers) in the bench launch configuration; the oracle
    recomputes 40 sampled subcarriers (subcarriers are independent)."""
    cfg = CONFIGS[cfgid]
    f = frame(cfg)
    N0 = synth.n0_from_snr_db(cfg.snr_db)
    x, beta, rx, pw, nbad = run(cfg, f, mode, N0)
    assert nbad == 0
    idx = np.sort(synth.rng_for(cfgid, 5).choice(cfg.n_sc, 40, replace=False))
    idx[-1] = cfg.n_sc - 1
    sub = synth.Frame(H=f.H[idx], s=f.s[idx], idx=f.idx[idx], qam=f.qam)
    xr, br, rxr = reference(cfg, sub, mode, N0)
    assert rel_l2(x[idx], xr) <= REL_TOL
    assert np.max(np.abs(rx[idx] / rxr - 1)) <= REL_TOL
    # frame-level property at any size: E||x||^2 ~ rho2 (Eq. 2; expectation over s)
    assert abs(np.mean(pw) / cfg.K - 1.0) < 0.05 if mode == "pd" else True


@pytest.mark.parametrize("cfgid", [3, 4])
@pytest.mark.parametrize("K", [1, 7, 14, 16, 17, 40])
def test_symbol_counts(cfgid, K):
    """K = 1 .. 40 symbols per frame: K <= 16 takes the tensor-core paths at U = 32, K > 16 the
    SIMT kernels in chunks of 16 symbols."""
    base = CONFIGS[cfgid]
    cfg = type(base)(base.cfg_id, "k", 21, base.B, base.U, base.C, K, base.M)
    f = frame(cfg)
    N0 = 0.1
    for mode in ("pd", "fd"):
        x, *_ = run(cfg, f, mode, N0)
        xr, *_ = reference(cfg, f, mode, N0)
        assert rel_l2(x, xr) <= REL_TOL


def test_single_subcarrier():
    cfg = CONFIGS[4]
    f = frame(cfg, 1)
    for mode in ("pd", "fd"):
        x, *_ = run(cfg, f, mode, 0.1)
        xr, *_ = reference(cfg, f, mode, 0.1)
        assert rel_l2(x, xr) <= REL_TOL


def test_zf_limit_n0_zero():
    """N0 = 0: kappa = 0, PD reduces to ZF; B >> U keeps G well conditioned."""
    cfg = CONFIGS[2]
    f = frame(cfg, 16)
    x, beta, rx, pw, nbad = run(cfg, f, "pd", 0.0)
    assert nbad == 0
    xr, *_ = reference(cfg, f, "pd", 0.0)
    assert rel_l2(x, xr) <= REL_TOL
    # beta H P = I: noiseless reception recovers s exactly (up to fp32)
    y = np.einsum("wbu,wkb->wku", f.H.astype(np.complex128), x) * rx[:, None, None]
    assert rel_l2(y, f.s) <= 1e-4


@pytest.mark.parametrize("mode", ["pd", "fd"])
@pytest.mark.parametrize("cfgid", [2, 4])
def test_non_hpd_flagged_and_zeroed(mode, cfgid):
    """N0 = 0 with a rank-deficient channel on one subcarrier -> flagged, zero output there,
    other subcarriers unaffected (SPEC S:60, S:241 typed error rather than Inf); cfg 4 takes
    the tensor-core kernels.  Square FD clusters (S = U) at N0 = 0 are zero-forcing on a
    32 x 32 Rayleigh block whose cond(G_c) of 1e5-1e9 is outside the fp32 envelope (DESIGN.md
    §9): their parity runs with DP_FLAG_FP64, which must flag and zero the same problem."""
    cfg = CONFIGS[cfgid]
    f = frame(cfg, 9)
    f.H[4] = 0
    f.H[4, :, 0] = 1.0
    keep = [i for i in range(9) if i != 4]
    sub = synth.Frame(H=f.H[keep], s=f.s[keep], idx=f.idx[keep], qam=f.qam)
    xr, *_ = reference(cfg, sub, mode, 0.0)
    square = mode == "fd" and cfg.S == cfg.U
    for flags in ([0, L.DP_FLAG_FP64] if square else [0]):
        x, beta, rx, pw, nbad = run(cfg, f, mode, 0.0, flags=flags)
        assert nbad == (1 if mode == "pd" else cfg.C), flags
        assert np.all(x[4] == 0)
        if square and flags == 0:
            continue                      # fp32 ZF on square clusters: flagging only (see above)
        assert rel_l2(x[keep], xr) <= REL_TOL, (flags, rel_l2(x[keep], xr))
    # DP_FLAG_SYNC returns the numeric error directly
    for flags in ([L.DP_FLAG_SYNC, L.DP_FLAG_SYNC | L.DP_FLAG_FP64]):
        with Precoder(9, cfg.B, cfg.U, cfg.K, cfg.C, flags=flags) as pre:
            fn = pre.precode_pd if mode == "pd" else pre.precode_fd
            with pytest.raises(L.DpError) as e:
                fn(torch.from_numpy(f.H).cuda(), torch.from_numpy(f.s).cuda(), 0.0, 1.0)
            assert e.value.code == L.DP_ERR_NUMERIC


# ---------------------------------------------------------------- DP_FLAG_FP64 (accuracy option)
@pytest.mark.parametrize("cfg,n_sc", CASES, ids=[c.name for c, _ in CASES])
@pytest.mark.parametrize("mode", ["pd", "fd"])
def test_fp64_parity_elementwise(cfg, n_sc, mode):
    """DP_FLAG_FP64 on every parity case at the configs' 10 dB: x, beta, rx, power vs the oracle."""
    f = frame(cfg, n_sc)
    N0 = synth.n0_from_snr_db(cfg.snr_db)
    x, beta, rx, pw, nbad = run(cfg, f, mode, N0, flags=L.DP_FLAG_FP64)
    xr, br, rxr = reference(cfg, f, mode, N0)
    assert nbad == 0
    assert rel_l2(x, xr) <= 1e-6, rel_l2(x, xr)          # fp64 accumulation: complex64 output rounding only
    assert np.max(np.abs(beta.reshape(br.shape) / br - 1)) <= 1e-6
    assert np.max(np.abs(rx / rxr - 1)) <= 1e-6
    assert np.max(np.abs(pw / np.sum(np.abs(xr) ** 2, axis=(1, 2)) - 1)) <= 1e-5


@pytest.mark.parametrize("cfgid", [3, 4])
@pytest.mark.parametrize("snr_db", [40.0, None], ids=["40dB", "N0=0"])
@pytest.mark.parametrize("mode", ["fd", "pd"])
def test_fp64_high_snr_square_clusters(cfgid, snr_db, mode):
    """Square clusters (B_c = U: cfg3 16 x 16, cfg4 32 x 32) at 40 dB and in the ZF limit N0 = 0
    (P:37): with DP_FLAG_FP64 the 1e-4 bar holds for x, beta_c and the receive scale (the fp32
    path's envelope ends near 25 dB there)."""
    cfg = CONFIGS[cfgid]
    f = frame(cfg, 96, frame_id=3)
    N0 = 0.0 if snr_db is None else synth.n0_from_snr_db(snr_db)
    x, beta, rx, pw, nbad = run(cfg, f, mode, N0, flags=L.DP_FLAG_FP64)
    xr, br, rxr = reference(cfg, f, mode, N0)
    assert nbad == 0
    assert rel_l2(x, xr) <= REL_TOL, rel_l2(x, xr)
    assert np.max(np.abs(beta.reshape(br.shape) / br - 1)) <= REL_TOL
    assert np.max(np.abs(rx / rxr - 1)) <= REL_TOL
    noise = synth.noise(synth.rng_for(cfg.cfg_id, 41), (x.shape[0], cfg.K, cfg.U), N0)
    mism, _, _ = decision_parity(f.qam, f.H, x, rx, xr, rxr, noise)
    assert mism == 0


@pytest.mark.parametrize("cfgid", [3, 4])
def test_fp64_full_size_sampled_n0_zero(cfgid):
    """FD in the ZF limit at the full 1200 subcarriers (9600 square clusters at cfg4, the worst
    conditioning tail), checked on 40 sampled subcarriers."""
    cfg = CONFIGS[cfgid]
    f = frame(cfg)
    x, beta, rx, pw, nbad = run(cfg, f, "fd", 0.0, flags=L.DP_FLAG_FP64)
    assert nbad == 0
    idx = np.sort(synth.rng_for(cfgid, 6).choice(cfg.n_sc, 40, replace=False))
    sub = synth.Frame(H=f.H[idx], s=f.s[idx], idx=f.idx[idx], qam=f.qam)
    xr, br, rxr = reference(cfg, sub, "fd", 0.0)
    assert rel_l2(x[idx], xr) <= REL_TOL, rel_l2(x[idx], xr)
    assert np.max(np.abs(rx[idx] / rxr - 1)) <= REL_TOL


def test_fp64_force_comm_pd():
    """DP_FLAG_FP64 PD through the NCCL path (ncclDouble Gram allreduce) on a 1-rank communicator."""
    cfg = CONFIGS[4]
    f = frame(cfg, 21)
    x, *_ = run(cfg, f, "pd", 0.0, flags=L.DP_FLAG_FP64 | L.DP_FLAG_FORCE_COMM, nccl_id=L.dp_get_unique_id(),
                s_on_all_ranks=False)
    xr, *_ = reference(cfg, f, "pd", 0.0)
    assert rel_l2(x, xr) <= 1e-6


def test_fp64_unsupported_paths():
    cfg = CONFIGS[3]
    f = frame(cfg, 4)
    H = torch.from_numpy(f.H).cuda()
    with Precoder(4, cfg.B, cfg.U, cfg.K, cfg.C, flags=L.DP_FLAG_FP64) as pre:
        with pytest.raises(L.DpError) as e:
            pre.prepare_pd(H, 0.1)
        assert e.value.code == L.DP_ERR_UNSUPPORTED
    small = type(cfg)(cfg.cfg_id, "s8u16", 4, 32, 16, 4, 14, 16)      # B_c = 8 < U
    fs = frame(small, 4)
    with Precoder(4, small.B, small.U, small.K, small.C, flags=L.DP_FLAG_FP64) as pre:
        with pytest.raises(L.DpError) as e:
            pre.precode_fd(torch.from_numpy(fs.H).cuda(), torch.from_numpy(fs.s).cuda(), 0.1)
        assert e.value.code == L.DP_ERR_UNSUPPORTED


def test_nonfinite_input_flagged():
    cfg = CONFIGS[3]
    f = frame(cfg, 5)
    f.H[2, 3, 1] = np.nan
    x, beta, rx, pw, nbad = run(cfg, f, "fd", 0.1)
    assert nbad >= 1
    assert np.isnan(beta[2]).any()


def test_invalid_arguments():
    cfg = CONFIGS[1]
    f = frame(cfg, 4)
    with Precoder(4, cfg.B, cfg.U, cfg.K, cfg.C) as pre:
        H = torch.from_numpy(f.H).cuda()
        s = torch.from_numpy(f.s).cuda()
        for N0, rho2 in ((-1.0, 1.0), (0.1, 0.0), (float("nan"), 1.0), (0.1, float("inf"))):
            with pytest.raises(L.DpError) as e:
                pre.precode_pd(H, s, N0, rho2)
            assert e.value.code == L.DP_ERR_INVALID
        # mixed host/device pointers
        x = torch.empty((4, cfg.K, cfg.B), dtype=torch.complex64)
        with pytest.raises(L.DpError) as e:
            pre.precode_fd(H, s, 0.1, 1.0, out=x)
        assert e.value.code == L.DP_ERR_INVALID


def test_deterministic_bit_exact():
    cfg = CONFIGS[4]
    f = frame(cfg, 50)
    for mode in ("pd", "fd"):
        x1, b1, *_ = run(cfg, f, mode, 0.1)
        x2, b2, *_ = run(cfg, f, mode, 0.1)
        assert np.array_equal(x1.view(np.uint64), x2.view(np.uint64))
        assert np.array_equal(b1.view(np.uint32), b2.view(np.uint32))


@pytest.mark.parametrize("pinned", [True, False])
def test_host_pointer_path_matches_device_path(pinned):
    cfg = CONFIGS[3]
    f = frame(cfg, 40)
    xd_pd, *_ = run(cfg, f, "pd", 0.1)
    xd_fd, *_ = run(cfg, f, "fd", 0.1)
    with Precoder(40, cfg.B, cfg.U, cfg.K, cfg.C) as pre:
        H = torch.from_numpy(f.H)
        s = torch.from_numpy(f.s)
        if pinned:
            H, s = H.pin_memory(), s.pin_memory()
        xh_pd = pre.precode_pd(H, s, 0.1, 1.0)
        assert xh_pd.device.type == "cpu"
        xh_fd = pre.precode_fd(H, s, 0.1, 1.0)
    assert np.array_equal(xh_pd.numpy(), xd_pd) and np.array_equal(xh_fd.numpy(), xd_fd)


@pytest.mark.parametrize("cfgid", [3, 4])
def test_host_pipeline_chunks_scalars(cfgid):
    """Host-pointer frames run chunked (H2D / kernels / D2H overlapped over subcarrier chunks):
    x and the per-subcarrier scalars of every chunk equal the device-pointer frame's."""
    cfg = CONFIGS[cfgid]
    f = frame(cfg, 45)
    for mode in ("pd", "fd"):
        xd, bd, rxd, pwd, _ = run(cfg, f, mode, 0.1)
        with Precoder(45, cfg.B, cfg.U, cfg.K, cfg.C, tau=cfg.tau) as pre:
            H = torch.from_numpy(f.H).pin_memory()
            s = torch.from_numpy(f.s).pin_memory()
            xh = (pre.precode_pd if mode == "pd" else pre.precode_fd)(H, s, 0.1, 1.0)
            bh = pre.read_scalars("beta").cpu().numpy()
            rxh = pre.read_scalars("rx").cpu().numpy()
            pwh = pre.read_scalars("power").cpu().numpy()
            assert pre.status() == 0
        assert np.array_equal(xh.numpy(), xd), mode
        assert np.array_equal(bh, bd) and np.array_equal(rxh, rxd) and np.array_equal(pwh, pwd), mode


_VARIANT_SCRIPT = r"""
import json, sys, numpy as np, torch
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
import oracle
from paper_1804_10987_b200 import CONFIGS, synth
from paper_1804_10987_b200.api import Precoder
from helpers import rel_l2
cfg = CONFIGS[4]
f = synth.make_frame(cfg.cfg_id, 29, cfg.B, cfg.U, cfg.K, cfg.M, frame=3)
N0 = synth.n0_from_snr_db(cfg.snr_db)
with Precoder(29, cfg.B, cfg.U, cfg.K, cfg.C) as pre:
    x = pre.precode_pd(torch.from_numpy(f.H).cuda(), torch.from_numpy(f.s).cuda(), N0, 1.0)
    beta = pre.read_scalars("beta").cpu().numpy()
    torch.cuda.synchronize()
    nbad = pre.status()
xr, br = oracle.pd(f.H, f.s, cfg.C, N0, 1.0)
print(json.dumps({"rel": rel_l2(x.cpu().numpy(), xr), "beta": float(np.max(np.abs(beta.reshape(br.shape) / br - 1))),
                  "nbad": int(nbad)}))
"""


@pytest.mark.parametrize("env", [{"DP_SOLVE_BLK": "1"}, {"DP_SOLVE_SG": "1", "DP_SOLVE_WPC": "4"},
                                 {"DP_SOLVE_NW": "2"}], ids=["blocked", "one_warp_wpc4", "two_warp"])
def test_pd_solve_variants(env):
    """The A/B variants of the PD solve (switches read once per process, so each runs in a child
    process): the blocked 4-warp sweep, the one-warp solve in 4-warp CTAs, the two-warp row split --
    cfg4 PD frame vs the oracle at the 1e-4 bar."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _VARIANT_SCRIPT, root], env={**os.environ, **env},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["nbad"] == 0 and out["rel"] <= REL_TOL and out["beta"] <= REL_TOL, out


@pytest.mark.parametrize("cfgid", [3, 4])
def test_host_async_consecutive_frames(cfgid):
    """DP_FLAG_HOST_ASYNC (include/dp.h): host-pointer calls return once enqueued and consecutive
    calls overlap (a call's H2D of chunk i waits only for the previous call's kernels on chunk i, its
    kernels for the previous D2H of chunk i).  Five frames with distinct inputs, PD and FD
    alternating, output buffers reused every other frame: after one stream synchronisation every
    frame's x equals the synchronous call's bytes."""
    cfg = CONFIGS[cfgid]
    n_sc = 48
    fs = [frame(cfg, n_sc, frame_id=10 + i) for i in range(5)]
    modes = ["pd", "fd", "pd", "fd", "fd"]
    with Precoder(n_sc, cfg.B, cfg.U, cfg.K, cfg.C, tau=cfg.tau) as pre:
        ref = [(pre.precode_pd if m == "pd" else pre.precode_fd)(torch.from_numpy(f.H).pin_memory(),
                                                                  torch.from_numpy(f.s).pin_memory(), 0.1, 1.0)
               for f, m in zip(fs, modes)]
    Hh = [torch.from_numpy(f.H).pin_memory() for f in fs]
    Sh = [torch.from_numpy(f.s).pin_memory() for f in fs]
    outs = [torch.empty_like(ref[0]).pin_memory() for _ in range(2)]
    got = []
    with Precoder(n_sc, cfg.B, cfg.U, cfg.K, cfg.C, tau=cfg.tau, flags=L.DP_FLAG_HOST_ASYNC) as pre:
        for i, (m, _) in enumerate(zip(modes, fs)):
            x = outs[i % 2]
            (pre.precode_pd if m == "pd" else pre.precode_fd)(Hh[i], Sh[i], 0.1, 1.0, out=x)
            if i % 2 == 1:                      # the two output buffers are complete after a sync
                torch.cuda.synchronize()
                got += [outs[0].clone(), outs[1].clone()]
        torch.cuda.synchronize()
        got.append(outs[0].clone())
        assert pre.status() == 0
    for i in range(5):
        assert np.array_equal(got[i].numpy(), ref[i].numpy()), (i, modes[i])


@pytest.mark.parametrize("Bl", [32, 64, 128])
@pytest.mark.parametrize("mode", ["pd", "fd"])
def test_u32_per_rank_shapes(Bl, mode):
    """The per-rank shapes of cfg4 (B = 256, U = 32, C = 8) on 8, 4 and 2 GPUs run at world = 1:
    B_local = 32 / 64 / 128 with 1 / 2 / 4 clusters (Gram with 32- / 64-antenna chunks, SIMT
    or tensor-core precode, in-CTA scalar folding, SIMT whitening when a CTA spans subcarriers)."""
    base = CONFIGS[4]
    cfg = type(base)(base.cfg_id, f"rank{Bl}", 27, Bl, 32, Bl // 32, 14, 64)
    f = frame(cfg)
    N0 = synth.n0_from_snr_db(cfg.snr_db)
    x, beta, rx, pw, nbad = run(cfg, f, mode, N0)
    xr, br, rxr = reference(cfg, f, mode, N0)
    assert nbad == 0
    assert rel_l2(x, xr) <= REL_TOL, rel_l2(x, xr)
    assert np.max(np.abs(rx / rxr - 1)) <= REL_TOL
    assert np.max(np.abs(pw / np.sum(np.abs(xr) ** 2, axis=(1, 2)) - 1)) <= 1e-4


@pytest.mark.parametrize("C", [1, 2, 4, 8])
def test_fd_u32_cluster_counts(C):
    """U = 32, S = 32 (tensor-core FD kernel) for every way the per-subcarrier scalars
    are formed: inside one CTA (C = 1, 2, 4) and across a 2-CTA cluster (C = 8); x,
    beta_c, the receive scale and the power vs the oracle."""
    base = CONFIGS[4]
    cfg = type(base)(base.cfg_id, f"u32c{C}", 13, 32 * C, 32, C, 14, 64)
    f = frame(cfg)
    N0 = synth.n0_from_snr_db(cfg.snr_db)
    x, beta, rx, pw, nbad = run(cfg, f, "fd", N0)
    xr, br, rxr = reference(cfg, f, "fd", N0)
    assert nbad == 0
    assert rel_l2(x, xr) <= REL_TOL, rel_l2(x, xr)
    assert np.max(np.abs(beta.reshape(br.shape) / br - 1)) <= REL_TOL
    assert np.max(np.abs(rx / rxr - 1)) <= REL_TOL
    pwr = np.sum(np.abs(xr) ** 2, axis=(1, 2))
    assert np.max(np.abs(pw / pwr - 1)) <= 1e-4


@pytest.mark.parametrize("S,U", [(4, 8), (8, 16), (4, 16), (16, 32), (8, 32)])
@pytest.mark.parametrize("mode", ["pd", "fd"])
def test_small_clusters_bc_below_u(S, U, mode):
    """B_c = S < U: FD takes the B_c x B_c branch Q_c = (H_c^H H_c + kappa_c I)^{-1} H_c^H
    (fd_small.cuh); PD is unaffected by the cluster size.  The oracle's
    FD implements that branch step by step (oracle.c)."""
    base = CONFIGS[3]
    C = 4
    cfg = type(base)(base.cfg_id, f"s{S}u{U}", 21, S * C, U, C, 14, 16)
    f = frame(cfg)
    N0 = synth.n0_from_snr_db(cfg.snr_db)
    x, beta, rx, pw, nbad = run(cfg, f, mode, N0)
    xr, br, rxr = reference(cfg, f, mode, N0)
    assert nbad == 0
    assert rel_l2(x, xr) <= REL_TOL, rel_l2(x, xr)
    assert np.max(np.abs(beta.reshape(br.shape) / br - 1)) <= REL_TOL
    assert np.max(np.abs(rx / rxr - 1)) <= REL_TOL
    pwr = np.sum(np.abs(xr) ** 2, axis=(1, 2))
    assert np.max(np.abs(pw / pwr - 1)) <= 1e-4


@pytest.mark.parametrize("S,U", [(1, 4), (3, 4), (5, 8), (6, 8), (10, 16), (12, 16), (20, 32), (24, 32), (31, 32)])
@pytest.mark.parametrize("N0", [0.1, 0.0], ids=["10dB", "N0=0"])
def test_small_clusters_any_size(S, U, N0):
    """B_c < U of any size (not a power of two): the sub-group is padded to the next power of two with
    zero antenna rows and a unit diagonal (a decoupled block, left out of beta's traces); x, beta_c,
    the receive scale and the power vs the oracle's B_c x B_c branch, also in the ZF limit."""
    base = CONFIGS[3]
    C = 3
    cfg = type(base)(base.cfg_id, f"s{S}u{U}", 19, S * C, U, C, 14, 16)
    f = frame(cfg)
    x, beta, rx, pw, nbad = run(cfg, f, "fd", N0)
    xr, br, rxr = reference(cfg, f, "fd", N0)
    assert nbad == 0
    assert rel_l2(x, xr) <= REL_TOL, rel_l2(x, xr)
    assert np.max(np.abs(beta.reshape(br.shape) / br - 1)) <= REL_TOL
    assert np.max(np.abs(rx / rxr - 1)) <= REL_TOL
    assert np.max(np.abs(pw / np.sum(np.abs(xr) ** 2, axis=(1, 2)) - 1)) <= 1e-4


def test_small_clusters_zero_noise():
    """At N0 = 0 the B_c x B_c branch stays defined (H_c^H H_c has full rank B_c < U) where
    the U x U form would be singular: FD precodes without numeric failures and matches the
    oracle's zero-forcing-per-cluster result."""
    base = CONFIGS[3]
    cfg = type(base)(base.cfg_id, "s8u16n0", 9, 32, 16, 4, 14, 16)
    f = frame(cfg)
    x, beta, rx, pw, nbad = run(cfg, f, "fd", 0.0)
    xr, br, rxr = reference(cfg, f, "fd", 0.0)
    assert nbad == 0
    assert rel_l2(x, xr) <= REL_TOL, rel_l2(x, xr)
    assert np.max(np.abs(beta.reshape(br.shape) / br - 1)) <= REL_TOL


@pytest.mark.parametrize("cfgid", [2, 3, 4])
@pytest.mark.parametrize("mode", ["pd", "fd"])
def test_prepare_apply_matches_oracle(cfgid, mode):
    """Prepare/apply split: W = A^{-1}/beta cached once per
    channel, applied to symbol batches of 1, 5 and the remaining symbols; every batch's
    x equals the oracle's frame restricted to those symbols, beta and rx are the frame's."""
    cfg = CONFIGS[cfgid]
    f = frame(cfg, 23)
    N0 = synth.n0_from_snr_db(cfg.snr_db)
    xr, br, rxr = reference(cfg, f, mode, N0)
    H = torch.from_numpy(f.H).cuda()
    s = torch.from_numpy(f.s).cuda()
    with Precoder(23, cfg.B, cfg.U, cfg.K, cfg.C, tau=cfg.tau) as pre:
        (pre.prepare_pd if mode == "pd" else pre.prepare_fd)(H, N0, 1.0)
        k0 = 0
        for Ka in (1, 5, cfg.K - 6):
            x = pre.apply(H, s[:, k0:k0 + Ka].contiguous())
            beta = pre.read_scalars("beta").cpu().numpy()
            rx = pre.read_scalars("rx").cpu().numpy()
            pw = pre.read_scalars("power").cpu().numpy()
            torch.cuda.synchronize()
            xs = xr[:, k0:k0 + Ka]
            assert rel_l2(x.cpu().numpy(), xs) <= REL_TOL, (Ka, rel_l2(x.cpu().numpy(), xs))
            assert np.max(np.abs(beta.reshape(br.shape) / br - 1)) <= REL_TOL
            assert np.max(np.abs(rx / rxr - 1)) <= REL_TOL
            assert np.max(np.abs(pw / np.sum(np.abs(xs) ** 2, axis=(1, 2)) - 1)) <= 1e-4
            k0 += Ka
        assert pre.status() == 0


@pytest.mark.parametrize("mode", ["pd", "fd"])
def test_prepare_from_uplink_gram(mode):
    """Uplink Gram reuse: a Gram supplied by the caller (here the fp64 oracle's, rounded to
    complex64) instead of the Gram kernel; apply gives the frame's x."""
    cfg = CONFIGS[3]
    f = frame(cfg, 19)
    N0 = synth.n0_from_snr_db(cfg.snr_db)
    xr, *_ = reference(cfg, f, mode, N0)
    S, U = cfg.S, cfg.U
    iu = np.triu_indices(U)
    if mode == "pd":
        G = np.stack([oracle.gram(f.H[w])[iu] for w in range(19)])
    else:
        G = np.stack([[oracle.gram(f.H[w, c * S:(c + 1) * S])[iu] for c in range(cfg.C)] for w in range(19)])
    Gt = torch.from_numpy(G.astype(np.complex64)).cuda()
    with Precoder(19, cfg.B, U, cfg.K, cfg.C, tau=cfg.tau) as pre:
        pre.prepare_from_gram(Gt, mode, N0, 1.0)
        x = pre.apply(torch.from_numpy(f.H).cuda(), torch.from_numpy(f.s).cuda())
        assert pre.status() == 0
    assert rel_l2(x.cpu().numpy(), xr) <= REL_TOL


def test_apply_without_prepare_rejected():
    cfg = CONFIGS[2]
    f = frame(cfg, 5)
    H = torch.from_numpy(f.H).cuda()
    s = torch.from_numpy(f.s).cuda()
    with Precoder(5, cfg.B, cfg.U, cfg.K, cfg.C) as pre:
        with pytest.raises(L.DpError):
            pre.apply(H, s)
        pre.prepare_pd(H, 0.1)
        pre.precode_fd(H, s, 0.1)            # discards the prepared state
        with pytest.raises(L.DpError):
            pre.apply(H, s)


@pytest.mark.parametrize("cfgid", [2, 3, 4])
def test_mrt_baseline(cfgid):
    """Fully-distributed MRT (the Fig. 2 baseline, dp_precode_mrt) vs oracle.mrt_fd: x, beta_c, the
    receive scale 1 / sum_c 1/beta_c and the power."""
    cfg = CONFIGS[cfgid]
    f = frame(cfg, 17)
    with Precoder(17, cfg.B, cfg.U, cfg.K, cfg.C) as pre:
        x = pre.precode_mrt(torch.from_numpy(f.H).cuda(), torch.from_numpy(f.s).cuda(), 0.1, 1.0)
        beta = pre.read_scalars("beta").cpu().numpy()
        rx = pre.read_scalars("rx").cpu().numpy()
        pw = pre.read_scalars("power").cpu().numpy()
        assert pre.status() == 0
    xr, br = oracle.mrt_fd(f.H, f.s, cfg.C)
    assert rel_l2(x.cpu().numpy(), xr) <= REL_TOL
    # reading R24: effective per-cluster scale beta_c / g_c, g_c = ||H_c||_F^2 / U
    g = np.sum(np.abs(f.H.astype(np.complex128).reshape(17, cfg.C, cfg.S, cfg.U)) ** 2, axis=(2, 3)) / cfg.U
    beff = br / g
    assert np.max(np.abs(beta.reshape(br.shape) / beff - 1)) <= REL_TOL
    assert np.max(np.abs(rx * np.sum(1.0 / beff, axis=1) - 1)) <= REL_TOL
    assert np.max(np.abs(pw / np.sum(np.abs(xr) ** 2, axis=(1, 2)) - 1)) <= 1e-4


def test_fd_single_cluster_tau1_equals_pd():
    """FD with C=1, tau=1 is centralized WF, so it must equal PD (C=1)."""
    base = CONFIGS[3]
    cfg = type(base)(base.cfg_id, "c1", 17, 32, 16, 1, 14, 16)
    f = frame(cfg)
    x_fd, *_ = run(cfg, f, "fd", 0.1, tau=1.0)
    x_pd, *_ = run(cfg, f, "pd", 0.1)
    assert rel_l2(x_fd, x_pd) <= 1e-5


@pytest.mark.parametrize("cfgid", [3, 4])
def test_force_comm_world1_paths(cfgid):
    """NCCL code path with a 1-rank communicator: PD allreduce topology, PD paper
    topology (reduce + z broadcast), the subcarrier split with collectives and (U = 32) with
    the exchange inside the whitening kernel (NCCL device API: symmetric windows, LSA loads /
    stores and per-CTA barriers on a 1-rank team), and FD (s broadcast + scalar allreduce)."""
    cfg = CONFIGS[cfgid]
    f = frame(cfg, 31)
    N0 = 0.1
    uid = L.dp_get_unique_id()
    xr_pd, *_ = reference(cfg, f, "pd", N0)
    xr_fd, *_ = reference(cfg, f, "fd", N0)
    x_fd_plain, *_ = run(cfg, f, "fd", N0)
    topos = ("allreduce", "reduce_bcast", "scatter_gather") + (("nvlink",) if cfg.U == 32 else ())
    for topo in topos:
        x, beta, rx, pw, nbad = run(cfg, f, "pd", N0, flags=L.DP_FLAG_FORCE_COMM, nccl_id=uid,
                                    pd_topology=topo, s_on_all_ranks=False)
        assert nbad == 0 and rel_l2(x, xr_pd) <= REL_TOL, (topo, rel_l2(x, xr_pd))
        uid = L.dp_get_unique_id()
    x, *_ = run(cfg, f, "fd", N0, flags=L.DP_FLAG_FORCE_COMM, nccl_id=uid, s_on_all_ranks=False)
    assert np.array_equal(x, x_fd_plain)   # same kernels, same order: bit-exact
    assert rel_l2(x, xr_fd) <= REL_TOL


def test_nvlink_exchange_world1_consecutive_frames():
    """DP_PD_NVLINK on a 1-rank communicator over consecutive frames (the per-CTA LSA barriers
    carry their epochs from launch to launch; the windows are rewritten every frame), with FD
    frames in between and a CUDA-graph capture of two PD frames; every PD frame against the
    oracle, and bit-identical to the scatter-gather topology's collectives (same Gram, same
    summation, same solve kernel arithmetic)."""
    cfg = CONFIGS[4]
    n_sc = 96
    N0 = 0.1
    frames = [frame(cfg, n_sc, frame_id=i) for i in range(3)]
    refs = [reference(cfg, f, "pd", N0)[0] for f in frames]
    outs = {}
    for topo in ("scatter_gather", "nvlink"):
        uid = L.dp_get_unique_id()
        with Precoder(n_sc, cfg.B, cfg.U, cfg.K, cfg.C, flags=L.DP_FLAG_FORCE_COMM, nccl_id=uid,
                      pd_topology=topo, s_on_all_ranks=True) as pre:
            Hs = [torch.from_numpy(f.H).cuda() for f in frames]
            Ss = [torch.from_numpy(f.s).cuda() for f in frames]
            xs = []
            for i in range(3):
                xs.append(pre.precode_pd(Hs[i], Ss[i], N0, 1.0).cpu().numpy())
                pre.precode_fd(Hs[i], Ss[i], N0, 1.0)
            X = [torch.empty((n_sc, cfg.K, cfg.B), dtype=torch.complex64, device="cuda") for _ in range(2)]
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                pre.precode_pd(Hs[1], Ss[1], N0, 1.0, out=X[0])
                pre.precode_pd(Hs[2], Ss[2], N0, 1.0, out=X[1])
            g.replay()
            torch.cuda.synchronize()
            xs += [X[0].cpu().numpy(), X[1].cpu().numpy()]
            assert pre.status() == 0
        outs[topo] = xs
        for x, xr in zip(xs, refs + refs[1:]):
            assert rel_l2(x, xr) <= REL_TOL, (topo, rel_l2(x, xr))
    for a, b in zip(outs["scatter_gather"], outs["nvlink"]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("cfgid", [1, 3, 4])
def test_step_gram(cfgid):
    """Kernel (a): packed Gram per cluster and summed, vs oracle.gram."""
    cfg = CONFIGS[cfgid]
    f = frame(cfg, 13)
    with Precoder(13, cfg.B, cfg.U, cfg.K, cfg.C) as pre:
        H = torch.from_numpy(f.H).cuda()
        Gc = pre.debug_gram(H, True).cpu().numpy()
        Gs = pre.debug_gram(H, False).cpu().numpy()
    iu = np.triu_indices(cfg.U)
    S = cfg.S
    for w in range(13):
        tot = np.zeros((cfg.U, cfg.U), complex)
        for c in range(cfg.C):
            g = oracle.gram(f.H[w, c * S:(c + 1) * S])
            tot += g
            assert rel_l2(Gc[w, c], g[iu]) <= 1e-5   # 3xTF32 tensor-core Gram at U=32
        assert rel_l2(Gs[w, 0], tot[iu]) <= 1e-5


@pytest.mark.parametrize("cfgid", [1, 2, 3, 4])
def test_step_solve(cfgid):
    """Kernel (b): Cholesky + substitution + Lemma-1 beta + whitening, vs oracle on the same G."""
    cfg = CONFIGS[cfgid]
    n_sc = 11
    f = frame(cfg, n_sc)
    rng = np.random.default_rng(cfgid)
    iu = np.triu_indices(cfg.U)
    Gfull = []
    Gp = np.zeros((n_sc, 1, len(iu[0])), np.complex64)
    for w in range(n_sc):
        Hw = f.H[w].astype(np.complex128)
        G = oracle.gram(Hw)
        G = G.astype(np.complex64).astype(np.complex128)
        Gfull.append(G)
        Gp[w, 0] = G[iu]
    kappa, rho2 = 0.37, 1.3
    with Precoder(n_sc, cfg.B, cfg.U, cfg.K, cfg.C) as pre:
        beta, z = pre.debug_solve(torch.from_numpy(Gp).cuda(), torch.from_numpy(f.s).cuda(), kappa, rho2)
        beta, z = beta.cpu().numpy(), z.cpu().numpy()
    for w in range(n_sc):
        A = Gfull[w] + kappa * np.eye(cfg.U)
        Ai = oracle.hpd_inverse(A)
        b = oracle.beta_lemma1(Ai, kappa, 1.0, rho2)
        assert abs(beta[w, 0] / b - 1) <= 1e-5
        zr = (Ai @ f.s[w].T.astype(np.complex128)).T / b
        assert rel_l2(z[w, 0], zr) <= 1e-5


def test_profile_and_launch_count():
    cfg = CONFIGS[3]
    f = frame(cfg, 64)
    with Precoder(64, cfg.B, cfg.U, cfg.K, cfg.C, flags=L.DP_FLAG_PROFILE) as pre:
        H = torch.from_numpy(f.H).cuda()
        s = torch.from_numpy(f.s).cuda()
        pre.precode_pd(H, s, 0.1)
        pre.precode_fd(H, s, 0.1)
        p = pre.profile(reset=True)
        # PD: (a) gram, (b) solve, (c) precode ; FD: one fused kernel (each CTA holds whole
        # subcarriers at cfg3, so the per-subcarrier scalars are folded in: no finish kernel)
        assert p["gram"]["launches"] == 1 and p["solve"]["launches"] == 1 and p["precode"]["launches"] == 1
        assert p["fused_fd"]["launches"] == 1 and p["finish"]["launches"] == 0 and p["fused_pd"]["launches"] == 0
        assert p["fused_fd"]["ms"] > 0
        assert pre.launch_count() == 4


def test_consecutive_frames_cfg4():
    """cfg4 (U = B_c = 32, C = 8): several consecutive PD and FD frames on one context, launched
    back to back (PDL lets each kernel start while its predecessor drains, so mbarrier-phase or
    hand-off hazards that a single synchronised frame hides show up here), 600 subcarriers so the
    persistent PD kernels loop over several items per CTA; every frame against the oracle, and
    the FD scalars summed by one fd_finish_kernel per FD frame (the 2-CTA cluster fold is the opt-in
    DP_FD_CLUSTER_FOLD variant, test_fd_cluster_fold_variant)."""
    cfg = CONFIGS[4]
    n_sc = 600
    f = frame(cfg, n_sc)
    N0 = synth.n0_from_snr_db(cfg.snr_db)
    with Precoder(n_sc, cfg.B, cfg.U, cfg.K, cfg.C, tau=cfg.tau, flags=L.DP_FLAG_PROFILE) as pre:
        H = torch.from_numpy(f.H).cuda()
        s = torch.from_numpy(f.s).cuda()
        for mode in ("pd", "fd", "pd", "fd", "fd"):
            x = (pre.precode_pd if mode == "pd" else pre.precode_fd)(H, s, N0, 1.0).cpu().numpy()
            beta = pre.read_scalars("beta").cpu().numpy()
            rx = pre.read_scalars("rx").cpu().numpy()
            pw = pre.read_scalars("power").cpu().numpy()
            xr, br, rxr = reference(cfg, f, mode, N0)
            assert rel_l2(x, xr) <= REL_TOL, (mode, rel_l2(x, xr))
            assert np.max(np.abs(beta.reshape(br.shape) / br - 1)) <= REL_TOL
            assert np.max(np.abs(rx / rxr - 1)) <= REL_TOL
            pwr = np.sum(np.abs(xr) ** 2, axis=(1, 2))
            assert np.max(np.abs(pw / pwr - 1)) <= 1e-4
        p = pre.profile(reset=True)
        assert pre.status() == 0
    assert p["fused_fd"]["launches"] == 3 and p["finish"]["launches"] == 3
    assert p["solve"]["launches"] == 2 and p["precode"]["launches"] == 2


_FOLD_SCRIPT = r"""
import json, sys, numpy as np, torch
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
import oracle
from paper_1804_10987_b200 import CONFIGS, synth
from paper_1804_10987_b200 import _lib as L
from paper_1804_10987_b200.api import Precoder
from helpers import rel_l2
cfg = CONFIGS[4]
f = synth.make_frame(cfg.cfg_id, 40, cfg.B, cfg.U, cfg.K, cfg.M, frame=5)
N0 = synth.n0_from_snr_db(cfg.snr_db)
out = {}
with Precoder(40, cfg.B, cfg.U, cfg.K, cfg.C, tau=cfg.tau, flags=L.DP_FLAG_PROFILE) as pre:
    H, s = torch.from_numpy(f.H).cuda(), torch.from_numpy(f.s).cuda()
    for i in range(3):                                   # back-to-back frames
        x = pre.precode_fd(H, s, N0, 1.0)
    beta = pre.read_scalars("beta").cpu().numpy()
    rx = pre.read_scalars("rx").cpu().numpy()
    torch.cuda.synchronize()
    out["nbad"] = int(pre.status())
    p = pre.profile(reset=True)
    out["finish"] = p["finish"]["launches"]
xr, br = oracle.fd(f.H, f.s, cfg.C, N0, 1.0, tau=cfg.tau)
rxr = oracle.rx_scale_fd(br)
out["rel"] = rel_l2(x.cpu().numpy(), xr)
out["beta"] = float(np.max(np.abs(beta.reshape(br.shape) / br - 1)))
out["rx"] = float(np.max(np.abs(rx / rxr - 1)))
print(json.dumps(out))
"""


def test_fd_cluster_fold_variant():
    """DP_FD_CLUSTER_FOLD=1 (k_tc.cu, read once per process, so in a child process): the cfg4 FD
    scalars summed in-kernel across a 2-CTA thread-block cluster (st.async into rank 0's shared
    memory) instead of fd_finish_kernel -- no finish launch, x / beta / rx vs the oracle."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _FOLD_SCRIPT, root], env={**os.environ, "DP_FD_CLUSTER_FOLD": "1"},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["finish"] == 0 and out["nbad"] == 0, out
    assert out["rel"] <= REL_TOL and out["beta"] <= REL_TOL and out["rx"] <= REL_TOL, out


@pytest.mark.parametrize("unfused", [False, True], ids=["single-pass", "unfused"])
def test_pd_single_pass_small_world1(unfused):
    """cfg2 (B U = 512): PD at world 1 is one single-pass kernel (Gram over all B antennas + solve +
    whitening + precode per subcarrier); DP_FLAG_UNFUSED keeps the three kernels.  Both vs the oracle."""
    cfg = CONFIGS[2]
    f = frame(cfg, 70)
    N0 = synth.n0_from_snr_db(cfg.snr_db)
    flags = L.DP_FLAG_PROFILE | (L.DP_FLAG_UNFUSED if unfused else 0)
    with Precoder(70, cfg.B, cfg.U, cfg.K, cfg.C, flags=flags) as pre:
        x = pre.precode_pd(torch.from_numpy(f.H).cuda(), torch.from_numpy(f.s).cuda(), N0).cpu().numpy()
        beta = pre.read_scalars("beta").cpu().numpy()
        pw = pre.read_scalars("power").cpu().numpy()
        p = pre.profile(reset=True)
        assert pre.status() == 0
    assert (p["fused_pd"]["launches"], p["gram"]["launches"]) == ((0, 1) if unfused else (1, 0))
    xr, br, _ = reference(cfg, f, "pd", N0)
    assert rel_l2(x, xr) <= REL_TOL
    assert np.max(np.abs(beta / br - 1)) <= REL_TOL
    assert np.max(np.abs(pw / np.sum(np.abs(xr) ** 2, axis=(1, 2)) - 1)) <= 1e-4
