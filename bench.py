"""bench.py — precoded Gbit/s and frame latency (device-timed) of PD-WF and FD-WF.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4|fig2a..fig2e] [--K 7]
                    [--impl ours|reference] [--mode both|pd|fd] [--fp64]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, NCCL)

Workload (BASELINE.json configs[3]): B=256 antennas, U=32 UEs,
C=8 clusters (S=32), N_sc=1200 subcarriers, K=14 OFDM symbols, 64-QAM, SNR
10 dB, tau=0.125.  A STEP is one pass of the whole hot path over one frame:
one PD-WF frame followed by one FD-WF frame, so
bits/step = 2 * N_sc * K * U * log2(M) for the whole job.  Scaling is STRONG
(the frame is fixed; clusters are sharded over the N GPUs, C/N per GPU).

Timing: W warm-up steps, then K steps (default 500 = 1000 frames, the steady
state of SURVEY §8(d)) bracketed by barrier + synchronize, CUDA events on the
launching stream, max over ranks.  Inputs rotate over R resident input sets
whose total size exceeds 2x L2 (126 MB), so every step reads H from HBM.
Single-frame latency p50 / p99 over 200 frames per precoder.  Rank 0 prints
ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "precoded Gbit/s and frame latency (device-timed) for PD/FD WF at 1/2/4/8 B200"
L2_BYTES = 126 * 1024 * 1024
SEED = 180410987
# builder-measured FP32 FFMA pipe peak (scripts/ffma2_probe.cu on the B200 pool, committed under
# profiles/); the fallback is the nominal clock product 148 SMs x 128 lanes x 2 flop x sm_max_mhz
FP32_PEAK_FILE = os.path.join(ROOT, "profiles", "fp32_peak.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="4", help="4 (default), 2, 3 or a paper point fig2a..fig2e")
    ap.add_argument("--K", type=int, default=0, help="override the symbols per frame (e.g. 7 to mirror the paper)")
    ap.add_argument("--rank-shape", type=int, default=0, help="world-1 run of one rank's shard of the config on N GPUs "
                    "(B/N antennas, C/N clusters): the per-rank shapes of the scaling curve")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="both", choices=["both", "pd", "fd"])
    ap.add_argument("--unfused", action="store_true", help="three-kernel path (a)(b)(c)")
    ap.add_argument("--fp64", action="store_true", help="DP_FLAG_FP64 accuracy option (fp64 accumulation)")
    ap.add_argument("--pd-topology", default="scatter_gather", choices=["allreduce", "reduce_bcast", "scatter_gather", "nvlink"],
                    help="PD exchange for N > 1 (DESIGN.md §6); scatter_gather splits the solve over the GPUs, nvlink "
                    "does the same with the exchange inside the whitening kernel (NVLink load/store, U = 32)")
    ap.add_argument("--force-comm", action="store_true", help="world 1: run the exchange path on a 1-rank NCCL "
                    "communicator (DP_FLAG_FORCE_COMM), e.g. to time --pd-topology nvlink against scatter_gather")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the sampled oracle check at N > 1")
    ap.add_argument("--latency-frames", type=int, default=200)
    ap.add_argument("--no-apply", action="store_true", help="skip the prepare/apply per-symbol latency")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target oracle CPU time for cpu_baseline")
    ap.add_argument("--profile-run", action="store_true", help="short run for ncu (no JSON extras)")
    ap.add_argument("--oracle-seconds", action="store_true", help="cpu_baseline leg only: fp64 oracle CPU seconds "
                    "for BASELINE configs[0] (cfg1) at OMP_NUM_THREADS=1 and at all cores (SURVEY §8(d))")
    ap.add_argument("--oracle-seconds-child", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--cluster-sizes", default="", help="comma list of C unequal cluster sizes B_c (dp_set_clusters, "
                    "P:157); FD only, power shares B_c / B")
    ap.add_argument("--eager", action="store_true", help="launch the timed steps eagerly (default: replay a CUDA "
                    "graph captured from the same K steps; host launch overhead out of the timed region)")
    return ap.parse_args()


def get_config(args):
    from paper_1804_10987_b200 import CONFIGS, PAPER_POINTS
    cfg = PAPER_POINTS[args.config] if args.config in PAPER_POINTS else CONFIGS[int(args.config)]
    if args.K:
        cfg = type(cfg)(cfg.cfg_id, f"{cfg.name}_K{args.K}", cfg.n_sc, cfg.B, cfg.U, cfg.C, args.K, cfg.M,
                        cfg.snr_db, cfg.tau)
    if args.rank_shape:
        n = args.rank_shape
        cfg = type(cfg)(cfg.cfg_id, f"{cfg.name}_rankshape{n}", cfg.n_sc, cfg.B // n, cfg.U, cfg.C // n, cfg.K,
                        cfg.M, cfg.snr_db, cfg.tau)
    return cfg


# ---------------------------------------------------------------- algorithmic work
def flops_problem(U: int, nb: int, K: int) -> dict:
    """Algorithmic real flops of one WF problem (one subcarrier x one cluster for FD, one
    subcarrier over nb antennas for PD); complex MAC = 8 flops.
    Gram: Hermitian half U(U+1)/2 entries x nb ; Cholesky U^3/6 ; L^-1 U^3/6 ; A^-1 = W0^H W0 U^3/6 ;
    whiten K U^2 ; precode K nb U.  For nb < U (FD branch B_c < U) the same terms in the
    nb x nb space: Gram U nb(nb+1)/2, solve nb^3/2, H^H s K nb U, apply W K nb^2."""
    if nb < U:
        cmac = {"gram": U * nb * (nb + 1) / 2, "solve": nb ** 3 / 2, "whiten": K * nb * nb, "precode": K * nb * U}
    else:
        cmac = {"gram": nb * U * (U + 1) / 2, "solve": U ** 3 / 2, "whiten": K * U * U, "precode": K * nb * U}
    return {k: 8.0 * v for k, v in cmac.items()}


def bytes_frame(cfg, Bl: int) -> dict:
    """Algorithmic HBM bytes per frame per GPU: H read once, s read once, x written once."""
    return {"H": cfg.n_sc * Bl * cfg.U * 8, "s": cfg.n_sc * cfg.K * cfg.U * 8, "x": cfg.n_sc * cfg.K * Bl * 8}


def load_peaks():
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        pass
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    fp32 = {"tflops": 148 * 128 * 2 * sm_max * 1e6 / 1e12, "source": f"nominal: 148 SMs x 128 lanes x 2 x {sm_max:.0f} MHz"}
    fp64 = {"tflops": fp32["tflops"] / 2, "source": "nominal: half the FP32 rate"}
    try:
        with open(FP32_PEAK_FILE) as f:
            m = json.load(f)
        fp32 = {"tflops": float(m["ffma_tflops"]), "source": f"builder-measured ({m['how']})"}
        if "dfma_tflops" in m:
            fp64 = {"tflops": float(m["dfma_tflops"]), "source": f"builder-measured ({m['how']})"}
    except Exception:
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    bf16 = float(peaks.get("bf16_tflops", 1590.0))
    # tf32 dense peak: the measured bf16 peak x the nominal tf32 / bf16 ratio (1.1 / 2.25 PFLOP/s)
    tf32 = bf16 * 1.1 / 2.25
    return {"fp32": fp32, "fp64": fp64, "hbm_gbs": hbm, "tf32_tflops": tf32,
            "hbm_source": "MEASURED_PEAKS.json hbm_gbs (of measured)" if "hbm_gbs" in peaks else "fallback 6650 GB/s"}


# ---------------------------------------------------------------- clocks sampler
class Clocks:
    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.device), "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return self

        def rd():
            for line in self.proc.stdout:
                self.rows.append([c.strip() for c in line.split(",")])

        self.thread = threading.Thread(target=rd, daemon=True)
        self.thread.start()
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ---------------------------------------------------------------- oracle CPU baseline
def _oracle_step(cfg, f, N0, modes=("pd", "fd")):
    import oracle

    if "pd" in modes:
        oracle.pd(f.H, f.s, cfg.C, N0)
    if "fd" in modes:
        oracle.fd(f.H, f.s, cfg.C, N0, tau=cfg.tau)


def cpu_baseline(cfg, target_s: float, modes, chunk: int = 96):
    """The fp64 oracle (oracle/, as it stands) on a bounded sample of the same workload:
    a chunk of `chunk` subcarriers of one frame (the bench's precoders), repeated until ~target_s
    of CPU work, on all host cores (OpenMP over subcarriers)."""
    import oracle
    from paper_1804_10987_b200 import synth

    N0 = synth.n0_from_snr_db(cfg.snr_db)
    f = synth.make_frame(cfg.cfg_id, chunk, cfg.B, cfg.U, cfg.K, cfg.M, frame=77)
    _oracle_step(cfg, f, N0, modes)               # warm (page-in, thread pool)
    reps, t0 = 0, time.perf_counter()
    while True:
        _oracle_step(cfg, f, N0, modes)
        reps += 1
        el = time.perf_counter() - t0
        if el >= target_s or reps >= 10000:
            break
    bits = len(modes) * reps * chunk * cfg.K * cfg.U * (cfg.M.bit_length() - 1)
    return {"value": bits / el / 1e9, "unit": "Gbit/s", "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"{reps} x {chunk} subcarriers of {cfg.name} ({'+'.join(m.upper() for m in modes)} frames, "
                      f"fp64 C oracle, OpenMP over subcarriers), {el:.1f} s"}


def oracle_seconds_child(reps: int = 5):
    """One process of --oracle-seconds: cfg1 PD + FD frames through the oracle, median of `reps`."""
    import oracle
    from paper_1804_10987_b200 import CONFIGS, synth
    cfg = CONFIGS[1]
    N0 = synth.n0_from_snr_db(cfg.snr_db)
    f = synth.make_frame(cfg.cfg_id, cfg.n_sc, cfg.B, cfg.U, cfg.K, cfg.M)
    _oracle_step(cfg, f, N0)
    ts = {"pd": [], "fd": []}
    for _ in range(reps):
        for m in ("pd", "fd"):
            t = time.perf_counter()
            _oracle_step(cfg, f, N0, (m,))
            ts[m].append(time.perf_counter() - t)
    print(json.dumps({"threads": oracle.num_threads(), **{m: statistics.median(v) for m, v in ts.items()}}))


def oracle_seconds():
    """BASELINE configs[0] ("fp64 oracle (CPU seconds)"): cfg1 frames at 1 thread and at all cores."""
    out = {"workload": "cfg1: B=16 U=4 C=2 N_sc=64 K=1 QPSK, one PD-WF and one FD-WF frame", "runs": []}
    for n in (1, os.cpu_count() or 1):
        env = dict(os.environ, OMP_NUM_THREADS=str(n))
        r = subprocess.run([sys.executable, os.path.abspath(__file__), "--oracle-seconds-child"], env=env,
                           capture_output=True, text=True, check=True)
        d = json.loads(r.stdout.strip().splitlines()[-1])
        d["cpu_seconds_frame_pd"], d["cpu_seconds_frame_fd"] = d.pop("pd"), d.pop("fd")
        out["runs"].append(d)
    try:
        out["cpu_model"] = next(l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name"))
    except Exception:
        pass
    out["nproc"] = os.cpu_count()
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------- reference arm
def run_reference(args, cfg, rank, world):
    """--impl reference: the oracle as it stands on the host cores (rank 0 only); each step
    is a bounded sample of the workload (a chunk of subcarriers, PD + FD)."""
    if rank != 0:
        return
    import oracle
    from paper_1804_10987_b200 import synth

    N0 = synth.n0_from_snr_db(cfg.snr_db)
    modes = ["pd", "fd"] if args.mode == "both" else [args.mode]
    chunk = 48
    f = synth.make_frame(cfg.cfg_id, chunk, cfg.B, cfg.U, cfg.K, cfg.M, frame=78)
    # bounded: the default 500 timed steps would run for minutes on the oracle; at most 20 steps
    steps = min(args.steps, 20)
    warm = min(args.warmup, 3)
    for _ in range(warm):
        _oracle_step(cfg, f, N0, modes)
    t = time.perf_counter()
    for _ in range(steps):
        _oracle_step(cfg, f, N0, modes)
    el = time.perf_counter() - t
    bits = len(modes) * chunk * cfg.K * cfg.U * (cfg.M.bit_length() - 1) * steps
    v = bits / el / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "Gbit/s", "n_gpus": world,
            "steps": steps, "warmup": warm, "ms_per_step": el / steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "complex128",
            "data": "synthetic",
            "config": {"workload": cfg.name, "step": f"{'+'.join(m.upper() for m in modes)} frames on {chunk} of "
                                                      f"{cfg.n_sc} subcarriers",
                       "steps_requested": args.steps},
            "cpu_baseline": {"value": v, "unit": "Gbit/s", "cores": oracle.num_threads(), "kind": "oracle",
                             "sample": f"{chunk} of {cfg.n_sc} subcarriers per step"},
            "e2e": {"value": v, "unit": "Gbit/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- roofline
def fd_pipes(cfg, U, S, K, n_problems, kernel_path):
    """Split the §8(d) algorithmic FD flops by the pipe each step runs on, for the kernel that ran."""
    fl = flops_problem(U, S, K)
    tot = {k: v * n_problems for k, v in fl.items()}
    if kernel_path == "fd_tc+wtc":                   # Gram and whitening on tcgen05 (3xTF32)
        tensor, simt = ["gram", "whiten"], ["solve", "precode"]
    elif kernel_path == "fd_tc":
        tensor, simt = ["gram"], ["solve", "whiten", "precode"]
    else:
        tensor, simt = [], ["gram", "solve", "whiten", "precode"]
    return tot, sum(tot[k] for k in tensor), sum(tot[k] for k in simt), tensor, simt


def roofline(cfg, world, prof, ms_prof, ms_step_unprof, steps, peaks, sizes, fp64, modes):
    Bl = cfg.B // world
    Cl = cfg.C // world
    bf = bytes_frame(cfg, Bl)
    fp32 = peaks["fp32"]["tflops"]
    hbm = peaks["hbm_gbs"]
    pipe = peaks["fp64"] if fp64 else peaks["fp32"]
    npk = cfg.U * (cfg.U + 1) // 2 * 8
    flp = flops_problem(cfg.U, Bl, cfg.K)
    # which FD kernel ran (dp_api.cu dispatch): fd_tc at U = B_c = 32, K <= 16 (tensor-core whitening when
    # a CTA's 4 problems share the subcarrier), the SIMT fused kernel otherwise, fd_f64 with --fp64
    if fp64:
        fd_path = "fd_f64"
    elif cfg.U == 32 and cfg.S == 32 and cfg.K <= 16:
        fd_path = "fd_tc+wtc" if Cl % 4 == 0 else "fd_tc"
    else:
        fd_path = "fd_fused" if cfg.S >= cfg.U else "fd_small"
    per = {}
    for k, v in prof.items():
        if not v["launches"]:
            continue
        kms = v["ms"] / v["launches"]
        e = {"ms_avg": kms, "launches": v["launches"]}
        if k == "gram":
            b = bf["H"] + cfg.n_sc * npk
            e.update(bound="hbm", bytes=b, achieved_gbs=b / (kms / 1e3) / 1e9, frac=b / (kms / 1e3) / 1e9 / hbm)
        elif k == "precode":
            b = bf["H"] + bf["s"] + bf["x"]
            e.update(bound="hbm", bytes=b, achieved_gbs=b / (kms / 1e3) / 1e9, frac=b / (kms / 1e3) / 1e9 / hbm)
        elif k == "solve":
            f_ = cfg.n_sc * (flp["solve"] + flp["whiten"])
            e.update(bound="alu", flops=f_, achieved_tflops=f_ / (kms / 1e3) / 1e12,
                     frac=f_ / (kms / 1e3) / 1e12 / pipe["tflops"],
                     note="1 U x U problem per subcarrier: latency-bound (SURVEY §8(d): reported, not graded)")
        elif k == "fused_pd":                        # PD single pass at world 1 (U < 32): all on the FP32 pipe
            allf = cfg.n_sc * sum(flp.values())
            b = bf["H"] + bf["s"] + bf["x"]
            t = kms / 1e3
            e.update(bound="alu", kernel_path="fd_fused(S=B)", method_flops=allf,
                     achieved_tflops=allf / t / 1e12, frac=allf / t / 1e12 / pipe["tflops"],
                     pipes={"simt_steps": ["gram", "solve", "whiten", "precode"], "simt_flops": allf,
                            "simt_frac": allf / t / 1e12 / pipe["tflops"], "hbm_bytes": b,
                            "hbm_frac": b / t / 1e9 / hbm})
        elif k == "fused_fd" and not sizes:
            tot, tflops, sflops, tn, sn = fd_pipes(cfg, cfg.U, cfg.S, cfg.K, cfg.n_sc * Cl, fd_path)
            allf = sum(tot.values())
            b = bf["H"] + bf["s"] + bf["x"]
            t = kms / 1e3
            e.update(bound="alu", kernel_path=fd_path, method_flops=allf,
                     achieved_tflops=allf / t / 1e12, frac=allf / t / 1e12 / pipe["tflops"],
                     pipes={"simt_steps": sn, "simt_flops": sflops, "simt_frac": sflops / t / 1e12 / pipe["tflops"],
                            "tensor_steps": tn, "tensor_flops_3xtf32": 3 * tflops,
                            "tensor_frac": 3 * tflops / t / 1e12 / peaks["tf32_tflops"],
                            "hbm_bytes": b, "hbm_frac": b / t / 1e9 / hbm})
        else:
            e.update(bound="latency", note="per-subcarrier scalar combine")
        per[k] = e
    # dominant kernel (or the whole FD frame for unequal clusters: its runs overlap on streams)
    if sizes:
        fl_tot = 0.0
        for bc in sizes[cfg.C // world * 0: cfg.C // world * 0 + Cl] if world > 1 else sizes:
            fl_tot += sum(flops_problem(cfg.U, bc, cfg.K).values()) * cfg.n_sc
        t = ms_step_unprof / 1e3
        return {"bound": "alu", "achieved": fl_tot / t / 1e12, "peak": pipe["tflops"], "unit": "TFLOP/s",
                "frac": fl_tot / t / 1e12 / pipe["tflops"], "traffic": None, "kernel": "fd_frame(unequal runs)",
                "kernel_ms_avg": ms_step_unprof, "kernel_share_of_step": 1.0,
                "kernel_timing": "unprofiled FD frame time (its runs overlap on up to 3 streams)",
                "algorithmic_flops_per_launch": fl_tot, "peak_note": pipe["source"], "per_kernel": per}
    dom = max(per, key=lambda k: per[k]["ms_avg"] * per[k]["launches"])
    d = per[dom]
    share = prof[dom]["ms"] / max(ms_prof, 1e-9)
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(f"{cfg.name}/{dom}/n{world}")
    except Exception:
        pass
    timing = ("CUDA events around each launch on its stream, in a second pass of the same "
              f"{steps} steps (profiled step {ms_prof / steps:.4f} ms vs {ms_step_unprof:.4f} ms unprofiled: events "
              "between kernels break the PDL overlap)")
    if d["bound"] == "hbm":
        r = {"bound": "hbm", "achieved": d["achieved_gbs"], "peak": hbm, "unit": "GB/s", "frac": d["frac"],
             "algorithmic_bytes_per_launch": d["bytes"], "peak_note": peaks["hbm_source"]}
    else:
        f_ = d.get("method_flops", d.get("flops", 0.0))
        r = {"bound": "alu", "achieved": f_ / (d["ms_avg"] / 1e3) / 1e12, "peak": pipe["tflops"], "unit": "TFLOP/s",
             "frac": f_ / (d["ms_avg"] / 1e3) / 1e12 / pipe["tflops"], "algorithmic_flops_per_launch": f_,
             "algorithmic_bytes_per_launch": bf["H"] + bf["s"] + bf["x"],
             "peak_note": ("FP64 DFMA pipe, " if fp64 else "FP32 FFMA pipe, ") + pipe["source"] +
                          "; achieved = the §8(d) whole-method flops of the launch (Gram + solve + whitening + "
                          "precode, wherever each runs) / its time; per_kernel[...].pipes splits them by pipe"}
    r.update(traffic=traffic, kernel=dom, kernel_ms_avg=d["ms_avg"], kernel_share_of_step=share,
             kernel_timing=timing, per_kernel=per)
    return r


# ---------------------------------------------------------------- N > 1: sampled parity vs the oracle
def parity_check(pre, cfg, world, rank, dev, Hs, Ss, modes, N0, nsamp=8):
    """Verification leg (not on the product path): every rank precodes one resident input set, the
    sampled subcarriers' H_local / x_local are gathered to rank 0, which recomputes them with the fp64
    oracle (subcarriers are independent).  Reported as relative L2 per precoder."""
    import numpy as np
    import torch
    import torch.distributed as dist

    idx = torch.linspace(0, cfg.n_sc - 1, nsamp, device=dev).round().long()
    out = {}
    for m in modes:
        x = (pre.precode_pd if m == "pd" else pre.precode_fd)(Hs[0], Ss[0], N0, 1.0)
        torch.cuda.synchronize(dev)
        hs = Hs[0][idx].contiguous()
        xs = x[idx].contiguous()
        if world > 1:
            hp = [torch.empty_like(hs) for _ in range(world)]
            xp = [torch.empty_like(xs) for _ in range(world)]
            dist.all_gather(hp, hs)
            dist.all_gather(xp, xs)
            hs, xs = torch.cat(hp, dim=1), torch.cat(xp, dim=2)
        if rank == 0:
            import oracle
            H = hs.cpu().numpy()
            s = Ss[0][idx].cpu().numpy()
            if m == "pd":
                xr, _ = oracle.pd(H, s, cfg.C, N0)
            else:
                xr, _ = oracle.fd(H, s, cfg.C, N0, tau=cfg.tau)
            xg = xs.cpu().numpy().astype(np.complex128)
            out[m] = float(np.linalg.norm(xg - xr) / np.linalg.norm(xr))
    if rank == 0:
        out["subcarriers"] = [int(v) for v in idx.tolist()]
        out["tol"] = 1e-4
        out["ok"] = all(out[m] <= 1e-4 for m in modes)
    return out


# ---------------------------------------------------------------- ours
def main():
    args = parse()
    if args.oracle_seconds_child:
        oracle_seconds_child()
        return
    if args.oracle_seconds:
        oracle_seconds()
        return
    cfg = get_config(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and world > 1:
        print(f"--gpus {args.gpus} != WORLD_SIZE {world}", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import torch
    import torch.distributed as dist

    from paper_1804_10987_b200 import _lib as L
    from paper_1804_10987_b200 import dist as D
    from paper_1804_10987_b200 import synth
    from paper_1804_10987_b200.api import Precoder

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if cfg.C % world:
        raise SystemExit(f"C={cfg.C} not divisible by {world} GPUs")
    Bl = cfg.B // world
    N0 = synth.n0_from_snr_db(cfg.snr_db)

    # Two contexts: `pre` times `value` with nothing between the kernels (events between
    # launches would break the programmatic-dependent-launch overlap), `pre_prof`
    # (DP_FLAG_PROFILE: CUDA events around every kernel, on the launching stream) runs the
    # same steps right after it for the per-kernel times of the roofline.
    flags = (L.DP_FLAG_UNFUSED if args.unfused else 0) | (L.DP_FLAG_FP64 if args.fp64 else 0)
    force = world == 1 and args.force_comm
    flags |= L.DP_FLAG_FORCE_COMM if force else 0
    mk = lambda fl: Precoder(cfg.n_sc, cfg.B, cfg.U, cfg.K, cfg.C, rank=rank, world=world, device=local,  # noqa: E731
                             tau=cfg.tau, pd_topology=args.pd_topology, s_on_all_ranks=(world == 1), flags=fl,
                             nccl_id=D.bootstrap_nccl_id() if world > 1 else (L.dp_get_unique_id() if force else None))
    pre = mk(flags)
    pre_prof = mk(flags | L.DP_FLAG_PROFILE)

    sizes = [int(v) for v in args.cluster_sizes.split(",")] if args.cluster_sizes else None
    if sizes:
        if len(sizes) != cfg.C:
            raise SystemExit(f"--cluster-sizes needs C={cfg.C} entries, got {len(sizes)}")
        if args.mode != "fd":
            raise SystemExit("--cluster-sizes applies to FD only: use --mode fd")
        for p_ in (pre, pre_prof):
            p_.set_clusters(sizes, [b / cfg.B for b in sizes])

    # ---------------- resident rotating input sets (> 2x L2 in total)
    bf = bytes_frame(cfg, Bl)
    per_set = bf["H"] + bf["s"] + bf["x"]
    R = max(3, math.ceil(2 * L2_BYTES / per_set))
    gen = torch.Generator(device=dev)
    gen.manual_seed(SEED + 1000 * cfg.cfg_id + rank)
    pts = torch.from_numpy(synth.QAM(cfg.M).points().astype("complex64")).to(dev)
    Hs, Ss, Xs = [], [], []
    for r in range(R):
        h = torch.randn((cfg.n_sc, Bl, cfg.U, 2), generator=gen, device=dev) * math.sqrt(0.5)
        Hs.append(torch.view_as_complex(h.contiguous()))
        idx = torch.randint(0, cfg.M, (cfg.n_sc, cfg.K, cfg.U), generator=gen, device=dev)
        Ss.append(pts[idx].contiguous())
        Xs.append(torch.empty((cfg.n_sc, cfg.K, Bl), dtype=torch.complex64, device=dev))
    stream = torch.cuda.current_stream(dev)

    modes = ["pd", "fd"] if args.mode == "both" else [args.mode]

    def step(i, p=None):
        # each frame of the step gets its own input set (the PD and the FD frame of a step never
        # share H, so FD cannot read the H that PD just pulled into L2)
        p = p or pre
        for q, m in enumerate(modes):
            j = (len(modes) * i + q) % R
            fn = p.precode_pd if m == "pd" else p.precode_fd
            fn(Hs[j], Ss[j], N0, 1.0, out=Xs[j])

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize(dev)

    for i in range(args.warmup):
        step(i)
        step(i, pre_prof)
    barrier()
    pre_prof.profile(reset=True)
    if args.profile_run:
        for i in range(args.steps):
            step(i, pre_prof)
        torch.cuda.synchronize(dev)
        if rank == 0:
            print(json.dumps({"profile_run": True, "profile": pre_prof.profile()}))
        pre.close()
        pre_prof.close()
        if world > 1:
            dist.destroy_process_group()
        return

    # ---------------- timed region: the K steps captured once into a CUDA graph (the library's
    # launches carry their PDL attributes into programmatic graph edges; NCCL calls are capturable)
    # and replayed, or launched eagerly (--eager, or if capture is refused)
    launches0 = pre.launch_count()
    pre.comm_ledger(reset=True)
    graph, launch_mode = None, "eager"
    if not args.eager:
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for i in range(args.steps):
                    step(args.warmup + i)
            g.replay()                                   # untimed warm replay
            barrier()
            graph, launch_mode = g, "CUDA graph of the K timed steps (captured once, replayed)"
        except Exception as e:                           # pragma: no cover - report and fall back
            launch_mode = f"eager (graph capture failed: {str(e)[:120]})"
            barrier()
    launches = pre.launch_count() - launches0
    ledger = pre.comm_ledger(reset=True)                 # payload of the captured (= timed) steps
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier()
        ev0.record(stream)
        if graph is not None:
            graph.replay()
        else:
            for i in range(args.steps):
                step(args.warmup + i)
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    if graph is None:
        launches = pre.launch_count() - launches0
        ledger = pre.comm_ledger(reset=True)
    del graph
    # per-kernel times: the same K steps again through the profiling context
    barrier()
    pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pe0.record(stream)
    for i in range(args.steps):
        step(args.warmup + i, pre_prof)
    pe1.record(stream)
    barrier()
    ms_prof = pe0.elapsed_time(pe1)
    prof = pre_prof.profile(reset=True)
    ms_max = D.max_over_ranks(ms, dev)
    bits_frame = cfg.bits_per_frame
    bits_step = bits_frame * len(modes)
    value = bits_step * args.steps / (ms_max / 1e3) / 1e9

    # ---------------- per-mode single-frame latency (p50 / p99 over --latency-frames frames each)
    lat = {}
    for m in modes:
        fn = pre.precode_pd if m == "pd" else pre.precode_fd
        xs = []
        for i in range(args.latency_frames):
            j = i % R
            barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn(Hs[j], Ss[j], N0, 1.0, out=Xs[j])
            b.record(stream)
            torch.cuda.synchronize(dev)
            xs.append(D.max_over_ranks(a.elapsed_time(b), dev))
        xs.sort()
        p50 = xs[len(xs) // 2]
        lat[m] = {"latency_ms_p50": p50, "latency_ms_p99": xs[min(len(xs) - 1, int(0.99 * len(xs)))],
                  "frames": len(xs), "gbps_at_p50": bits_frame / (p50 / 1e3) / 1e9}
        # steady state of this precoder alone: back-to-back frames (rotating resident inputs) captured
        # into one CUDA graph and replayed, so consecutive frames overlap under PDL as in the step
        if len(modes) > 1 and not args.eager:
            nf = max(20, min(args.steps, 200))
            try:
                g1 = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g1):
                    for i in range(nf):
                        j = i % R
                        fn(Hs[j], Ss[j], N0, 1.0, out=Xs[j])
                g1.replay()
                barrier()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                g1.replay()
                b.record(stream)
                barrier()
                sms = D.max_over_ranks(a.elapsed_time(b), dev) / nf
                lat[m].update({"steady_ms_per_frame": sms, "steady_frames": nf,
                               "gbps_steady": bits_frame / (sms / 1e3) / 1e9})
                del g1
            except Exception as e:                       # pragma: no cover - report, keep the line
                lat[m]["steady_error"] = str(e)[:120]
    pre.profile(reset=True)

    # ---------------- prepare / apply: W = A^{-1}/beta cached once per
    # channel, then one OFDM symbol per dp_apply call (whitening + precode [+ s broadcast]); p50 / p99
    apply = None
    if not args.no_apply and not args.fp64 and not sizes:
        apply = {}
        s1 = [S[:, :1].contiguous() for S in Ss]
        x1 = torch.empty((cfg.n_sc, 1, Bl), dtype=torch.complex64, device=dev)
        for m in modes:
            prep = pre.prepare_pd if m == "pd" else pre.prepare_fd
            tp, ta = [], []
            for i in range(max(20, args.latency_frames // 10)):
                j = i % R
                barrier()
                a, b, c_ = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                a.record(stream)
                prep(Hs[j], N0, 1.0)
                b.record(stream)
                for q in range(10):
                    pre.apply(Hs[j], s1[(j + q) % R], out=x1)
                c_.record(stream)
                torch.cuda.synchronize(dev)
                tp.append(D.max_over_ranks(a.elapsed_time(b), dev))
                ta.append(D.max_over_ranks(b.elapsed_time(c_) / 10, dev))
            tp.sort()
            ta.sort()
            apply[m] = {"prepare_ms_p50": tp[len(tp) // 2], "apply_1symbol_ms_p50": ta[len(ta) // 2],
                        "apply_1symbol_ms_p99": ta[min(len(ta) - 1, int(0.99 * len(ta)))], "samples": len(ta),
                        "note": "apply = one symbol for all subcarriers (z = W s, x = H^H z), averaged over 10 "
                                "back-to-back calls per sample; device-timed, max over ranks"}
        pre.profile(reset=True)

    # ---------------- e2e through the C-ABI with pinned HOST buffers (H2D + compute + D2H per call)
    e2e = None
    if not args.no_e2e:
        Hh = Hs[0].cpu().pin_memory()
        Sh = Ss[0].cpu().pin_memory()
        Xh = torch.empty((cfg.n_sc, cfg.K, Bl), dtype=torch.complex64).pin_memory()
        ne = max(3, min(args.steps, 20))

        def e2e_ms(p):
            for m in modes:  # warm the staging buffers
                (p.precode_pd if m == "pd" else p.precode_fd)(Hh, Sh, N0, 1.0, out=Xh)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for i in range(ne):
                for m in modes:
                    (p.precode_pd if m == "pd" else p.precode_fd)(Hh, Sh, N0, 1.0, out=Xh)
            e1.record(stream)
            barrier()
            return D.max_over_ranks(e0.elapsed_time(e1), dev)

        s_ms = e2e_ms(pre)                       # each call returns after its D2H
        a_ms = None
        if world == 1 and not force:             # DP_FLAG_HOST_ASYNC: consecutive calls overlap
            pre_a = mk(flags | L.DP_FLAG_HOST_ASYNC)
            if sizes:
                pre_a.set_clusters(sizes, [b / cfg.B for b in sizes])
            a_ms = e2e_ms(pre_a)
            pre_a.close()
        e_ms = a_ms if a_ms is not None else s_ms
        e2e = {"value": bits_step * ne / (e_ms / 1e3) / 1e9, "unit": "Gbit/s",
               "h2d_bytes_per_step": len(modes) * (bf["H"] + bf["s"]),
               "d2h_bytes_per_step": len(modes) * bf["x"], "ms_per_step": e_ms / ne,
               "sync_calls_value": bits_step * ne / (s_ms / 1e3) / 1e9,
               "note": "pinned host H, s, x through dp_precode_* (chunked H2D / kernels / D2H inside each call)"
                       + ("; calls with DP_FLAG_HOST_ASYNC (a call's H2D overlaps the previous call's last "
                          "kernels and D2H; the timed region ends after every D2H); sync_calls_value: each "
                          "call returning after its D2H" if a_ms is not None else "")}
        pre.profile(reset=True)

    peaks = load_peaks()
    roof = roofline(cfg, world, prof, ms_prof, ms / args.steps, args.steps, peaks, sizes, args.fp64, modes)

    parity = None
    if world > 1 and not args.no_parity:
        parity = parity_check(pre, cfg, world, rank, dev, Hs, Ss, modes, N0)
    comm = pre.comm_info()

    cpu = None
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        cpu = cpu_baseline(cfg, args.cpu_seconds, modes)

    clocks = clk.summary()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Gbit/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64-accumulate, complex64 I/O" if args.fp64 else "complex64",
            "data": "synthetic",
            "config": {"workload": f"{cfg.name}: B={cfg.B} U={cfg.U} C={cfg.C} S={cfg.S} N_sc={cfg.n_sc} "
                                   f"K={cfg.K} {cfg.M}-QAM SNR={cfg.snr_db} dB tau={cfg.tau}",
                       "step": "+".join(m.upper() + "-WF frame" for m in modes),
                       "bits_per_step": bits_step, "clusters_per_gpu": cfg.C // world,
                       **({"cluster_sizes": sizes} if sizes else {}),
                       "parallelism": f"cluster-sharded x{world}" + ("" if world == 1 else f", PD {args.pd_topology}"),
                       "l2": f"{R} rotating resident input sets of {per_set / 2**20:.1f} MiB (> 2x L2)",
                       "path": ("fp64 accumulation (DP_FLAG_FP64)" if args.fp64 else
                                "unfused (a)(b)(c)" if args.unfused else "fused single pass"),
                       "launch": launch_mode},
            "modes": lat,
            "apply": apply,
            "roofline": roof,
            "comm": {"bytes_per_step": 4 * sum(ledger.values()) / args.steps,
                     "by_kind_bytes_per_step": {k: 4 * v / args.steps for k, v in ledger.items()},
                     "nccl_nranks": comm["nranks"], "nccl_version": comm["nccl_version"],
                     "note": "payload this rank handed to NCCL per step (dp_comm_ledger), rank 0"},
            "parity": parity,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clocks,
            "gpu_launches": launches,
            "gpu_name": torch.cuda.get_device_name(dev),
        }
        print(json.dumps(line), flush=True)
    pre.close()
    pre_prof.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
