"""bench.py — precoded Gbit/s and frame latency (device-timed) of PD-WF and FD-WF.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, NCCL)

Workload (BASELINE.json configs[3]): B=256 antennas, U=32 UEs,
C=8 clusters (S=32), N_sc=1200 subcarriers, K=14 OFDM symbols, 64-QAM, SNR
10 dB, tau=0.125.  A STEP is one pass of the whole hot path over one frame:
one PD-WF frame followed by one FD-WF frame, so
bits/step = 2 * N_sc * K * U * log2(M) for the whole job.  Scaling is STRONG
(the frame is fixed; clusters are sharded over the N GPUs, C/N per GPU).

Timing: W warm-up steps, then K steps bracketed by barrier + synchronize,
CUDA events on the launching stream, max over ranks.  Inputs rotate over R
resident input sets whose total size exceeds 2x L2 (126 MB), so every step
reads H from HBM.  Rank 0 prints ONE JSON line.
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="both", choices=["both", "pd", "fd"])
    ap.add_argument("--unfused", action="store_true", help="three-kernel path (a)(b)(c)")
    ap.add_argument("--pd-topology", default="scatter_gather", choices=["allreduce", "reduce_bcast", "scatter_gather"],
                    help="PD exchange for N > 1 (DESIGN.md §6); scatter_gather splits the solve over the GPUs")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target oracle CPU time for cpu_baseline")
    ap.add_argument("--profile-run", action="store_true", help="short run for ncu (no JSON extras)")
    ap.add_argument("--cluster-sizes", default="", help="comma list of C unequal cluster sizes B_c (dp_set_clusters, "
                    "P:157); FD only, power shares B_c / B")
    ap.add_argument("--eager", action="store_true", help="launch the timed steps eagerly (default: replay a CUDA "
                    "graph captured from the same K steps; host launch overhead out of the timed region)")
    return ap.parse_args()


# ---------------------------------------------------------------- algorithmic work
def flops_problem(U: int, nb: int, K: int) -> dict:
    """Algorithmic real flops of one WF problem (one subcarrier x one cluster for FD, one
    subcarrier over nb antennas for PD); complex MAC = 8 flops.
    Gram: Hermitian half U(U+1)/2 entries x nb ; Cholesky U^3/6 ; L^-1 U^3/6 ; A^-1 = W0^H W0 U^3/6 ;
    whiten K U^2 ; precode K nb U."""
    cmac = {
        "gram": nb * U * (U + 1) / 2,
        "solve": U ** 3 / 2,
        "whiten": K * U * U,
        "precode": K * nb * U,
    }
    return {k: 8.0 * v for k, v in cmac.items()}


def bytes_frame(cfg, Bl: int) -> dict:
    """Algorithmic HBM bytes per frame per GPU: H read once, s read once, x written once."""
    return {"H": cfg.n_sc * Bl * cfg.U * 8, "s": cfg.n_sc * cfg.K * cfg.U * 8, "x": cfg.n_sc * cfg.K * Bl * 8}


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
def _oracle_step(cfg, f, N0):
    import oracle

    oracle.pd(f.H, f.s, cfg.C, N0)
    oracle.fd(f.H, f.s, cfg.C, N0, tau=cfg.tau)


def cpu_baseline(cfg, target_s: float, chunk: int = 96):
    """The fp64 oracle (oracle/, as it stands) on a bounded sample of the same workload:
    a chunk of `chunk` subcarriers of one frame (PD + FD), repeated until ~target_s of
    CPU work, on all host cores (OpenMP over subcarriers)."""
    import oracle
    from paper_1804_10987_b200 import synth

    N0 = synth.n0_from_snr_db(cfg.snr_db)
    f = synth.make_frame(cfg.cfg_id, chunk, cfg.B, cfg.U, cfg.K, cfg.M, frame=77)
    _oracle_step(cfg, f, N0)                      # warm (page-in, thread pool)
    reps, t0 = 0, time.perf_counter()
    while True:
        _oracle_step(cfg, f, N0)
        reps += 1
        el = time.perf_counter() - t0
        if el >= target_s or reps >= 10000:
            break
    bits = 2 * reps * chunk * cfg.K * cfg.U * (cfg.M.bit_length() - 1)
    return {"value": bits / el / 1e9, "unit": "Gbit/s", "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"{reps} x {chunk} subcarriers of {cfg.name} (PD + FD frames, fp64 C oracle, "
                      f"OpenMP over subcarriers), {el:.1f} s"}


# ---------------------------------------------------------------- reference arm
def run_reference(args, cfg, rank, world):
    """--impl reference: the oracle as it stands on the host cores (rank 0 only); each step
    is a bounded sample of the workload (a chunk of subcarriers, PD + FD)."""
    if rank != 0:
        return
    import oracle
    from paper_1804_10987_b200 import synth

    N0 = synth.n0_from_snr_db(cfg.snr_db)
    chunk = 48
    f = synth.make_frame(cfg.cfg_id, chunk, cfg.B, cfg.U, cfg.K, cfg.M, frame=78)
    for _ in range(args.warmup):
        _oracle_step(cfg, f, N0)
    t = time.perf_counter()
    for _ in range(args.steps):
        _oracle_step(cfg, f, N0)
    el = time.perf_counter() - t
    bits = 2 * chunk * cfg.K * cfg.U * (cfg.M.bit_length() - 1) * args.steps
    v = bits / el / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "Gbit/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "complex128",
            "data": "synthetic",
            "config": {"workload": cfg.name, "step": f"PD + FD frames on {chunk} of {cfg.n_sc} subcarriers"},
            "cpu_baseline": {"value": v, "unit": "Gbit/s", "cores": oracle.num_threads(), "kind": "oracle",
                             "sample": f"{chunk} of {cfg.n_sc} subcarriers per step, PD + FD"},
            "e2e": {"value": v, "unit": "Gbit/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- ours
def main():
    args = parse()
    from paper_1804_10987_b200 import CONFIGS
    cfg = CONFIGS[args.config]
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

    # NCCL id for the library's own communicator
    # Two contexts: `pre` times `value` with nothing between the kernels (events between
    # launches would break the programmatic-dependent-launch overlap), `pre_prof`
    # (DP_FLAG_PROFILE: CUDA events around every kernel, on the launching stream) runs the
    # same steps right after it for the per-kernel times of the roofline.
    flags = L.DP_FLAG_UNFUSED if args.unfused else 0
    pre = Precoder(cfg.n_sc, cfg.B, cfg.U, cfg.K, cfg.C, rank=rank, world=world, device=local, tau=cfg.tau,
                   pd_topology=args.pd_topology, s_on_all_ranks=(world == 1), flags=flags,
                   nccl_id=D.bootstrap_nccl_id() if world > 1 else None)
    pre_prof = Precoder(cfg.n_sc, cfg.B, cfg.U, cfg.K, cfg.C, rank=rank, world=world, device=local, tau=cfg.tau,
                        pd_topology=args.pd_topology, s_on_all_ranks=(world == 1), flags=flags | L.DP_FLAG_PROFILE,
                        nccl_id=D.bootstrap_nccl_id() if world > 1 else None)

    sizes = [int(v) for v in args.cluster_sizes.split(",")] if args.cluster_sizes else None
    if sizes:
        for p_ in (pre, pre_prof):
            p_.set_clusters(sizes, [b / cfg.B for b in sizes])

    # ---------------- resident rotating input sets (> 2x L2 in total)
    bf = bytes_frame(cfg, Bl)
    per_set = bf["H"] + bf["s"] + bf["x"]
    R = max(2, math.ceil(2 * L2_BYTES / per_set))
    gen = torch.Generator(device=dev)
    gen.manual_seed(SEED + 1000 * args.config + rank)
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
        p = p or pre
        j = i % R
        for m in modes:
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
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    bits_frame = cfg.bits_per_frame
    bits_step = bits_frame * len(modes)
    value = bits_step * args.steps / (ms_max / 1e3) / 1e9

    # ---------------- per-mode single-frame latency (p50 / p99 over 40 frames each)
    lat = {}
    for m in modes:
        fn = pre.precode_pd if m == "pd" else pre.precode_fd
        xs = []
        for i in range(40):
            j = i % R
            barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn(Hs[j], Ss[j], N0, 1.0, out=Xs[j])
            b.record(stream)
            torch.cuda.synchronize(dev)
            tt = torch.tensor([a.elapsed_time(b)], device=dev)
            if world > 1:
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            xs.append(float(tt.item()))
        xs.sort()
        p50 = xs[len(xs) // 2]
        lat[m] = {"latency_ms_p50": p50, "latency_ms_p99": xs[min(len(xs) - 1, int(0.99 * len(xs)))],
                  "gbps_at_p50": bits_frame / (p50 / 1e3) / 1e9}
    pre.profile(reset=True)

    # ---------------- e2e through the C-ABI with pinned HOST buffers (H2D + compute + D2H per call)
    e2e = None
    if not args.no_e2e:
        Hh = Hs[0].cpu().pin_memory()
        Sh = Ss[0].cpu().pin_memory()
        Xh = torch.empty((cfg.n_sc, cfg.K, Bl), dtype=torch.complex64).pin_memory()
        for m in modes:  # warm the staging buffers
            (pre.precode_pd if m == "pd" else pre.precode_fd)(Hh, Sh, N0, 1.0, out=Xh)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ne = max(3, min(args.steps, 20))
        e0.record(stream)
        for i in range(ne):
            for m in modes:
                (pre.precode_pd if m == "pd" else pre.precode_fd)(Hh, Sh, N0, 1.0, out=Xh)
        e1.record(stream)
        barrier()
        et = torch.tensor([e0.elapsed_time(e1)], device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e_ms = float(et.item())
        e2e = {"value": bits_step * ne / (e_ms / 1e3) / 1e9, "unit": "Gbit/s",
               "h2d_bytes_per_step": len(modes) * (bf["H"] + bf["s"]),
               "d2h_bytes_per_step": len(modes) * bf["x"], "ms_per_step": e_ms / ne,
               "note": "pinned host H, s, x through dp_precode_*: H2D, kernels, D2H inside each call"}
        pre.profile(reset=True)

    # ---------------- roofline of the dominant kernel (measured in the timed region)
    dom = max(prof, key=lambda k: prof[k]["ms"])
    dom_ms = prof[dom]["ms"] / max(prof[dom]["launches"], 1)
    step_ms_local = ms / args.steps
    share = prof[dom]["ms"] / max(ms_prof, 1e-9)
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        pass
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    fp32_peak = 148 * 128 * 2 * sm_max * 1e6 / 1e12            # TFLOP/s, FFMA pipe
    Cl = cfg.C // world
    if dom == "fused_fd":
        # U = 32: the cluster Gram runs on the tensor cores (fd_tc.cuh), so the FP32-pipe
        # roofline counts the SIMT steps only (solve + whiten + precode); the Gram's flops are
        # reported beside it (tensor-core time at its 3xTF32 rate is ~3 us, not the bound).
        fl = flops_problem(cfg.U, cfg.S, cfg.K)
        simt = fl["solve"] + fl["whiten"] + fl["precode"] + (0.0 if cfg.U == 32 else fl["gram"])
        flops_launch = cfg.n_sc * Cl * simt
        bytes_launch = bf["H"] + bf["s"] + bf["x"]
    else:
        # PD kernels (a) gram: H -> packed G ; (b) solve: G, s -> z ; (c) precode: H, z -> x
        fl = flops_problem(cfg.U, Bl, cfg.K)
        npk = cfg.U * (cfg.U + 1) // 2 * 8
        flops_launch = cfg.n_sc * {"gram": fl["gram"], "solve": fl["solve"] + fl["whiten"],
                                   "precode": fl["precode"]}.get(dom, sum(fl.values()))
        bytes_launch = {"gram": bf["H"] + cfg.n_sc * npk,
                        "solve": cfg.n_sc * npk + bf["s"] + bf["s"],
                        "precode": bf["H"] + bf["s"] + bf["x"]}.get(dom, bf["H"])
    achieved = flops_launch / (dom_ms / 1e3) / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        traffic = tr.get(f"{cfg.name}/{dom}/n{world}")
    except Exception:
        pass
    roof = {"bound": "alu", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
            "frac": achieved / fp32_peak, "traffic": traffic, "kernel": dom,
            "kernel_ms_avg": dom_ms, "kernel_share_of_step": share,
            "kernel_timing": "CUDA events around each launch on its stream, in a second pass of the same "
                             f"{args.steps} steps (profiled step {ms_prof / args.steps:.4f} ms vs {ms / args.steps:.4f} ms "
                             "unprofiled: events between kernels break the PDL overlap)",
            "algorithmic_flops_per_launch": flops_launch, "algorithmic_bytes_per_launch": bytes_launch,
            "hbm_achieved_gbs": bytes_launch / (dom_ms / 1e3) / 1e9,
            "hbm_peak_gbs": peaks.get("hbm_gbs", 6544.0),
            "peak_note": f"FP32 FFMA pipe: 148 SMs x 128 lanes x 2 flop x {sm_max:.0f} MHz (sm_max_mhz of MEASURED_PEAKS.json); achieved counts the SIMT steps (solve + whiten + precode), the U=32 cluster Gram runs on the tensor cores",
            "kernels": {k: {"ms_avg": v["ms"] / max(v["launches"], 1), "launches": v["launches"]}
                        for k, v in prof.items() if v["launches"]}}

    # every kernel against its own bound: gram / precode move H through HBM with
    # the contraction on the tensor cores (bound "hbm"); solve and the FD kernel are FP32-pipe work
    hbm_peak = float(peaks.get("hbm_gbs", 6544.0))
    flp = flops_problem(cfg.U, Bl, cfg.K)
    flf = flops_problem(cfg.U, cfg.S, cfg.K)
    npk = cfg.U * (cfg.U + 1) // 2 * 8
    per = {}
    for k, v in prof.items():
        if not v["launches"]:
            continue
        kms = v["ms"] / v["launches"]
        if k == "gram":
            b = bf["H"] + cfg.n_sc * npk
            per[k] = {"bound": "hbm", "bytes": b, "achieved_gbs": b / (kms / 1e3) / 1e9, "frac": b / (kms / 1e3) / 1e9 / hbm_peak}
        elif k == "precode":
            b = bf["H"] + bf["s"] + bf["x"]
            per[k] = {"bound": "hbm", "bytes": b, "achieved_gbs": b / (kms / 1e3) / 1e9, "frac": b / (kms / 1e3) / 1e9 / hbm_peak}
        elif k == "solve":
            f_ = cfg.n_sc * (flp["solve"] + flp["whiten"])
            per[k] = {"bound": "alu", "flops": f_, "achieved_tflops": f_ / (kms / 1e3) / 1e12,
                      "frac": f_ / (kms / 1e3) / 1e12 / fp32_peak,
                      "note": "1 U x U problem per subcarrier: latency-bound (SURVEY §8(d))"}
        elif k == "fused_fd":
            simt = flf["solve"] + flf["whiten"] + flf["precode"] + (0.0 if cfg.U == 32 else flf["gram"])
            f_ = cfg.n_sc * Cl * simt
            per[k] = {"bound": "alu", "flops": f_, "achieved_tflops": f_ / (kms / 1e3) / 1e12,
                      "frac": f_ / (kms / 1e3) / 1e12 / fp32_peak,
                      "tensor_core_gram_flops": cfg.n_sc * Cl * flf["gram"] if cfg.U == 32 else 0.0}
        else:                                    # fd_finish_kernel (U < 32): per-subcarrier scalars
            per[k] = {"bound": "latency", "note": "tiny per-subcarrier combine"}
        per[k]["ms_avg"] = kms
    roof["per_kernel"] = per

    cpu = None
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        cpu = cpu_baseline(cfg, args.cpu_seconds)

    clocks = clk.summary()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Gbit/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "complex64", "data": "synthetic",
            "config": {"workload": f"{cfg.name}: B={cfg.B} U={cfg.U} C={cfg.C} S={cfg.S} N_sc={cfg.n_sc} "
                                   f"K={cfg.K} {cfg.M}-QAM SNR={cfg.snr_db} dB tau={cfg.tau}",
                       "step": "+".join(m.upper() + "-WF frame" for m in modes),
                       "bits_per_step": bits_step, "clusters_per_gpu": Cl,
                       **({"cluster_sizes": sizes} if sizes else {}),
                       "parallelism": f"cluster-sharded x{world}" + ("" if world == 1 else f", PD {args.pd_topology}"),
                       "l2": f"{R} rotating resident input sets of {per_set / 2**20:.1f} MiB (> 2x L2)",
                       "path": "unfused (a)(b)(c)" if args.unfused else "fused single pass",
                       "launch": launch_mode},
            "modes": lat,
            "roofline": roof,
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
