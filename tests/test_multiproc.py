"""World-size-2 gloo tests (CPU) of the multi-GPU host logic and of the exchange
pattern the library implements over NCCL:

* cluster sharding and antenna gathers;
* NCCL-id bootstrap over torch.distributed;
* max-over-ranks timing;
* the distributed decomposition itself, evaluated with the oracle's steps:
  PD  = local Gram -> allreduce (or reduce + z broadcast, or reduce-scatter over subcarrier
        blocks + z all-gather) -> solve -> local precode,
  FD  = s broadcast -> local clusters -> allreduce of [sum_c 1/beta_c, power],
  each equal to the single-process oracle.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn_name, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = globals()[fn_name](rank, world)
        q.put((rank, "ok", out))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback

        q.put((rank, "err", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def run_world(fn_name, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for r, status, out in res:
        assert status == "ok", out
    return {r: out for r, _, out in res}


# ---------------------------------------------------------------- workers
def w_shard_and_gather(rank, world):
    from paper_1804_10987_b200 import dist as D

    sh = D.cluster_shard(256, 8, world, rank)
    assert (sh.b1 - sh.b0) == 256 // world and (sh.c1 - sh.c0) == 8 // world
    H = torch.arange(3 * 256 * 4, dtype=torch.float32).reshape(3, 256, 4)
    Hl = D.local_channel(H, sh)
    assert torch.equal(Hl, H[:, rank * 128:(rank + 1) * 128])
    x_full = torch.arange(3 * 2 * 256, dtype=torch.float32).reshape(3, 2, 256)
    x_local = x_full[:, :, sh.b0:sh.b1]
    assert torch.equal(D.gather_antennas(x_local), x_full)
    assert D.max_over_ranks(10.0 + rank) == 10.0 + world - 1
    return True


def w_bootstrap(rank, world):
    from paper_1804_10987_b200 import dist as D

    uid = D.bootstrap_nccl_id(make_id=lambda: bytes(range(128)))
    assert uid == bytes(range(128))
    return uid[:4]


def _frame():
    from paper_1804_10987_b200 import synth

    return synth.make_frame(cfg_id=9, n_sc=6, B=32, U=4, K=3, M=16)


def w_pd_decomposition(rank, world):
    """PD over ranks with the library's exchange pattern, evaluated with oracle steps."""
    import oracle
    from paper_1804_10987_b200 import dist as D

    f = _frame()
    C, N0, rho2 = 4, 0.2, 1.0
    U = f.H.shape[2]
    sh = D.cluster_shard(32, C, world, rank)
    Hl = f.H[:, sh.b0:sh.b1].astype(np.complex128)
    outs = {}
    for topo in ("allreduce", "reduce_bcast", "scatter_gather"):
        # (a) local Gram: this rank's clusters (first adder-tree levels)
        G = torch.from_numpy(np.stack([oracle.gram(Hl[w]) for w in range(Hl.shape[0])]))
        n_sc = Hl.shape[0]
        nb = n_sc // world
        mine = range(n_sc)                           # subcarriers this rank whitens
        if topo == "allreduce":
            dist.all_reduce(G)                       # every rank holds G
        elif topo == "reduce_bcast":
            dist.reduce(G, dst=0)                    # master holds G
            mine = range(n_sc) if rank == 0 else range(0)
        else:
            # reduce-scatter over subcarrier blocks (gloo: all-reduce, keep this rank's block)
            dist.all_reduce(G)
            mine = range(rank * nb, (rank + 1) * nb)
        z = torch.zeros((n_sc, 3, U), dtype=torch.complex128)
        kappa = U * N0 / rho2
        for w in mine:
            Ai = oracle.hpd_inverse(G[w].numpy() + kappa * np.eye(U))
            beta = oracle.beta_lemma1(Ai, kappa, 1.0, rho2)
            z[w] = torch.from_numpy((Ai @ f.s[w].T.astype(np.complex128)).T / beta)
        if topo == "reduce_bcast":
            dist.broadcast(z, src=0)                 # master broadcasts z
        elif topo == "scatter_gather":
            blocks = [torch.zeros((nb, 3, U), dtype=torch.complex128) for _ in range(world)]
            dist.all_gather(blocks, z[rank * nb:(rank + 1) * nb].contiguous())
            z = torch.cat(blocks, dim=0)
        # (c) local precode x_c = H_c^H z
        x_local = np.einsum("wbu,wku->wkb", np.conj(Hl), z.numpy())
        x = D.gather_antennas(torch.from_numpy(x_local)).numpy()
        xr, _ = oracle.pd(f.H, f.s, C, N0, rho2)
        outs[topo] = float(np.linalg.norm(x - xr) / np.linalg.norm(xr))
    return outs


def w_fd_decomposition(rank, world):
    """FD over ranks: s broadcast, local clusters, scalar allreduce [sum 1/beta_c, power]."""
    import oracle
    from paper_1804_10987_b200 import dist as D

    f = _frame()
    C, N0, rho2, tau = 4, 0.2, 1.0, 0.125
    sh = D.cluster_shard(32, C, world, rank)
    s = torch.from_numpy(f.s.astype(np.complex128)) if rank == 0 else torch.zeros(f.s.shape, dtype=torch.complex128)
    dist.broadcast(s, src=0)                        # "s is the only signal that must be broadcast"
    Hl = f.H[:, sh.b0:sh.b1]
    # this rank's clusters with the global per-cluster budget rho_c^2 = rho^2/C and
    # kappa_c = tau U N0 / rho_c^2 (Eq. 9): fd(H_local, C_local, N0, rho^2 C_local/C) has exactly those
    Cl = C // world
    xl, bl = oracle.fd(Hl, s.numpy(), Cl, N0, rho2 * Cl / C, tau=tau)
    sc = torch.from_numpy(np.stack([np.sum(1.0 / bl, axis=1), np.sum(np.abs(xl) ** 2, axis=(1, 2))], axis=1))
    dist.all_reduce(sc)
    x = D.gather_antennas(torch.from_numpy(xl)).numpy()
    xr, br = oracle.fd(f.H, f.s, C, N0, rho2, tau=tau)
    rx_ref = oracle.rx_scale_fd(br)
    return (float(np.linalg.norm(x - xr) / np.linalg.norm(xr)),
            float(np.max(np.abs(1.0 / sc[:, 0].numpy() / rx_ref - 1))),
            float(np.max(np.abs(sc[:, 1].numpy() / np.sum(np.abs(xr) ** 2, axis=(1, 2)) - 1))))


# ---------------------------------------------------------------- tests
def test_shard_and_gather_world2():
    assert all(run_world("w_shard_and_gather").values())


def test_nccl_id_bootstrap_world2():
    out = run_world("w_bootstrap")
    assert out[0] == out[1] == bytes(range(4))


def test_pd_exchange_pattern_world2():
    for r, errs in run_world("w_pd_decomposition").items():
        assert errs["allreduce"] < 1e-12 and errs["reduce_bcast"] < 1e-12 and errs["scatter_gather"] < 1e-12, errs


def test_fd_exchange_pattern_world2():
    for r, (ex, erx, epw) in run_world("w_fd_decomposition").items():
        assert ex < 1e-12 and erx < 1e-12 and epw < 1e-12


def test_cluster_shard_validation():
    from paper_1804_10987_b200 import dist as D

    with pytest.raises(ValueError):
        D.cluster_shard(256, 8, 3, 0)
    with pytest.raises(ValueError):
        D.cluster_shard(250, 8, 1, 0)
    sh = D.cluster_shard(256, 8, 8, 7)
    assert (sh.b0, sh.b1, sh.c0, sh.c1) == (224, 256, 7, 8)


def test_bench_reference_arm_torchrun_world2():
    """bench.py --impl reference under torchrun (gloo-free: rank 0 alone runs and prints)."""
    env = dict(os.environ, PYTHONPATH=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "2", "--warmup", "1", "--config", "2",
           "--cpu-seconds", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    import json

    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
