"""Worker of tests/test_multigpu.py, one process per GPU under torchrun (NCCL).

Every rank precodes its cluster shard of a seeded frame through libdp (its own NCCL
communicator, bootstrapped over torch.distributed); the shards are gathered on rank 0, which
checks:
  * PD in all three exchange topologies (allreduce, reduce + z broadcast P:280-281/P:296,
    reduce-scatter + all-gather) against the fp64 oracle (stacked x, relative L2 <= 1e-4);
  * FD bit-identical to the 1-GPU run (same kernels on the same clusters; only s and the
    per-subcarrier scalars cross ranks) and within 1e-4 of the oracle;
  * the receive scale and power scalars after the scalar allreduce;
  * the library's communicator has `world` ranks (dp_comm_info).
Prints one JSON line on rank 0; exits non-zero on any failure.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import numpy as np
    import torch
    import torch.distributed as dist

    from helpers import REL_TOL, rel_l2
    from paper_1804_10987_b200 import CONFIGS, synth
    from paper_1804_10987_b200 import dist as D
    from paper_1804_10987_b200.api import Precoder

    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    cfgid = int(os.environ.get("MGPU_CFG", "4"))
    n_sc = int(os.environ.get("MGPU_NSC", "48"))
    cfg = CONFIGS[cfgid]
    f = synth.make_frame(cfg.cfg_id, n_sc, cfg.B, cfg.U, cfg.K, cfg.M, frame=11)
    N0 = synth.n0_from_snr_db(cfg.snr_db)
    sh = D.cluster_shard(cfg.B, cfg.C, world, rank)
    Hl = torch.from_numpy(np.ascontiguousarray(f.H[:, sh.b0:sh.b1])).to(dev)
    s = torch.from_numpy(f.s).to(dev)
    res = {"world": world, "cfg": cfg.name, "n_sc": n_sc}
    ok = True

    def gather(x):
        return D.gather_antennas(x).cpu().numpy()

    for topo in ("allreduce", "reduce_bcast", "scatter_gather") + (("nvlink",) if cfg.U == 32 else ()):
        with Precoder(n_sc, cfg.B, cfg.U, cfg.K, cfg.C, rank=rank, world=world, device=local, tau=cfg.tau,
                      pd_topology=topo, s_on_all_ranks=False, nccl_id=D.bootstrap_nccl_id()) as pre:
            x = pre.precode_pd(Hl, s if rank == 0 else None, N0, 1.0)
            rx = pre.read_scalars("rx").cpu().numpy()
            pw = pre.read_scalars("power").cpu().numpy()
            nranks = pre.comm_info()["nranks"]
            assert pre.status() == 0
        xs = gather(x)
        if rank == 0:
            import oracle
            xr, br = oracle.pd(f.H, f.s, cfg.C, N0)
            e = rel_l2(xs, xr)
            eb = float(np.max(np.abs(rx / br - 1)))
            ep = float(np.max(np.abs(pw / np.sum(np.abs(xr) ** 2, axis=(1, 2)) - 1)))
            res[f"pd_{topo}"] = {"rel_l2": e, "rx": eb, "power": ep, "nranks": nranks}
            ok = ok and e <= REL_TOL and eb <= REL_TOL and ep <= 1e-4 and nranks == world
    with Precoder(n_sc, cfg.B, cfg.U, cfg.K, cfg.C, rank=rank, world=world, device=local, tau=cfg.tau,
                  s_on_all_ranks=False, nccl_id=D.bootstrap_nccl_id()) as pre:
        x = pre.precode_fd(Hl, s if rank == 0 else None, N0, 1.0)
        rx = pre.read_scalars("rx").cpu().numpy()
        beta = pre.read_scalars("beta")
        assert pre.status() == 0
    xs = gather(x)
    bl = [torch.empty_like(beta) for _ in range(world)]
    dist.all_gather(bl, beta)
    if rank == 0:
        import oracle
        bs = torch.cat(bl, dim=1).cpu().numpy()
        with Precoder(n_sc, cfg.B, cfg.U, cfg.K, cfg.C, device=local, tau=cfg.tau) as one:
            x1 = one.precode_fd(torch.from_numpy(f.H).to(dev), s, N0, 1.0).cpu().numpy()
            b1 = one.read_scalars("beta").cpu().numpy()
            rx1 = one.read_scalars("rx").cpu().numpy()
        xr, br = oracle.fd(f.H, f.s, cfg.C, N0, tau=cfg.tau)
        bit = bool(np.array_equal(xs.view(np.uint64), x1.view(np.uint64)) and
                   np.array_equal(bs.view(np.uint32), b1.view(np.uint32)))
        e = rel_l2(xs, xr)
        erx = float(np.max(np.abs(rx / rx1 - 1)))
        res["fd"] = {"bit_identical_to_1gpu": bit, "rel_l2": e, "rx_vs_1gpu": erx}
        ok = ok and bit and e <= REL_TOL and erx <= 1e-6
        res["ok"] = ok
        print(json.dumps(res), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0 and not ok:
        sys.exit(1)


if __name__ == "__main__":
    main()
