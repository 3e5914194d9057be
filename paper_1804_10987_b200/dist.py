"""Multi-GPU host logic: cluster sharding, NCCL-id bootstrap, gathers and timing.

One process per GPU (torch.distributed, launched by torchrun).  The antenna
array is split into C equal clusters; rank r of `world` owns clusters
[r*C/world, (r+1)*C/world), i.e. the contiguous antenna block
[r*B/world, (r+1)*B/world) — "each process controls a GPU"
with the cluster count decoupled from the GPU count.  Only the exchange steps
of the method cross ranks (inside libdp.so, over NCCL):
  PD: the Gram adder tree G = sum_c G_c (allreduce or the paper's
      reduce-to-master + z broadcast) and s;
  FD: s and 2*n_sc normalisation scalars.
This module holds no arithmetic of the method.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    b0: int   # first antenna of this rank
    b1: int   # one past the last antenna
    c0: int   # first cluster
    c1: int   # one past the last cluster


def cluster_shard(B: int, C: int, world: int, rank: int) -> Shard:
    if B % C:
        raise ValueError(f"B={B} not divisible by C={C} (equal clusters, P:157)")
    if C % world:
        raise ValueError(f"C={C} clusters cannot be split evenly over {world} ranks")
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    S = B // C
    cpr = C // world
    return Shard(rank, world, rank * cpr * S, (rank + 1) * cpr * S, rank * cpr, (rank + 1) * cpr)


def local_channel(H: torch.Tensor, shard: Shard) -> torch.Tensor:
    """H[n_sc][B][U] -> this rank's contiguous H_local[n_sc][B/world][U]."""
    return H[:, shard.b0:shard.b1, :].contiguous()


def bootstrap_nccl_id(make_id=None, src: int = 0, group=None) -> bytes:
    """Rank `src` creates the 128-byte ncclUniqueId (libdp's dp_get_unique_id by
    default) and every rank receives the same bytes over torch.distributed."""
    if make_id is None:
        from . import _lib

        make_id = _lib.dp_get_unique_id
    obj = [make_id() if dist.get_rank(group) == src else None]
    dist.broadcast_object_list(obj, src=src, group=group)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise RuntimeError("bad NCCL unique id")
    return bytes(uid)


def gather_antennas(x_local: torch.Tensor, group=None) -> torch.Tensor:
    """Stack the ranks' x_local[n_sc][K][B/world] along the antenna axis -> x[n_sc][K][B]."""
    world = dist.get_world_size(group)
    parts = [torch.empty_like(x_local) for _ in range(world)]
    dist.all_gather(parts, x_local.contiguous(), group=group)
    return torch.cat(parts, dim=-1)


def max_over_ranks(v: float, device=None, group=None) -> float:
    """Device-timed numbers are reported as the max over ranks."""
    t = torch.tensor([float(v)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
