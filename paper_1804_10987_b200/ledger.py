"""Exchange ledger: what crosses between clusters / GPUs per frame.

Two views, both exact integers:

* ``paper_ledger`` — the paper's feedforward architectures (Fig. 1, Sec. IV-C) with one
  cluster per node: PD sums the C partial Grams over a balanced binary adder tree (C - 1 edges,
  depth ceil(log2 C), U x U complex scalars per subcarrier per edge: "scaling with
  N_sc x U x U") and broadcasts z from the master to the C - 1 other clusters
  (N_sc x K x U per link); FD only broadcasts s. Closed forms
  (C-1) N_sc U^2 and (C-1) N_sc K U (SPEC "Ledger exactness").
* ``library_payload`` — what libdp hands to NCCL per rank and frame (fp32 elements, the
  counters of ``dp_comm_ledger``): the Gram is exchanged as its packed Hermitian upper
  triangle, U (U + 1) / 2 complex per subcarrier (reading: the lower half is redundant), and
  the per-subcarrier scalars [n_sc][2] (receive scale, power) are one extra allreduce.

``ring_link_floats`` converts a per-rank allreduce / broadcast payload into the per-link
volume of a ring (NCCL's bandwidth-optimal schedule), and ``alpha_beta_us`` is the affine
latency model alpha + bytes / beta the SPEC describes; its parameters are inputs —
this repo runs on one GPU, so no fit is claimed.
"""
from __future__ import annotations

import math


def paper_ledger(C: int, n_sc: int, K: int, U: int, mode: str) -> dict:
    """Complex scalars moved per frame over the cluster fabric (all links together)."""
    if C < 1:
        raise ValueError("C >= 1")
    gram = (C - 1) * n_sc * U * U if mode == "pd" else 0
    if mode == "pd":
        bcast = (C - 1) * n_sc * K * U          # z from the master
    elif mode == "fd":
        bcast = (C - 1) * n_sc * K * U          # s to every cluster
    else:
        raise ValueError(mode)
    return {"gram": gram, "bcast": bcast, "tree_edges": C - 1 if mode == "pd" else 0,
            "tree_depth": math.ceil(math.log2(C)) if (mode == "pd" and C > 1) else 0,
            "total": gram + bcast}


def library_payload(world: int, n_sc: int, K: int, U: int, mode: str, topology: str = "allreduce",
                    s_on_all_ranks: bool = False, comm: bool | None = None) -> dict:
    """fp32 elements this rank passes to each collective kind for one frame (dp_comm_ledger).
    comm: whether collectives run at all (world > 1, or DP_FLAG_FORCE_COMM at world 1)."""
    comm = (world > 1) if comm is None else comm
    out = {"gram": 0, "s_bcast": 0, "z_bcast": 0, "scalars": 0}
    if not comm:
        return out
    s_floats = n_sc * K * U * 2
    out["scalars"] = 2 * n_sc
    if mode == "fd":
        out["s_bcast"] = 0 if s_on_all_ranks else s_floats
        return out
    out["gram"] = n_sc * U * (U + 1) // 2 * 2
    if topology == "reduce_bcast":
        out["z_bcast"] = s_floats + n_sc        # z and beta from rank 0
    elif topology in ("scatter_gather", "nvlink"):   # nvlink: the same payload, moved by the solve kernel
        out["s_bcast"] = 0 if s_on_all_ranks else s_floats
        out["z_bcast"] = (n_sc // world) * K * U * 2 + n_sc // world   # this rank's z / beta block
    else:
        out["s_bcast"] = 0 if s_on_all_ranks else s_floats
    return out


def ring_link_floats(payload: int, world: int, kind: str) -> float:
    """Per-link volume of a ring schedule over `world` ranks for a per-rank payload."""
    if world <= 1:
        return 0.0
    if kind == "allreduce":
        return 2.0 * (world - 1) / world * payload
    if kind in ("reduce", "broadcast"):
        return float(payload) * (world - 1) / world if kind == "reduce" else float(payload)
    raise ValueError(kind)


def alpha_beta_us(nbytes: float, alpha_us: float, beta_gbs: float) -> float:
    """Affine latency model alpha + bytes / beta; parameters are inputs."""
    return alpha_us + nbytes / (beta_gbs * 1e3)
