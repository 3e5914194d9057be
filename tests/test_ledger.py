"""Exchange ledger: closed forms pinned to the SPEC's worked numbers, and
the library's own counters (dp_comm_ledger) against them on a 1-rank communicator."""
from __future__ import annotations

import numpy as np
import pytest

from paper_1804_10987_b200 import ledger


def test_paper_ledger_worked_numbers():
    # SPEC gram_reduce_tree: C=8, U=16, N_sc=1200 -> (C-1) N_sc U^2 = 2,150,400 complex scalars
    pd = ledger.paper_ledger(8, 1200, 7, 16, "pd")
    assert pd["gram"] == 2_150_400 and pd["tree_edges"] == 7 and pd["tree_depth"] == 3
    # SPEC run_pd_wf: broadcast volume per link N_sc K U = 134,400 (U=16, N_sc=1200, K=7)
    assert pd["bcast"] // 7 == 134_400
    # C = 4 binary tree: 3 edges, depth 2 (SPEC example); C = 1: no messages
    assert ledger.paper_ledger(4, 1, 1, 2, "pd")["tree_edges"] == 3
    assert ledger.paper_ledger(4, 1, 1, 2, "pd")["tree_depth"] == 2
    assert ledger.paper_ledger(1, 1200, 14, 16, "pd")["total"] == 0
    # FD omits the whole Gram term: less traffic than PD for every C >= 2
    for C in (2, 4, 8):
        assert ledger.paper_ledger(C, 1200, 14, 32, "fd")["total"] < ledger.paper_ledger(C, 1200, 14, 32, "pd")["total"]


def test_library_payload_forms():
    p = ledger.library_payload(8, 1200, 14, 32, "pd")
    assert p["gram"] == 1200 * 528 * 2 and p["s_bcast"] == 1200 * 14 * 32 * 2 and p["scalars"] == 2400
    assert ledger.library_payload(8, 1200, 14, 32, "pd", topology="reduce_bcast")["z_bcast"] == 1200 * 14 * 32 * 2 + 1200
    assert ledger.library_payload(8, 1200, 14, 32, "fd", s_on_all_ranks=True) == \
        {"gram": 0, "s_bcast": 0, "z_bcast": 0, "scalars": 2400}
    assert ledger.library_payload(1, 1200, 14, 32, "pd") == {"gram": 0, "s_bcast": 0, "z_bcast": 0, "scalars": 0}
    # the packed Hermitian Gram moves (U+1)/(2U) of the paper's U^2 per subcarrier
    assert ledger.library_payload(2, 10, 1, 16, "pd")["gram"] / 2 / (10 * 16 * 16) == pytest.approx(17 / 32)
    assert ledger.ring_link_floats(100, 4, "allreduce") == pytest.approx(150.0)
    assert ledger.alpha_beta_us(1e6, 5.0, 100.0) == pytest.approx(15.0)


@pytest.mark.gpu
@pytest.mark.parametrize("mode,topology", [("pd", "allreduce"), ("pd", "reduce_bcast"), ("pd", "scatter_gather"),
                                           ("pd", "nvlink"), ("fd", "allreduce")])
def test_library_counters_match(mode, topology):
    import torch

    from paper_1804_10987_b200 import CONFIGS, synth
    from paper_1804_10987_b200 import _lib as L
    from paper_1804_10987_b200 import dist as D
    from paper_1804_10987_b200.api import Precoder
    cfg = CONFIGS[4] if topology == "nvlink" else CONFIGS[3]   # the fused-exchange kernel is U = 32
    n_sc = 11
    f = synth.make_frame(cfg.cfg_id, n_sc, cfg.B, cfg.U, cfg.K, cfg.M)
    uid = L.dp_get_unique_id()
    with Precoder(n_sc, cfg.B, cfg.U, cfg.K, cfg.C, flags=L.DP_FLAG_FORCE_COMM, nccl_id=uid,
                  pd_topology=topology, s_on_all_ranks=False) as pre:
        H = torch.from_numpy(f.H).cuda()
        s = torch.from_numpy(f.s).cuda()
        (pre.precode_pd if mode == "pd" else pre.precode_fd)(H, s, 0.1, 1.0)
        torch.cuda.synchronize()
        got = pre.comm_ledger(reset=True)
    want = ledger.library_payload(1, n_sc, cfg.K, cfg.U, mode, topology=topology, s_on_all_ranks=False, comm=True)
    assert got == want, (got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("force_comm", [False, True])
def test_prepare_pd_ledger_world1(force_comm):
    """dp_prepare_pd counts the Gram exchange only when a collective is issued: nothing at
    world 1 without a communicator, the packed Gram payload with a (forced) 1-rank one."""
    import torch

    from paper_1804_10987_b200 import CONFIGS, synth
    from paper_1804_10987_b200 import _lib as L
    from paper_1804_10987_b200.api import Precoder
    cfg = CONFIGS[3]
    n_sc = 7
    f = synth.make_frame(cfg.cfg_id, n_sc, cfg.B, cfg.U, cfg.K, cfg.M)
    kw = dict(flags=L.DP_FLAG_FORCE_COMM, nccl_id=L.dp_get_unique_id()) if force_comm else {}
    with Precoder(n_sc, cfg.B, cfg.U, cfg.K, cfg.C, **kw) as pre:
        pre.prepare_pd(torch.from_numpy(f.H).cuda(), 0.1, 1.0)
        torch.cuda.synchronize()
        got = pre.comm_ledger(reset=True)
    want = n_sc * cfg.U * (cfg.U + 1) // 2 * 2 if force_comm else 0
    assert got == {"gram": want, "s_bcast": 0, "z_bcast": 0, "scalars": 0}, got
