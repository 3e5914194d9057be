"""Multi-GPU parity of libdp on 2, 4 and 8 GPUs (-m gpu; skipped when the box has fewer GPUs).

Runs tests/mgpu_worker.py under torchrun (one process per GPU, NCCL over NVLink): PD in its three
exchange topologies against the fp64 oracle, FD bit-identical to the 1-GPU run.
This is the check the first SCALE run relies on: it is the first time rank > 0 code paths
(s landing buffer, subcarrier-block offsets, Reduce/Bcast to a real root) execute.
"""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("cfgid", [3, 4])
def test_multigpu_parity(world, cfgid):
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs (have {torch.cuda.device_count() if torch.cuda.is_available() else 0})")
    env = dict(os.environ, MGPU_CFG=str(cfgid), MGPU_NSC="48", NCCL_DEBUG="WARN")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tests", "mgpu_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0 and lines, (r.returncode, r.stdout[-2000:], r.stderr[-4000:])
    res = json.loads(lines[-1])
    assert res["ok"], res
