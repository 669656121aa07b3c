"""The distributed stage 1 and the sharded stage 2 on REAL ranks, one process per
GPU over NCCL / NVLink (torch.distributed.run): Pi, Lambda_2, D and L of the
world-2/4/8 factorization bit-identical to the one-GPU path, S22 identical on every
rank (tools/dist_check.py).  Skipped when fewer GPUs are present (this run's
boxes have one; the same code path is covered on one GPU by the G-rank emulation
of tests/test_gpu_dist.py)."""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("name", ["P2048", "C1"])
def test_real_ranks_bitwise(world, name):
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tools", "dist_check.py"), name]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert '"S22_identical_on_ranks": true' in r.stdout
