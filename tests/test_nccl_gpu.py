"""The collectives the N > 1 step issues, run through NCCL itself (a one-process NCCL group
on cuda:0, in a subprocess so no process group leaks into the other tests).  NCCL rejects a
coalesced allreduce of mixed dtypes; the step's aggregates (int64 counters, fp64 loss) must
go per dtype."""
import os
import socket
import subprocess
import sys

import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_step_collectives_through_nccl():
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "nccl_probe.py")], env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "NCCL per-dtype coalesced allreduce OK" in r.stdout
