"""Transport all-to-all: byte-exact delivery of variable, skewed and empty
messages (tests/a2a_worker.py) -- one rank per GPU over NVLink on a 2+ GPU
box, two ranks sharing cuda:0 on a 1-GPU box."""
import os
import subprocess
import sys

import pytest

from test_ring_gpu import ranks_and_env

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_alltoall_byte_exact():
    n, env = ranks_and_env()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29534", os.path.join(HERE, "a2a_worker.py"), "4"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "A2A_OK" in r.stdout
