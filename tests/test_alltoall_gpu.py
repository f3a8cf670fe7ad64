"""Transport all-to-all over NVLink (2+ GPUs): byte-exact delivery of
variable, skewed and empty messages (tests/a2a_worker.py)."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs >= 2 GPUs")
def test_alltoall_byte_exact():
    n = min(torch.cuda.device_count(), 8)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29534", os.path.join(HERE, "a2a_worker.py"), "4"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "A2A_OK" in r.stdout


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() >= 2,
                    reason="the multi-GPU variant above runs instead")
def test_alltoall_two_ranks_one_device():
    """A 1-GPU box: two ranks share cuda:0 (CUDA IPC between processes,
    device-side flags), byte-exact delivery incl. empty / incast messages."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29536", os.path.join(HERE, "a2a_worker.py"), "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=dict(os.environ, CN_SHARE_DEVICE="1"))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "A2A_OK" in r.stdout
