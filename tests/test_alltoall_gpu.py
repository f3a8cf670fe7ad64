"""Transport all-to-all over NVLink (2+ GPUs): byte-exact delivery of
variable, skewed and empty messages (tests/a2a_worker.py).  One GPU per
rank (see tests/test_ring_gpu.py); bench.py's N > 1 MoE leg verifies every
slice of the dispatch and combine it times."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs >= 2 GPUs (one rank per GPU; waiting kernels must not share a GPU)")
def test_alltoall_byte_exact():
    n = min(torch.cuda.device_count(), 8)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29534", os.path.join(HERE, "a2a_worker.py"), "4"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "A2A_OK" in r.stdout
