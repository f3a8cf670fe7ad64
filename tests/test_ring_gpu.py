"""Device ring all-reduce: bit-exact vs the oracle fold.  One rank per GPU
over NVLink when the box has 2+ GPUs; on a 1-GPU box two ranks (processes)
share cuda:0 -- the same CUDA IPC peer mappings, copy-engine pushes and
device-side progress flags, time-sliced on one device."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def ranks_and_env():
    n = torch.cuda.device_count()
    if n >= 2:
        return min(n, 8), dict(os.environ)
    return 2, dict(os.environ, CN_SHARE_DEVICE="1")


@pytest.mark.parametrize("dtype,piece,mode", [("f32", 32 << 20, "eager"), ("bf16", 32 << 20, "eager"),
                                              ("f32", 256 << 10, "eager"), ("bf16", 192 << 10, "graph")])
def test_ring_allreduce_bit_exact(dtype, piece, mode):
    """Whole segments per step, and 4-8 pipelined pieces per step (eager
    launches and a captured CUDA graph replayed in place)."""
    n, env = ranks_and_env()
    count = (1 << 20) + 37 if n > 2 or "CN_SHARE_DEVICE" not in env else (1 << 18) + 37
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29533",
           os.path.join(HERE, "ring_worker.py"), str(count), dtype, "3", str(piece), mode]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "RING_OK" in r.stdout
