"""Device ring all-reduce over NVLink (2+ GPUs): bit-exact vs the oracle fold."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs >= 2 GPUs")
@pytest.mark.parametrize("dtype,piece,mode", [("f32", 32 << 20, "eager"), ("bf16", 32 << 20, "eager"),
                                              ("f32", 256 << 10, "eager"), ("bf16", 192 << 10, "graph")])
def test_ring_allreduce_bit_exact(dtype, piece, mode):
    """Whole segments per step, and 4-8 pipelined pieces per step (eager
    launches and a captured CUDA graph replayed in place)."""
    n = min(torch.cuda.device_count(), 8)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29533",
           os.path.join(HERE, "ring_worker.py"), str((1 << 20) + 37), dtype, "3", str(piece), mode]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "RING_OK" in r.stdout


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() >= 2,
                    reason="the multi-GPU variant above runs instead")
@pytest.mark.parametrize("dtype,piece,mode", [("f32", 256 << 10, "eager"), ("bf16", 192 << 10, "graph")])
def test_ring_allreduce_two_ranks_one_device(dtype, piece, mode):
    """A 1-GPU box: two ranks (processes) share cuda:0 -- the same CUDA IPC
    peer mappings, copy-engine pushes and device-side flags as over NVLink,
    time-sliced on one device -- bit-exact vs the oracle fold."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29535",
           os.path.join(HERE, "ring_worker.py"), str((1 << 18) + 37), dtype, "2", str(piece), mode]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=dict(os.environ, CN_SHARE_DEVICE="1"))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "RING_OK" in r.stdout
