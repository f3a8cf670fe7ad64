"""Device ring all-reduce over NVLink (2+ GPUs): bit-exact vs the oracle fold.

Needs one GPU per rank: the ranks' progress counters are device-side spins
on flags another rank writes, and such waiting kernels must never share a
GPU (B200_PROFILING.md: ranks as processes on one GPU raised Xid 109).  On
a 1-GPU box the same schedule is checked on the CPU with gloo ranks
(tests/test_ring_cpu.py) and bench.py's N > 1 legs verify every all-reduce
they time (bench.ring_parity)."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs >= 2 GPUs (one rank per GPU; waiting kernels must not share a GPU)")
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
