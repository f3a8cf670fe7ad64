"""Profiling helper (not a test): bench.py's fused-reduce leg alone (for A/B
runs of two library builds via CHUNKNET_B200_LIB)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
data1, meta, _ = bench.load_trace("cfg2_32k")
data = bench.interleave(data1, 4)
peak, _ = bench.peaks()
r = bench.fused_reduce_bench(dev, data, meta, 4, peak)
print(os.environ.get("CHUNKNET_B200_LIB", "current"), json.dumps({k: r[k]["kernel_ms"] for k in ("fp32", "bf16")}))
