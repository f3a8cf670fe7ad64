"""Profiling helper (not a test): the sender-engine leg of bench.py at
several host counts (one warp per source host: occupancy hides latency)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
for c in (1024, 2048, 4096, 8192):
    r = bench.sender_bench(dev, conns=c)
    print(c, json.dumps({k: r[k] for k in ("acks_per_s", "ms", "parity_chunk_rtx")}), flush=True)
