"""Profiling helper (not a test): configs[4] sweep points alone (for A/B runs
of library builds via CHUNKNET_B200_LIB)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
r = bench.sweep_bench(dev, 1, 0, sizes=(1 << 20, 16 << 20, 256 << 20))
print(os.path.basename(os.environ.get("CHUNKNET_B200_LIB", "current")), os.environ.get("CN_ARENA_PAD_KB", ""),
      [(x["msg_bytes"] >> 20, x["msgs_per_conn"], x["ms_per_batch"]) for x in r if x["msgs_per_conn"] == 1])
