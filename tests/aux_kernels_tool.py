"""Profiling helper (not a test): one run each of the sender-engine,
EQDS-pacer and scheduler benches (bench.py's configurations), for ncu."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if __name__ == "__main__":
    import bench
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    out = {}
    if which in ("all", "sender"):
        out["sender"] = bench.sender_bench("cuda:0", reps=1)
    if which in ("all", "eqds"):
        out["eqds"] = bench.eqds_bench("cuda:0", reps=1)
    if which in ("all", "sched"):
        out["sched"] = bench.sched_bench("cuda:0")
    print(json.dumps({k: {kk: vv for kk, vv in v.items() if not kk.startswith("cpu")} for k, v in out.items()}))
