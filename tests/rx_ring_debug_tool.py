"""Debug helper (not a test): replays a golden trace in small batches
through a receiver with a small chunk pool / arena / generation table and
prints the ring occupancy after each batch.  Usage:
    python tests/rx_ring_debug_tool.py NAME NSPLIT POOL ARENA_BLOCKS MAX_MSGS"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    name, nsplit, pool, ab, mm = sys.argv[1], *map(int, sys.argv[2:6])
    from conftest import load_golden
    from oracle import oracle as O
    import paper_2504_17307_b200 as cn
    data, acks_ref, cpls_ref, meta = load_golden(name)
    cb = meta["chunk_bytes"]
    tr = cn.Transport(cn.TransportConfig(chunk_bytes=cb, carry_payload=True), chunk_pool=pool,
                      arena_bytes=ab * cb, max_msgs=mm, max_batch=1 << 17)
    cuts = np.linspace(0, len(data), nsplit + 1).astype(int)
    for a, b in zip(cuts[:-1], cuts[1:]):
        hd = cn.to_device_records(data[a:b])
        pl = torch.from_numpy(O.fill_staging(data[a:b], stride=4032)).cuda()
        try:
            out = tr.handle_packets(hd, pl)
            nc = len(out.completions_np())
        except Exception as e:  # noqa: BLE001
            print(a, b, "ERROR", e, tr.usage())
            return
        print(a, b, "cpl", nc, tr.usage())


if __name__ == "__main__":
    main()
