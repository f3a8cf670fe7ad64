"""Profiling helper (not a test): the MoE dispatch alone through AllToAll,
timed per call, with parts of the protocol switched off by CN_A2A_SKIP
(comma list: rx = no receive path, hdr = no header copies) -- to locate
what slows the copy engine below the bare protocol's rate (tools/p2p_probe.py).
    torchrun --nproc-per-node 2 tools/a2a_probe.py"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import bench
    from paper_2504_17307_b200.alltoall import AllToAll
    world, rank = dist.get_world_size(), dist.get_rank()
    tokens, hidden = 4096, 7168
    row = hidden * 2
    routing = bench.moe_routing(world, tokens)
    rows = np.stack([r_[1] for r_ in routing])
    rows_self = rows.copy()
    np.fill_diagonal(rows, 0)
    tok, _ = routing[rank]
    x = torch.randn(tokens, hidden, device="cuda").to(torch.bfloat16)
    send = x.index_select(0, torch.from_numpy(tok).cuda()).view(torch.uint8).reshape(-1)
    offs = np.concatenate([[0], np.cumsum(rows_self[rank])[:-1]]) * row
    sc, rc = rows[rank] * row, rows[:, rank] * row
    cap = int(max(rows.max() * row, 16))
    for pb_mb, tail in ((64, 0), (32, 2), (48, 2), (32, 3), (64, 1)):
        for direct in (True, False):
            a2a = AllToAll(cap, piece_bytes=pb_mb << 20, direct=direct, tail=tail)
            for _ in range(3):
                a2a.run(send, sc, rc, send_offsets=offs)
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                a2a.run(send, sc, rc, send_offsets=offs)
            e1.record()
            torch.cuda.synchronize()
            a2a.check()
            t = torch.tensor([e0.elapsed_time(e1) / 5], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            hot = int(rows[:, 0].sum()) * row
            if rank == 0:
                print(f"dispatch only, pieces {pb_mb} MiB tail {tail}, direct={direct}: {float(t.item()):.3f} ms = "
                      f"{hot / (float(t.item()) * 1e-3) / 1e9:.1f} GB/s into the hot rank "
                      f"(skip={os.environ.get('CN_A2A_SKIP', '')})", flush=True)
            a2a.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
