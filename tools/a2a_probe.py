"""Profiling helper (not a test): the MoE dispatch and combine through
AllToAll, each phase alone, alternating, synchronized between, and with a
freshly written combine source -- to locate what slows a phase below the
bare protocol's rate (tools/p2p_probe.py).
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
    direct = os.environ.get("CN_A2A_DIRECT", "1") == "1"
    pb = int(os.environ.get("CN_A2A_PIECE_MB", "64")) << 20
    a2a = AllToAll(cap, piece_bytes=pb, direct=direct)
    a2c = AllToAll(cap, piece_bytes=pb, direct=direct)
    coffs = [s_ * a2a.cap for s_ in range(world)]
    recv = a2a.run(send, sc, rc, send_offsets=offs)
    variants = {
        "dispatch only": lambda: a2a.run(send, sc, rc, send_offsets=offs),
        "combine only": lambda: a2c.run(recv, rc, sc, send_offsets=coffs),
        "dispatch + combine": lambda: (a2a.run(send, sc, rc, send_offsets=offs),
                                       a2c.run(recv, rc, sc, send_offsets=coffs)),
        "dispatch + combine, synchronized between": None,
        "dispatch only, alternating two AllToAll objects": "alt",
        "combine only, its source rewritten before each call": "rewrite",
    }
    scratch = torch.empty_like(recv)
    a2b = AllToAll(cap, piece_bytes=pb, direct=direct)
    alt = [0]
    for name, fn in variants.items():
        def step():
            if fn == "rewrite":
                recv.copy_(scratch)  # the combine's source freshly written (dirty in L2)
                a2c.run(recv, rc, sc, send_offsets=coffs)
            elif fn == "alt":
                (a2a if alt[0] % 2 == 0 else a2b).run(send, sc, rc, send_offsets=offs)
                alt[0] += 1
            elif fn is not None:
                fn()
            else:
                a2a.run(send, sc, rc, send_offsets=offs)
                torch.cuda.synchronize()
                dist.barrier()
                a2c.run(recv, rc, sc, send_offsets=coffs)
                torch.cuda.synchronize()
                dist.barrier()
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        import time
        h0 = time.perf_counter()
        e0.record()
        for _ in range(5):
            step()
        e1.record()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - h0) * 1e3 / 5
        t = torch.tensor([e0.elapsed_time(e1) / 5], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            print(f"{name}: {float(t.item()):.3f} ms (wall {wall:.3f} ms), pieces {pb >> 20} MiB, direct={direct}",
                  flush=True)
    a2a.check()
    a2c.check()
    a2a.close()
    a2c.close()
    a2b.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
