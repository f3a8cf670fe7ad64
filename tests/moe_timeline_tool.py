"""Profiling helper (not a test): rank-0 / rank-1 GPU timelines of the MoE
all-to-all step (bench.moe_bench's workload).
    torchrun --nproc-per-node 2 tests/moe_timeline_tool.py"""
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
    pb = int(os.environ.get("CN_A2A_PIECE_MB", "113")) << 20
    direct = os.environ.get("CN_A2A_DIRECT", "1") == "1"
    a2a, a2c = AllToAll(cap, piece_bytes=pb, direct=direct), AllToAll(cap, piece_bytes=pb, direct=direct)
    coffs = [s_ * a2a.cap for s_ in range(world)]

    def step():
        recv = a2a.run(send, sc, rc, send_offsets=offs)
        a2c.run(recv, rc, sc, send_offsets=coffs)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(2):
            step()
        torch.cuda.synchronize()
    dist.barrier()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    rows_ = sorted((e.time_range.start, e.time_range.end, e.name) for e in evs)
    # a common origin over the ranks (CUPTI stamps are host-clock based)
    t0t = torch.tensor([float(rows_[0][0])], device="cuda", dtype=torch.float64)
    dist.all_reduce(t0t, op=dist.ReduceOp.MIN)
    for who in range(world):
        if who == rank:
            st_ = [r_ for r_ in rows_[len(rows_) // 2:]]
            print(f"==== rank {rank} step span {(st_[-1][1] - st_[0][0]):.1f} us over the last step")
            t0 = float(t0t.item())
            print(f"==== rank {rank}")
            for a, b, nm in rows_[len(rows_) // 2:]:
                short = nm.split("(")[0].replace("void ", "").replace("cnb::", "")[:30]
                if b - a > 3 or "Memcpy" in nm:
                    print(f"{a - t0:9.1f} {b - t0:9.1f} {b - a:7.1f}  {short}")
            sys.stdout.flush()
        dist.barrier()
    a2a.close()
    a2c.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
