"""Profiling helper (not a test): rank-0 GPU timeline (kernels and copies,
CUPTI via torch.profiler) of pipelined ring all-reduce iterations.
    torchrun --nproc-per-node 2 tests/ring_timeline_tool.py [piece_mb] [iters]"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    piece = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2504_17307_b200.collective import RingAllreduce
    count = (1 << 30) // 4
    ring = RingAllreduce(count, torch.float32, piece_bytes=piece << 20)
    ring.buffer().normal_()
    ring.run()
    ring.capture()
    for _ in range(3):
        ring.run()
    torch.cuda.synchronize()
    dist.barrier()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(iters):
            ring.run()
        torch.cuda.synchronize()
    dist.barrier()
    if dist.get_rank() == 0:
        evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
        rows = sorted((e.time_range.start, e.time_range.end, e.name) for e in evs)
        t0 = rows[0][0]
        agg = {}
        for a, b, nm in rows:
            short = nm.split("(")[0].replace("void ", "").replace("cnb::", "")[:34]
            agg.setdefault(short, [0, 0.0])
            agg[short][0] += 1
            agg[short][1] += b - a
            if os.environ.get("ALL") or "Memcpy" in nm or "k_copy" in nm or "k_ingest" in nm:
                print(f"{a - t0:9.1f} {b - t0:9.1f} {b - a:7.1f}  {short}")
        print("span us", rows[-1][1] - t0)
        for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            print(f"{k:36s} n={c:4d} total={t:9.1f} us")
    ring.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
