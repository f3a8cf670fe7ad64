"""Profiling helper (not a test): phase timing of RingAllreduce.run on rank 0."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2504_17307_b200.collective import RingAllreduce, packetize
    count = (1 << 30) // 4
    x = torch.randn(count, device="cuda")
    ring = RingAllreduce(count, torch.float32)
    for _ in range(2):
        ring.run(x)
    torch.cuda.synchronize()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    e = [ev() for _ in range(4)]
    nb = ring.seg_bytes[0]
    nch = (nb + ring.cb - 1) // ring.cb
    e[0].record()
    for _ in range(5):
        ring.sched.select("p2_rtt", offsets=ring.path_offs, out=ring.paths_all)
    e[1].record()
    for _ in range(5):
        packetize(nb, ring.cb, src=0, dst=1, chunk_paths=ring.paths_all[:nch], out=ring.hdrs[1])
    e[2].record()
    for _ in range(5):
        ring.rx_rs.reset()
    e[3].record()
    torch.cuda.synchronize()
    if dist.get_rank() == 0:
        print("select ms", e[0].elapsed_time(e[1]) / 5, "packetize ms", e[1].elapsed_time(e[2]) / 5,
              "reset ms", e[2].elapsed_time(e[3]) / 5, "chunks", nch)
    ring.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
