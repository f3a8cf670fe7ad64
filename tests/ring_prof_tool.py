"""Profiling helper (not a test): per-kernel receive-path times inside the
ring all-reduce (serial profiling mode) and the whole-iteration time."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2504_17307_b200.collective import RingAllreduce
    count = (1 << 30) // 4
    ring = RingAllreduce(count, torch.float32)
    ring.buffer().normal_()
    for _ in range(2):
        ring.run()
    torch.cuda.synchronize()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    e0, e1 = ev(), ev()
    e0.record()
    for _ in range(5):
        ring.run()
    e1.record()
    torch.cuda.synchronize()
    it = e0.elapsed_time(e1) / 5
    for rx in (ring.rx_rs, ring.rx_ag):
        rx.set_profiling(True)
        rx.kernel_profile()
    e0.record()
    for _ in range(3):
        ring.run()
    e1.record()
    torch.cuda.synchronize()
    p1, n1 = ring.rx_rs.kernel_profile()
    p2, n2 = ring.rx_ag.kernel_profile()
    if dist.get_rank() == 0:
        print(f"n={ring.n} iter ms {it:.3f} (serial-profiled {e0.elapsed_time(e1) / 3:.3f})")
        print("rs", {k: round(v / n1, 4) for k, v in p1.items()}, "ag", {k: round(v / n2, 4) for k, v in p2.items()})
    ring.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
