"""torchrun worker: device ring all-reduce vs the oracle fold (bit-exact)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    count = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 20) + 37
    dtype_s = sys.argv[2] if len(sys.argv) > 2 else "f32"
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    piece = int(sys.argv[4]) if len(sys.argv) > 4 else 32 << 20
    graph = len(sys.argv) > 5 and sys.argv[5] == "graph"
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n, r = dist.get_world_size(), dist.get_rank()
    from paper_2504_17307_b200.collective import RingAllreduce
    from oracle import oracle as O
    rs = np.random.RandomState(99)
    xs = rs.uniform(-1, 1, size=(n, count)).astype(np.float32)
    if dtype_s == "bf16":
        u = xs.view(np.uint32).astype(np.uint64)
        xs = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
        x = torch.from_numpy(xs[r].view(np.int16).copy()).view(torch.bfloat16).cuda()
        dt = torch.bfloat16
    else:
        x = torch.from_numpy(xs[r].copy()).cuda()
        dt = torch.float32
    ring = RingAllreduce(count, dt, chunk_bytes=32768, paths=8, piece_bytes=piece)
    want = O.ring_allreduce(xs, quantum=ring.quantum)
    if graph:
        ring.capture()
    for it in range(iters):
        if graph:  # in place: the captured iteration reduces the accumulator
            ring.buffer().copy_(x)
            out = ring.run()
        else:
            out = ring.run(x)
        torch.cuda.synchronize()
        ring.check()
        got = out.view(torch.int16).cpu().numpy().view(np.uint16) if dt == torch.bfloat16 \
            else out.cpu().numpy()
        assert np.array_equal(got, want), f"rank {r} iter {it}: mismatch"
    # tolerance vs an fp64 sum: fp32 rtol 1e-5*N
    if dt == torch.float32:
        exact = xs.astype(np.float64).sum(0)
        assert np.abs(got - exact).max() <= 1e-5 * n * max(1.0, np.abs(exact).max())
    dist.barrier()
    ring.close()
    if r == 0:
        print(f"RING_OK n={n} count={count} dtype={dtype_s} iters={iters} pieces={ring.pieces} graph={graph}")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
