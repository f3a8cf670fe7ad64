"""torchrun worker: transport all-to-all (paper_2504_17307_b200.alltoall)
delivers every peer's message byte-exactly into the right receive slot, for
varying (incl. empty and skewed) message sizes across calls."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def counts_matrix(n, it, cap):
    rs = np.random.RandomState(100 + it)
    m = rs.randint(0, cap // 16, size=(n, n)) * 16
    m[:, 0] = np.minimum(cap, m[:, 0] * 4)  # rank 0 is the hot receiver (incast)
    m[rs.rand(n, n) < 0.15] = 0            # some empty messages
    np.fill_diagonal(m, 0)
    return m


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n, r = dist.get_world_size(), dist.get_rank()
    from paper_2504_17307_b200.alltoall import AllToAll
    cap = 3 << 20
    for direct in (True, False):  # bytes straight into the receive slots / staged + scattered
        run_mode(AllToAll(cap, direct=direct), n, r, iters, cap)
    # several pieces per message: the receive path on the whole message once its
    # headers land (early), or piece by piece as each lands
    for early in (True, False):
        run_mode(AllToAll(cap, direct=True, piece_bytes=1 << 20, early=early), n, r, iters, cap)
    # odd message sizes: unaligned pieces fall back from SM stores to the copy engines
    run_mode(AllToAll(cap, direct=True), n, r, 2, cap, odd=3)
    dist.barrier()
    if r == 0:
        print(f"A2A_OK n={n} iters={iters}")
    dist.destroy_process_group()


def run_mode(a2a, n, r, iters, cap, odd=0):
    for it in range(iters):
        m = counts_matrix(n, it, cap)
        if odd:
            m = np.where(m > 0, np.minimum(m + odd, cap), m)
        g = torch.Generator(device="cuda")
        g.manual_seed(1000 * it + r)
        send = torch.randint(0, 256, (int(m[r].sum()) + 16,), dtype=torch.uint8, device="cuda", generator=g)
        recv = a2a.run(send, list(m[r]), list(m[:, r]))
        torch.cuda.synchronize()
        a2a.check()
        # every source's send buffer, regenerated from its seed
        for s in range(n):
            if s == r or m[s, r] == 0:
                continue
            gs = torch.Generator(device="cuda")
            gs.manual_seed(1000 * it + s)
            ss = torch.randint(0, 256, (int(m[s].sum()) + 16,), dtype=torch.uint8, device="cuda", generator=gs)
            off = int(m[s, :r].sum())
            want = ss[off: off + int(m[s, r])]
            got = recv[s * a2a.cap: s * a2a.cap + int(m[s, r])]
            assert torch.equal(got, want), f"rank {r} iter {it} direct={a2a.direct} from {s}: mismatch"
    dist.barrier()
    a2a.close()


if __name__ == "__main__":
    main()
