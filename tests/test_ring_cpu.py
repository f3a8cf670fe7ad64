"""The ring schedule of paper_2504_17307_b200.collective (steps, segments,
tags, fold order) executed by world_size-2/3/8 gloo processes on CPU, against
the oracle's same-order fold (bit-exact).  Test infrastructure for the N>1
host logic; the device path is tests/test_ring_gpu.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_17307_b200.collective import ring_schedule, seg_bounds


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, n, port, count, dtype, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=n)
    rs = np.random.RandomState(1234)
    xs = rs.uniform(-1, 1, size=(n, count)).astype(np.float32)
    if dtype == "bf16":
        u = xs.view(np.uint32).astype(np.uint64)
        xs = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    acc = xs[rank].copy()
    nxt, prv = (rank + 1) % n, (rank - 1) % n
    for (k, ph, s, snd, rcv, tag) in ring_schedule(n, rank):
        if ph == "init":
            continue
        a, b = seg_bounds(count, n, snd)
        c, d = seg_bounds(count, n, rcv)
        out = torch.from_numpy(acc[a:b].copy())
        inc = torch.empty(d - c, dtype=out.dtype)
        if rank % 2 == 0:
            dist.send(out, nxt)
            dist.recv(inc, prv)
        else:
            dist.recv(inc, prv)
            dist.send(out, nxt)
        recv = inc.numpy()
        if ph == "rs":
            if dtype == "f32":
                acc[c:d] = acc[c:d] + recv
            else:
                f = ((acc[c:d].astype(np.uint32) << 16).view(np.float32) +
                     (recv.astype(np.uint32) << 16).view(np.float32))
                u = f.view(np.uint32).astype(np.uint64)
                acc[c:d] = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
        else:
            acc[c:d] = recv
    q.put((rank, acc))
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [2, 3, 8])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_ring_schedule_matches_oracle_fold(n, dtype):
    from oracle import oracle as O
    count = 1000 + n
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, n, port, count, dtype, q)) for r in range(n)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(n))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    rs = np.random.RandomState(1234)
    xs = rs.uniform(-1, 1, size=(n, count)).astype(np.float32)
    if dtype == "bf16":
        u = xs.view(np.uint32).astype(np.uint64)
        xs = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    want = O.ring_allreduce(xs)
    for r in range(n):
        assert np.array_equal(res[r], want), r


def test_schedule_covers_every_segment_once():
    for n in (2, 4, 8):
        for r in range(n):
            st = ring_schedule(n, r)
            rs_recv = [x[4] for x in st if x[1] == "rs"]
            ag_recv = [x[4] for x in st if x[1] == "ag"]
            assert len(set(rs_recv)) == n - 1 and (r + 1) % n not in ag_recv
            assert sorted(ag_recv + [(r + 1) % n]) == list(range(n))
            # what r sends at (phase, s) is what r+1 receives at (phase, s)
            nxt = ring_schedule(n, (r + 1) % n)
            for a, b in zip(st[1:], nxt[1:]):
                assert a[3] == b[4] and a[5] == b[5]
