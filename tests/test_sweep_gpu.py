"""configs[4] traffic (bench.synth_trace: many connections into one
receiver, S3-scheduled paths, round-robin + windowed reordering): the device
receive path equals the oracle -- ack stream, completions, buffers -- for
several message sizes, in one batch and split."""
import numpy as np
import pytest

from oracle import oracle as O
from oracle.records import CPL_FIELDS, ack_equal

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("conns,size,msgs", [(64, 4096, 1), (48, 64 * 1024 + 17, 1), (9, 1 << 20, 1),
                                             (300, 100, 1), (256, 4096, 4), (40, 64 * 1024, 4),
                                             (1024, 4096, 12)])
def test_synthetic_many_connections_match_oracle(conns, size, msgs):
    """msgs > 1: several concurrent messages per connection (the sweep's
    small-message batches); 12,288 messages in one batch: the batch plan
    built by the grid in 1,024-message slices (4,096 per third)."""
    import bench
    import paper_2504_17307_b200 as cn
    data = bench.synth_trace(conns, size, seed=size % 97, msgs=msgs)
    o_acks, o_cpls, o_arena, cnt = O.OracleRx().batch(data, O.fill_staging(data))
    assert cnt.n_completions == conns * msgs
    conns *= msgs
    for nsplit in (1, 3):
        tr = cn.Transport(cn.TransportConfig(chunk_bytes=32768, carry_payload=True), device="cuda",
                          arena_bytes=conns * (size + 64) + (1 << 20), chunk_pool=4 * conns * (-(-size // 32768)) + 64,
                          max_batch=len(data), max_conns=2 * conns + 8, max_msgs=2 * conns + 8)
        cuts = np.linspace(0, len(data), nsplit + 1).astype(int)
        acks, cpls = [], []
        for a, b in zip(cuts[:-1], cuts[1:]):
            out = tr.handle_packets(cn.to_device_records(data[a:b]),
                                    __import__("torch").from_numpy(O.fill_staging(data[a:b])).cuda())
            ak = out.acks_np().copy()
            ak["pkt_index"] += np.uint32(a)
            acks.append(ak)
            cp = out.completions_np().copy()
            cp["pkt_index"] += np.uint32(a)
            cpls.append(cp)
            arena = tr.arena()
            for c in out.completions_np():
                buf = arena[int(c["buf_offset"]): int(c["buf_offset"]) + int(c["len"])].cpu().numpy()
                assert (buf == O.pattern_bytes(int(c["len"]), int(c["tag"]))).all()
        ok, bad = ack_equal(np.concatenate(acks), o_acks)
        assert ok, (nsplit, bad)
        cp = np.concatenate(cpls)
        for f in ("tag", "src", "dst", "len", "msg_seq", "pkt_index", "msg_id"):
            assert (cp[f] == o_cpls[f]).all(), f


def test_many_messages_pipelined_generations_match_oracle():
    """4,096 messages per batch through a pipelined receiver, generation j =
    the same traffic with msg_seq + j, back to back (no reset): each batch's
    ack stream and completions equal a stateful oracle's, each generation's
    bytes are checked once the next batch returned.  Every batch retires
    4,096 messages into a 16K-slot message table (the tombstone compaction
    after retirement keeps it usable; the rebuild backstop at 1/4 would
    otherwise fire every batch), and the plan is the grid-built one."""
    import torch

    import bench
    import paper_2504_17307_b200 as cn
    conns, size, msgs, gens = 512, 4096, 8, 8
    base = bench.synth_trace(conns, size, seed=5, msgs=msgs)
    nmsg = conns * msgs
    orx = O.OracleRx()
    tr = cn.Transport(cn.TransportConfig(chunk_bytes=32768, carry_payload=True), device="cuda",
                      arena_bytes=4 * nmsg * (size + 512) + (1 << 20), chunk_pool=4 * nmsg + 64,
                      max_batch=len(base), max_conns=2 * conns + 8, max_msgs=2 * nmsg + 16, pipeline=True)
    prev = None
    for j in range(gens + 1):
        if j < gens:
            data = base.copy()
            data["msg_seq"] += j
            o_acks, o_cpls, _, cnt = orx.batch(data, O.fill_staging(data))
            assert cnt.n_completions == nmsg
            out = tr.handle_packets(cn.to_device_records(data), torch.from_numpy(O.fill_staging(data)).cuda())
            ak = out.acks_np().copy()
            ok, bad = ack_equal(ak, o_acks)
            assert ok, (j, bad)
            cp = out.completions_np().copy()
            for f in ("tag", "src", "dst", "len", "msg_seq", "pkt_index", "msg_id"):
                assert (cp[f] == o_cpls[f]).all(), (j, f)
        else:
            tr.flush()
            cp = None
        torch.cuda.synchronize()
        if prev is not None:  # the previous generation's bytes are final now
            arena = tr.arena()
            for c in prev[:: 7]:
                buf = arena[int(c["buf_offset"]): int(c["buf_offset"]) + int(c["len"])].cpu().numpy()
                assert (buf == O.pattern_bytes(int(c["len"]), int(c["tag"]))).all(), (j, int(c["tag"]))
        prev = cp
