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
                                             (300, 100, 1), (256, 4096, 4), (40, 64 * 1024, 4)])
def test_synthetic_many_connections_match_oracle(conns, size, msgs):
    """msgs > 1: several concurrent messages per connection (the sweep's
    small-message batches)."""
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
