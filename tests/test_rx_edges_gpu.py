"""Edge cases of the receive path through the C ABI, each against the C
oracle or the reference's contract: an empty batch, a batch replayed after
delivery (every packet stale), a malformed header and an exhausted pool
(both loud errors, never a silent fallback), a batch above max_batch."""
import numpy as np
import pytest
import torch

from conftest import load_golden
from oracle import oracle as O
from oracle.records import ack_equal

pytestmark = pytest.mark.gpu


def _transport(meta, **kw):
    import paper_2504_17307_b200 as cn
    kw.setdefault("arena_bytes", 64 << 20)
    kw.setdefault("max_batch", 1 << 16)
    kw.setdefault("chunk_pool", 1 << 16)
    return cn.Transport(cn.TransportConfig(chunk_bytes=meta["chunk_bytes"], carry_payload=True), **kw)


def _dev(data):
    import paper_2504_17307_b200 as cn
    return cn.to_device_records(data), torch.from_numpy(O.fill_staging(data)).cuda()


def test_empty_batch_is_a_no_op():
    data, acks_ref, cpls_ref, meta = load_golden("cfg1")
    tr = _transport(meta)
    hd, pl = _dev(data[:0])
    out = tr.handle_packets(hd, pl)
    assert len(out.acks_np()) == 0 and len(out.completions_np()) == 0
    hd, pl = _dev(data)  # the state is untouched: the full trace still matches
    out = tr.handle_packets(hd, pl)
    ok, bad = ack_equal(out.acks_np(), acks_ref)
    assert ok, bad


def test_replayed_batch_is_all_stale_like_the_oracle():
    """The whole trace again after delivery: every data packet is a stale
    generation (transport.cpp:602-615) -- the stale re-acks, no completion."""
    data, acks_ref, cpls_ref, meta = load_golden("multipath_k4")
    st = O.fill_staging(data)
    orc = O.OracleRx()
    orc.batch(data, st)
    o_acks, o_cpls, _, _ = orc.batch(data, st)
    tr = _transport(meta)
    hd, pl = _dev(data)
    tr.handle_packets(hd, pl)
    out = tr.handle_packets(hd, pl)
    ok, bad = ack_equal(out.acks_np(), o_acks)
    assert ok, bad
    assert len(out.completions_np()) == len(o_cpls) == 0
    assert len(o_acks) > 0


def test_malformed_header_fails_loudly():
    import paper_2504_17307_b200 as cn
    data, _, _, meta = load_golden("cfg1")
    bad = data.copy()
    bad[5]["payload_len"] += 1  # not the length the chunk's packetisation implies
    tr = _transport(meta)
    hd, pl = _dev(bad)
    with pytest.raises(cn.ChunknetError):
        tr.handle_packets(hd, pl)


def test_pool_exhaustion_fails_loudly_and_reset_recovers():
    import paper_2504_17307_b200 as cn
    data, acks_ref, _, meta = load_golden("cfg1")  # one 1 MiB message of 256 chunks
    tr = _transport(meta, chunk_pool=128)
    hd, pl = _dev(data)
    with pytest.raises(cn.ChunknetError):
        tr.handle_packets(hd, pl)
    tr2 = _transport(meta, chunk_pool=256)
    out = tr2.handle_packets(hd, pl)
    ok, bad = ack_equal(out.acks_np(), acks_ref)
    assert ok, bad


def test_batch_above_max_batch_is_rejected():
    import paper_2504_17307_b200 as cn
    data, _, _, meta = load_golden("cfg1")
    tr = _transport(meta, max_batch=256)
    hd, pl = _dev(data)
    with pytest.raises(cn.ChunknetError):
        tr.handle_packets(hd, pl)
