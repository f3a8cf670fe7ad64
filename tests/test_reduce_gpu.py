"""Fused reassembly + ring-reduction step: the receive
path's scatter with dst = dst + payload, over the reference's recorded
packet traces (reordering, duplicates, retransmissions).  Bit-exact vs the
elementwise fold acc0 + msg (each element added once, IEEE fp32 add;
bf16: fp32 add then round-to-nearest-even)."""
import numpy as np
import pytest
import torch

from conftest import load_golden
from oracle.records import ack_equal

pytestmark = pytest.mark.gpu

TRACES = ["cfg1", "k8_4x1m", "multigen_k8", "csn_wrap", "multipath_k4", "lossy_2m"]


def bf16_bits(x):
    u = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def bf16_to_f32(b):
    return (b.astype(np.uint32) << 16).view(np.float32)


def make_messages(data, dtype, seed):
    rs = np.random.RandomState(seed)
    msgs = {}
    for tag, ln in sorted({(int(t), int(l)) for t, l in zip(data["msg_tag"], data["msg_len"])}):
        if dtype == "f32":
            v = rs.uniform(-1, 1, size=ln // 4).astype(np.float32)
            a = rs.uniform(-1, 1, size=ln // 4).astype(np.float32)
            msgs[tag] = (v.view(np.uint8), a.view(np.uint8), (a + v).view(np.uint8))
        else:
            v = bf16_bits(rs.uniform(-1, 1, size=ln // 2))
            a = bf16_bits(rs.uniform(-1, 1, size=ln // 2))
            want = bf16_bits(bf16_to_f32(a) + bf16_to_f32(v))
            msgs[tag] = (v.view(np.uint8), a.view(np.uint8), want.view(np.uint8))
    return msgs


def staging_of(data, msgs, stride=4032):
    st = np.zeros(len(data) * stride, dtype=np.uint8)
    for i, p in enumerate(data):
        off = int(p["chunk_offset"]) + int(p["seq_in_chunk"]) * 4032
        ln = int(p["payload_len"])
        st[i * stride: i * stride + ln] = msgs[int(p["msg_tag"])][0][off: off + ln]
    return st


@pytest.mark.parametrize("name", TRACES)
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_fused_reduce_bit_exact(name, dtype):
    import paper_2504_17307_b200 as cn
    data, acks_ref, cpls_ref, meta = load_golden(name)
    msgs = make_messages(data, dtype, 7)
    tr = cn.Transport(cn.TransportConfig(chunk_bytes=meta["chunk_bytes"], carry_payload=True),
                      reduce="sum_f32" if dtype == "f32" else "sum_bf16", max_posts=64,
                      arena_bytes=1 << 20, chunk_pool=1 << 18, max_batch=1 << 16)
    bufs = {}
    for tag, (v, a, want) in msgs.items():
        bufs[tag] = torch.from_numpy(a.copy()).cuda()
        tr.post(tag, bufs[tag])
    out = tr.handle_packets(cn.to_device_records(data),
                            torch.from_numpy(staging_of(data, msgs)).cuda())
    ok, bad = ack_equal(out.acks_np(), acks_ref)  # bookkeeping unchanged by the fusion
    assert ok, bad
    cp = out.completions_np()
    assert len(cp) == len(cpls_ref)
    for c in cp:
        assert int(c["reserved"]) == bufs[int(c["tag"])].data_ptr()
    for tag, (v, a, want) in msgs.items():
        assert np.array_equal(bufs[tag].cpu().numpy(), want), tag


def test_zero_copy_source_addressing():
    """payload_stride 0: payloads read in place from the sender's message
    buffer (the NVLink peer-read mode of the ring)."""
    import paper_2504_17307_b200 as cn
    data, acks_ref, _, meta = load_golden("k8_4x1m")
    msgs = make_messages(data, "f32", 3)
    tr = cn.Transport(cn.TransportConfig(chunk_bytes=meta["chunk_bytes"], carry_payload=True),
                      reduce="sum_f32", max_posts=16, arena_bytes=1 << 20, max_batch=1 << 14,
                      chunk_pool=1 << 16)
    hd = cn.to_device_records(data)
    for tag, (v, a, want) in msgs.items():
        # one message per batch: the in-place source is that message's buffer
        sel = data["msg_tag"] == tag
        buf = torch.from_numpy(a.copy()).cuda()
        src = torch.from_numpy(v.copy()).cuda()
        tr.post(tag, buf)
        out = tr.handle_packets(cn.to_device_records(data[sel]), src, stride=0)
        assert out.result.n_completions == 1
        assert np.array_equal(buf.cpu().numpy(), want)
