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


def bf16_fold_rne(f):
    """The fold's rounding (oracle/chunknet_oracle.c canon_nan +
    f32_to_bf16_rne): round to nearest even; a NaN sum is the canonical
    quiet NaN 0x7FFF."""
    u = f.astype(np.float32).view(np.uint32).astype(np.uint64)
    nan = ((u & 0x7F800000) == 0x7F800000) & ((u & 0x7FFFFF) != 0)
    r = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    r = np.where(nan, 0x7FFF, r)
    return r.astype(np.uint16)


def test_fused_reduce_bf16_special_values():
    """bf16 reduce on the values a rounding shortcut gets wrong: NaNs with
    payloads (the sum is the canonical quiet NaN), infinities, sums that
    overflow or round up to infinity, subnormals, signed zeros, ties to even."""
    import paper_2504_17307_b200 as cn
    data, acks_ref, cpls_ref, meta = load_golden("k8_4x1m")
    rs = np.random.RandomState(3)
    special = np.array([0x7FC1, 0x7F81, 0xFF85, 0x7F80, 0xFF80, 0x7F7F, 0xFF7F, 0x0001, 0x8001, 0x007F,
                        0x0000, 0x8000, 0x3F80, 0xBF80, 0x4000, 0x3F81], dtype=np.uint16)
    msgs = {}
    for tag, ln in sorted({(int(t), int(l)) for t, l in zip(data["msg_tag"], data["msg_len"])}):
        n = ln // 2
        v = rs.randint(0, 1 << 16, size=n).astype(np.uint16)
        a = rs.randint(0, 1 << 16, size=n).astype(np.uint16)
        k = rs.randint(0, 4, size=n) == 0  # a quarter from the special values, both operands
        v[k] = special[rs.randint(0, len(special), size=int(k.sum()))]
        a[k] = special[rs.randint(0, len(special), size=int(k.sum()))]
        want = bf16_fold_rne(bf16_to_f32(a) + bf16_to_f32(v))
        msgs[tag] = (v.view(np.uint8), a.view(np.uint8), want.view(np.uint8))
    tr = cn.Transport(cn.TransportConfig(chunk_bytes=meta["chunk_bytes"], carry_payload=True),
                      reduce="sum_bf16", max_posts=64, arena_bytes=1 << 20, chunk_pool=1 << 18,
                      max_batch=1 << 16)
    bufs = {}
    for tag, (v, a, want) in msgs.items():
        bufs[tag] = torch.from_numpy(a.copy()).cuda()
        tr.post(tag, bufs[tag])
    tr.handle_packets(cn.to_device_records(data), torch.from_numpy(staging_of(data, msgs)).cuda())
    for tag, (v, a, want) in msgs.items():
        got = bufs[tag].cpu().numpy().view(np.uint16)
        bad = np.nonzero(got != want.view(np.uint16))[0]
        assert len(bad) == 0, (tag, [(int(a.view(np.uint16)[j]), int(v.view(np.uint16)[j]), int(got[j]),
                                       int(want.view(np.uint16)[j])) for j in bad[:5]])


def test_fused_reduce_f32_special_values():
    """fp32 reduce: NaN payloads (canonical quiet NaN sum), inf - inf,
    overflow, subnormals, signed zeros."""
    import paper_2504_17307_b200 as cn
    data, acks_ref, cpls_ref, meta = load_golden("k8_4x1m")
    rs = np.random.RandomState(5)
    special = np.array([0x7FC00001, 0x7F800001, 0xFF812345, 0x7F800000, 0xFF800000, 0x7F7FFFFF, 0xFF7FFFFF,
                        0x00000001, 0x80000001, 0x007FFFFF, 0x00000000, 0x80000000, 0x3F800000],
                       dtype=np.uint32)
    msgs = {}
    for tag, ln in sorted({(int(t), int(l)) for t, l in zip(data["msg_tag"], data["msg_len"])}):
        n = ln // 4
        v = rs.uniform(-1, 1, size=n).astype(np.float32).view(np.uint32)
        a = rs.uniform(-1, 1, size=n).astype(np.float32).view(np.uint32)
        k = rs.randint(0, 4, size=n) == 0
        v[k] = special[rs.randint(0, len(special), size=int(k.sum()))]
        a[k] = special[rs.randint(0, len(special), size=int(k.sum()))]
        with np.errstate(all="ignore"):
            s_ = a.view(np.float32) + v.view(np.float32)
        want = np.where(np.isnan(s_), np.uint32(0x7FFFFFFF), s_.view(np.uint32)).astype(np.uint32)
        msgs[tag] = (v.view(np.uint8), a.view(np.uint8), want.view(np.uint8))
    tr = cn.Transport(cn.TransportConfig(chunk_bytes=meta["chunk_bytes"], carry_payload=True),
                      reduce="sum_f32", max_posts=64, arena_bytes=1 << 20, chunk_pool=1 << 18, max_batch=1 << 16)
    bufs = {}
    for tag, (v, a, want) in msgs.items():
        bufs[tag] = torch.from_numpy(a.copy()).cuda()
        tr.post(tag, bufs[tag])
    tr.handle_packets(cn.to_device_records(data), torch.from_numpy(staging_of(data, msgs)).cuda())
    for tag, (v, a, want) in msgs.items():
        got = bufs[tag].cpu().numpy().view(np.uint32)
        bad = np.nonzero(got != want.view(np.uint32))[0]
        assert len(bad) == 0, (tag, [(hex(int(a.view(np.uint32)[j])), hex(int(v.view(np.uint32)[j])),
                                       hex(int(got[j])), hex(int(want.view(np.uint32)[j]))) for j in bad[:5]])
