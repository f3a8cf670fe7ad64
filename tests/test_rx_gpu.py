"""Parity of the sm_100a receive path (csrc/rx.cu via the C ABI) with the
reference receive path (golden ack streams / completions generated from the
compiled reference, oracle/gen_fixtures.py) and the C oracle."""
import numpy as np
import pytest
import torch

from conftest import golden_names, load_golden, load_psn
from oracle import oracle as O
from oracle.records import ACK_FIELDS, CPL_FIELDS, PKT_DTYPE, ack_equal
from paper_2504_17307_b200.records import ACK_DTYPE, CPL_DTYPE

pytestmark = pytest.mark.gpu


def _transport(meta, carry=True, **kw):
    import paper_2504_17307_b200 as cn
    cfg = cn.TransportConfig(chunk_bytes=meta["chunk_bytes"], carry_payload=carry,
                             reliability="ordered" if meta.get("record", {}).get("ordered") else "selective")
    kw.setdefault("arena_bytes", 256 << 20)
    kw.setdefault("max_batch", 1 << 17)
    kw.setdefault("chunk_pool", 1 << 20)
    return cn.Transport(cfg, **kw)


def _dev(data, stride=4032):
    import paper_2504_17307_b200 as cn
    staging = O.fill_staging(data, stride=stride)
    return cn.to_device_records(data), torch.from_numpy(staging).cuda()


def _psn(name, a=0, b=None):
    p = load_psn(name)
    return None if p is None else torch.from_numpy(np.ascontiguousarray(p[a:b]).astype(np.int64)).cuda()


def _check_completions(tr, out, cpls_ref, index_base=0):
    got = out.completions_np()
    assert len(got) == len(cpls_ref)
    for f in ("tag", "src", "dst", "len"):
        assert (got[f] == cpls_ref[f]).all(), f
    assert ((got["pkt_index"] + index_base) == cpls_ref["pkt_index"]).all()
    arena = tr.arena()
    for c in got:
        buf = arena[int(c["buf_offset"]): int(c["buf_offset"]) + int(c["len"])].cpu().numpy()
        assert (buf == O.pattern_bytes(int(c["len"]), int(c["tag"]))).all(), int(c["tag"])


@pytest.mark.parametrize("name", golden_names())
def test_rx_matches_reference(name):
    data, acks_ref, cpls_ref, meta = load_golden(name)
    tr = _transport(meta)
    hd, pl = _dev(data)
    out = tr.handle_packets(hd, pl, psn=_psn(name))
    ok, bad = ack_equal(out.acks_np(), acks_ref)
    assert ok, bad
    _check_completions(tr, out, cpls_ref)
    assert tr.stats().acks_sent == meta["des_stats"]["acks_sent"]
    assert tr.stats().nacks_sent == int((acks_ref["flags"] & 4 != 0).sum())


@pytest.mark.parametrize("name", ["cfg1", "concurrent_k4", "multigen_k8", "k8_4x1m", "csn_wrap", "trim_swift",
                                  "trim_storm", "ordered_loss", "ordered_trim"])
@pytest.mark.parametrize("nsplit", [2, 7, 64])
def test_rx_batch_split_invariance(name, nsplit):
    """Persistent device state: any split of the packet sequence into
    batches yields the identical ack stream and completions."""
    data, acks_ref, cpls_ref, meta = load_golden(name)
    tr = _transport(meta)
    rs = np.random.RandomState(nsplit)
    cuts = np.unique(np.concatenate([[0, len(data)], rs.randint(0, len(data), nsplit - 1)]))
    acks, cpls, seen = [], [], []
    for a, b in zip(cuts[:-1], cuts[1:]):
        hd, pl = _dev(data[a:b])
        out = tr.handle_packets(hd, pl, psn=_psn(name, a, b))
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
    ok, bad = ack_equal(np.concatenate(acks), acks_ref)
    assert ok, bad
    cp = np.concatenate(cpls)
    for f in CPL_FIELDS:
        assert (cp[f] == cpls_ref[f]).all(), f


@pytest.mark.parametrize("name,nsplit,pool,arena_units,max_msgs", [
    ("multigen_k8", 64, 52, 392, 2), ("concurrent_k4", 40, 300, 4464, 8), ("closed_w4", 30, 384, 6456, 4)])
def test_rx_steady_state_reclaims(name, nsplit, pool, arena_units, max_msgs):
    """A long-running receiver whose chunk pool, arena and generation table
    are several times smaller than the trace's total: delivered messages
    hand their chunk range, arena blocks and table slot back (the reference
    frees MsgRecv state and buffer at delivery, transport.cpp:794-803), so
    the stream runs without a capacity error and with the identical acks,
    completions and buffers.  Sizes: the smallest rings that hold the trace
    at this batching (a ring's tail waits for its oldest live message)."""
    data, acks_ref, cpls_ref, meta = load_golden(name)
    cb = meta["chunk_bytes"]
    total = sum((int(L) + cb - 1) // cb for L in cpls_ref["len"])
    assert total > pool and sum((int(L) + 511) // 512 for L in cpls_ref["len"]) > arena_units  # rings wrap
    tr = _transport(meta, chunk_pool=pool, arena_bytes=arena_units * 512, max_msgs=max_msgs)
    cuts = np.linspace(0, len(data), nsplit + 1).astype(int)
    acks, cpls = [], []
    for a, b in zip(cuts[:-1], cuts[1:]):
        hd, pl = _dev(data[a:b])
        out = tr.handle_packets(hd, pl, psn=_psn(name, a, b))
        ak = out.acks_np().copy()
        ak["pkt_index"] += np.uint32(a)
        acks.append(ak)
        cp = out.completions_np().copy()
        cp["pkt_index"] += np.uint32(a)
        cpls.append(cp)
        arena = tr.arena()
        for c in out.completions_np():
            assert int(c["buf_offset"]) + int(c["len"]) <= 2 * arena_units * 512  # ring + overhang
            buf = arena[int(c["buf_offset"]): int(c["buf_offset"]) + int(c["len"])].cpu().numpy()
            assert (buf == O.pattern_bytes(int(c["len"]), int(c["tag"]))).all()
    ok, bad = ack_equal(np.concatenate(acks), acks_ref)
    assert ok, bad
    cp = np.concatenate(cpls)
    for f in CPL_FIELDS:
        assert (cp[f] == cpls_ref[f]).all(), f


def test_rx_no_payload_mode_same_acks():
    data, acks_ref, cpls_ref, meta = load_golden("cfg2_32k")
    tr = _transport(meta, carry=False)
    import paper_2504_17307_b200 as cn
    out = tr.handle_packets(cn.to_device_records(data), None)
    ok, bad = ack_equal(out.acks_np(), acks_ref)
    assert ok, bad
    assert out.completions_np()["buf_offset"][0] == np.uint64(2**64 - 1)


def test_rx_wide_staging_stride():
    data, acks_ref, cpls_ref, meta = load_golden("k8_4x1m")
    tr = _transport(meta)
    hd, pl = _dev(data, stride=4096)
    out = tr.handle_packets(hd, pl, stride=4096)
    ok, bad = ack_equal(out.acks_np(), acks_ref)
    assert ok, bad
    _check_completions(tr, out, cpls_ref)


def test_rx_selective_ack_contract_forged():
    """test_transport.cpp:152-203 on the device path."""
    import paper_2504_17307_b200 as cn
    h = np.zeros(9, dtype=PKT_DTYPE)
    for i, c in enumerate(list(range(1, 9)) + [0]):
        h[i]["src"], h[i]["dst"] = 0, 1
        h[i]["hdr"] = cn.encode_header(9, 0, c, c == 8)
        h[i]["chunk_offset"] = c * 4032
        h[i]["chunk_len"] = 4032
        h[i]["payload_len"] = 4032
        h[i]["msg_seq"] = 1
        h[i]["msg_len"] = 9 * 4032
    tr = _transport({"chunk_bytes": 4032}, carry=False)
    out = tr.handle_packets(cn.to_device_records(h), None)
    a = out.acks_np()
    assert len(a) == 9
    for i in range(8):
        assert not (a[i]["flags"] & 1)
        assert (a[i]["hdr"] >> 9) & 0xFF == i + 1
        assert bin(int(a[i]["sack0"])).count("1") + bin(int(a[i]["sack1"])).count("1") == i + 1
    assert a[8]["flags"] & 1 and a[8]["cum_csn"] == 8 and (a[8]["hdr"] >> 9) & 0xFF == 0
    assert a[8]["sack0"] == 0 and a[8]["sack1"] == 0
    assert len(out.completions_np()) == 1


def test_rx_reset_and_rerun_identical():
    data, acks_ref, cpls_ref, meta = load_golden("multipath_k4")
    tr = _transport(meta)
    hd, pl = _dev(data)
    for _ in range(3):
        tr.reset()
        out = tr.handle_packets(hd, pl)
        ok, bad = ack_equal(out.acks_np(), acks_ref)
        assert ok, bad
        _check_completions(tr, out, cpls_ref)


def test_rx_completion_callback():
    data, acks_ref, cpls_ref, meta = load_golden("concurrent_k4")
    tr = _transport(meta)
    got = []
    tr.set_on_complete(lambda tag, src, dst, ln, t, d: got.append(
        (tag, src, dst, ln, t, bytes(d.cpu().numpy()) == bytes(O.pattern_bytes(ln, tag)))))
    hd, pl = _dev(data)
    tr.handle_packets(hd, pl)
    assert [g[:5] for g in got] == [(int(c["tag"]), int(c["src"]), int(c["dst"]), int(c["len"]),
                                     int(c["pkt_index"])) for c in cpls_ref]
    assert all(g[5] for g in got)


@pytest.mark.parametrize("frac,seed", [(0.05, 1), (0.3, 2)])
def test_rx_trimmed_headers_match_oracle(frac, seed):
    """Forged trim-mode arrivals on cfg1: a fraction of the deliveries turned
    into trimmed headers, each re-delivered a little later as a full packet
    (the retransmission a NACK asks for), some trimmed twice.  NACK records (one per chunk until a
    new packet clears `nacked`), acks and completions equal the oracle's,
    in one batch and split over batches."""
    data, _, _, meta = load_golden("cfg1")
    rs = np.random.RandomState(seed)
    tr_mask = rs.rand(len(data)) < frac
    trimmed = data.copy()
    trimmed["flags"][tr_mask] |= 4
    # keep the sender's 128-chunk window (the DES trace already reorders up
    # to ~125 chunks): re-deliveries follow within 11 packets, a second
    # trimmed copy within 5
    keys, pk = list(np.arange(len(data), dtype=np.float64)), [trimmed]
    idx = np.nonzero(tr_mask)[0]
    red = idx  # every trimmed packet is resent (the NACK's purpose) within the window
    r = data[red].copy()
    r["flags"] |= 1
    keys += list(red + rs.randint(1, 12, len(red)) + 0.5)
    pk.append(r)
    dup = idx[rs.rand(len(idx)) < 0.3]
    keys += list(dup + rs.randint(1, 6, len(dup)) + 0.25)
    pk.append(trimmed[dup])
    allp = np.concatenate(pk)
    forged = allp[np.argsort(np.array(keys), kind="stable")]
    o_acks, o_cpls, _, cnt = O.OracleRx().batch(forged, O.fill_staging(forged))
    assert cnt.n_nacks > 0 and int(((o_acks["flags"] & 4) != 0).sum()) == cnt.n_nacks
    for nsplit in (1, 5):
        tr = _transport(meta)
        cuts = np.unique(np.concatenate([[0, len(forged)], rs.randint(0, len(forged), nsplit - 1)]))
        acks = []
        for a, b in zip(cuts[:-1], cuts[1:]):
            hd, pl = _dev(forged[a:b])
            ak = tr.handle_packets(hd, pl).acks_np().copy()
            ak["pkt_index"] += np.uint32(a)
            acks.append(ak)
        ok, bad = ack_equal(np.concatenate(acks), o_acks)
        assert ok, (nsplit, bad)
        assert tr.stats().nacks_sent == cnt.n_nacks


def test_rx_interleaved_connections_independent():
    """Three concurrent connections (cfg1 copies from distinct source hosts,
    round-robin interleaved): each connection's ack subsequence equals the
    single-connection reference stream."""
    import paper_2504_17307_b200 as cn
    data, acks_ref, cpls_ref, meta = load_golden("cfg1")
    K = 3
    mix = np.empty(len(data) * K, dtype=data.dtype)
    for j in range(K):
        c = data.copy()
        c["src"] = j
        c["msg_tag"] = 100 + j
        mix[j::K] = c
    tr = _transport(meta)
    hd, pl = _dev(mix)
    out = tr.handle_packets(hd, pl)
    a = out.acks_np()
    for j in range(K):
        sub = a[a["dst"] == j].copy()
        sub["pkt_index"] = (sub["pkt_index"] - j) // K
        want = acks_ref.copy()
        want["dst"] = j
        ok, bad = ack_equal(sub, want)
        assert ok, (j, bad)
    assert len(out.completions_np()) == K
    arena = tr.arena()
    for c in out.completions_np():
        buf = arena[int(c["buf_offset"]): int(c["buf_offset"]) + int(c["len"])].cpu().numpy()
        assert (buf == O.pattern_bytes(int(c["len"]), int(c["tag"]))).all()


@pytest.mark.parametrize("name", ["cfg1", "cfg2_32k", "concurrent_k4", "multigen_k8", "trim_storm", "ordered_loss"])
@pytest.mark.parametrize("nsplit", [3, 16])
def test_rx_pipelined_receiver(name, nsplit):
    """cn_rx_config::pipeline: the scatter of batch k runs beside batch k+1
    and joins at its end.  Batches are enqueued back to back with their own
    output buffers and no host synchronisation: the ack streams and
    completions are the reference's, batch k's message bytes are final once
    batch k+1 has returned (checked after each batch), the last batch's after
    cn_rx_flush."""
    import ctypes

    from paper_2504_17307_b200 import _lib
    data, acks_ref, cpls_ref, meta = load_golden(name)
    tr = _transport(meta, pipeline=True)
    L = _lib.lib()
    s = torch.cuda.current_stream()
    rs = np.random.RandomState(nsplit)
    cuts = np.unique(np.concatenate([[0, len(data)], rs.randint(0, len(data), nsplit - 1)]))
    keep, outs = [], []

    def check_bytes(cp):
        arena = tr.arena()
        for c in cp:
            buf = arena[int(c["buf_offset"]): int(c["buf_offset"]) + int(c["len"])].cpu().numpy()
            assert (buf == O.pattern_bytes(int(c["len"]), int(c["tag"]))).all(), int(c["tag"])

    for j, (a, b) in enumerate(zip(cuts[:-1], cuts[1:])):
        hd, pl = _dev(data[a:b])
        n = b - a
        acks = torch.empty((n + 16) * 64, dtype=torch.uint8, device="cuda")
        cpls = torch.empty((n + 16) * 64, dtype=torch.uint8, device="cuda")
        res = torch.zeros(24, dtype=torch.uint8, device="cuda")
        psn = _psn(name, a, b)
        args = (hd.data_ptr(), pl.data_ptr(), 4032, n, acks.data_ptr(), n + 16, cpls.data_ptr(), n + 16,
                res.data_ptr(), ctypes.c_void_p(s.cuda_stream))
        if psn is not None:
            _lib.check(L.cn_rx_batch_psn(tr._h, args[0], psn.data_ptr(), *args[1:]), "cn_rx_batch_psn")
        else:
            _lib.check(L.cn_rx_batch(tr._h, *args), "cn_rx_batch")
        keep.append((hd, pl, psn))
        outs.append((a, acks, cpls, res))
        if j % 4 == 3:  # now and then: batch j-1's bytes are final once batch j returned
            torch.cuda.synchronize()
            if j >= 1:
                r = _lib.RxResult.from_buffer_copy(bytes(outs[j - 1][3].cpu().numpy()))
                check_bytes(outs[j - 1][2][: r.n_completions * 64].cpu().numpy().view(CPL_DTYPE))
    tr.flush()
    torch.cuda.synchronize()
    all_acks, all_cpls = [], []
    for a, acks, cpls, res in outs:
        r = _lib.RxResult.from_buffer_copy(bytes(res.cpu().numpy()))
        assert r.status == 0
        ak = acks[: r.n_acks * 64].cpu().numpy().view(ACK_DTYPE).copy()
        ak["pkt_index"] += np.uint32(a)
        all_acks.append(ak)
        cp = cpls[: r.n_completions * 64].cpu().numpy().view(CPL_DTYPE).copy()
        check_bytes(cp)
        cp["pkt_index"] += np.uint32(a)
        all_cpls.append(cp)
    ok, bad = ack_equal(np.concatenate(all_acks), acks_ref)
    assert ok, bad
    cp = np.concatenate(all_cpls)
    for f in CPL_FIELDS:
        assert (cp[f] == cpls_ref[f]).all(), f


@pytest.mark.parametrize("name", ["cfg1", "cfg2_32k", "concurrent_k4", "multigen_k8", "odd_chunk", "ordered_loss"])
def test_rx_message_data_pointers(name):
    """The send_message_data path (transport.hpp:88-91): each packet carries
    its message's data (Packet::msg_data, set by send_chunk :486) and
    accept_payload copies from it (:719-730).  Here every packet names a
    device buffer holding its message's bytes (cn_rx_batch_msgdata); the ack
    stream, completions and reassembled buffers are the reference's."""
    data, acks_ref, cpls_ref, meta = load_golden(name)
    tr = _transport(meta)
    bufs, ptr = {}, np.zeros(len(data), dtype=np.int64)
    for i, (tag, ln) in enumerate(zip(data["msg_tag"], data["msg_len"])):
        k = (int(tag), int(ln))
        if k not in bufs:
            bufs[k] = torch.from_numpy(O.pattern_bytes(k[1], k[0]).copy()).cuda()
        ptr[i] = bufs[k].data_ptr()
    import paper_2504_17307_b200 as cn
    out = tr.handle_packets(cn.to_device_records(data), None, psn=_psn(name),
                            msg_data=torch.from_numpy(ptr).cuda())
    ok, bad = ack_equal(out.acks_np(), acks_ref)
    assert ok, bad
    _check_completions(tr, out, cpls_ref)


@pytest.mark.parametrize("name", ["cfg1", "cfg2_32k", "odd_chunk", "multigen_k8", "trim_storm"])
def test_rx_bulk_copy_variant(name, monkeypatch):
    """The scatter on the bulk-copy (TMA) engine (k_copy_tma, CN_COPY_TMA=1):
    identical buffers, incl. the 16-byte tails and the misaligned packets of
    a 5000-byte chunk size that take the warp-cooperative path."""
    monkeypatch.setenv("CN_COPY_TMA", "1")
    data, acks_ref, cpls_ref, meta = load_golden(name)
    tr = _transport(meta)
    hd, pl = _dev(data)
    out = tr.handle_packets(hd, pl, psn=_psn(name))
    ok, bad = ack_equal(out.acks_np(), acks_ref)
    assert ok, bad
    _check_completions(tr, out, cpls_ref)


@pytest.mark.parametrize("name", ["cfg1", "cfg2_32k", "odd_chunk", "trim_storm", "ordered_loss"])
def test_rx_packed_payloads(name):
    """cn_rx_batch_packed: payloads packed back to back (a NIC ring's
    variable-size packet buffers), packet i at payload + offset[i]; shuffled
    offsets too.  Same acks, completions and buffers as the reference."""
    import paper_2504_17307_b200 as cn
    data, acks_ref, cpls_ref, meta = load_golden(name)
    st = O.fill_staging(data)
    pl = data["payload_len"].astype(np.int64)
    order = np.random.RandomState(1).permutation(len(data))  # packets stored in a shuffled order
    off = np.zeros(len(data), dtype=np.int64)
    off[order] = np.concatenate([[0], np.cumsum(pl[order])[:-1]])
    packed = np.zeros(int(pl.sum()) + 16, dtype=np.uint8)
    for i in range(len(data)):
        packed[off[i]: off[i] + pl[i]] = st[i * 4032: i * 4032 + pl[i]]
    tr = _transport(meta)
    out = tr.handle_packets(cn.to_device_records(data), torch.from_numpy(packed).cuda(), psn=_psn(name),
                            offsets=torch.from_numpy(off).cuda())
    ok, bad = ack_equal(out.acks_np(), acks_ref)
    assert ok, bad
    _check_completions(tr, out, cpls_ref)
