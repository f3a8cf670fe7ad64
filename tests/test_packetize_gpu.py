"""S7 packetization (Transport::send_chunk, transport.cpp:433-494) on the
device: cn_packetize's 64-B records against the reference's own packets.

* test_transport.cpp:101-146: a 32,768 B message in one chunk is nine
  packets, eight 4,032 B payloads and a 512 B runt, seq 0..8, csn 0, last.
* Every first-transmission packet the reference DES delivered (golden
  traces; packets lost on the wire are simply absent) equals the record
  cn_packetize writes for its (message, chunk, packet) given the chunk's
  path: src, dst, path, header word (conn id, msg id, csn, last), chunk
  offset / length, payload length, seq in chunk, rtx flag, msg seq / tag /
  length.  tx_time is the caller's (the reference stamps each chunk's own
  send time; the device call stamps one time per message)."""
import numpy as np
import pytest
import torch

from conftest import load_golden

pytestmark = pytest.mark.gpu
MAX_PL = 4032
FIELDS = ("src", "dst", "path_id", "hdr", "chunk_offset", "chunk_len", "payload_len", "seq_in_chunk",
          "msg_seq", "msg_tag", "msg_len")


def _records(t):
    from oracle.records import PKT_DTYPE
    return t.cpu().numpy().view(PKT_DTYPE)


def test_packetize_single_chunk_nine_packets():
    from paper_2504_17307_b200.collective import packetize
    r = _records(packetize(32768, 32768, src=0, dst=1, conn_id=0, msg_id=0, msg_seq=1, tag=7))
    assert len(r) == 9
    assert list(r["seq_in_chunk"]) == list(range(9))
    assert list(r["payload_len"]) == [4032] * 8 + [512]
    assert ((r["hdr"] >> 9) & 0xFF == 0).all() and ((r["hdr"] >> 8) & 1 == 1).all()
    assert (r["chunk_offset"] == 0).all() and (r["chunk_len"] == 32768).all()


@pytest.mark.parametrize("name", ["cfg1", "cfg2_32k", "odd_chunk", "concurrent_k4", "multipath_k4", "csn_wrap"])
def test_packetize_matches_reference_first_transmissions(name):
    from paper_2504_17307_b200 import _lib
    from paper_2504_17307_b200.collective import packetize
    data, _, _, meta = load_golden(name)
    cb = meta["chunk_bytes"]
    first = data[(data["flags"] & 1) == 0]
    n_checked = 0
    keys = sorted({(int(s), int(d), int(q)) for s, d, q in zip(first["src"], first["dst"], first["msg_seq"])})
    for src, dst, seq in keys:
        pk = first[(first["src"] == src) & (first["dst"] == dst) & (first["msg_seq"] == seq)]
        length, tag, hdr0 = int(pk["msg_len"][0]), int(pk["msg_tag"][0]), int(pk["hdr"][0])
        nch = (length + cb - 1) // cb
        chunk = (pk["chunk_offset"] // cb).astype(np.int64)
        paths = np.zeros(nch, dtype=np.int32)
        paths[chunk] = pk["path_id"]
        out = packetize(length, cb, src=src, dst=dst, conn_id=hdr0 >> 24, msg_id=(hdr0 >> 17) & 0x7F,
                        msg_seq=seq, tag=tag, chunk_paths=torch.from_numpy(paths).cuda())
        r = _records(out)
        # packet counts: ceil(len_c / max_payload) per chunk (transport.cpp:277)
        lens = [min(cb, length - c * cb) for c in range(nch)]
        assert len(r) == sum((x + MAX_PL - 1) // MAX_PL for x in lens) == \
            _lib.lib().cn_packet_count(length, cb, MAX_PL)
        ppc = (cb + MAX_PL - 1) // MAX_PL
        idx = chunk * ppc + pk["seq_in_chunk"].astype(np.int64)
        for f in FIELDS:
            bad = np.nonzero(r[idx][f] != pk[f])[0]
            assert len(bad) == 0, (src, dst, seq, f, int(bad[0]), r[idx][bad[0]], pk[bad[0]])
        assert ((r["flags"] & 1) == 0).all()
        n_checked += len(pk)
    assert n_checked > 0
