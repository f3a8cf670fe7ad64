"""Record dtypes of the C ABI (include/chunknet_b200.h): cn_pkt_hdr,
cn_ack_rec, cn_completion -- numpy mirrors of the data/ack fields of
chunknet::Packet (/root/reference/proj/include/chunknet/packet.hpp:33-86).
"""
import numpy as np

PKT_DTYPE = np.dtype([
    ("src", "<i4"), ("dst", "<i4"), ("path_id", "<i4"), ("hdr", "<u4"),
    ("chunk_offset", "<u8"), ("chunk_len", "<u4"), ("payload_len", "<u2"),
    ("seq_in_chunk", "u1"), ("flags", "u1"), ("tx_time", "<i8"),
    ("msg_seq", "<u8"), ("msg_tag", "<u8"), ("msg_len", "<u8"),
])
assert PKT_DTYPE.itemsize == 64

ACK_DTYPE = np.dtype([
    ("src", "<i4"), ("dst", "<i4"), ("hdr", "<u4"), ("echo_path_id", "<i4"),
    ("cum_csn", "u1"), ("flags", "u1"), ("reserved", "<u2"), ("pkt_index", "<u4"),
    ("msg_seq", "<u8"), ("sack0", "<u8"), ("sack1", "<u8"),
    ("echo_tx_time", "<i8"), ("aux", "<i8"),
])
assert ACK_DTYPE.itemsize == 64

CPL_DTYPE = np.dtype([
    ("tag", "<u8"), ("src", "<i4"), ("dst", "<i4"), ("len", "<u8"),
    ("msg_seq", "<u8"), ("pkt_index", "<u4"), ("msg_id", "<u4"),
    ("buf_offset", "<u8"), ("bytes", "<u8"), ("reserved", "<u8"),
])
assert CPL_DTYPE.itemsize == 64

PKT_RTX, PKT_ECN, PKT_TRIMMED = 1, 2, 4
ACK_CUM_VALID, ACK_ECN_ECHO = 1, 2

# Fields of an ack record that the reference defines (aux is a recorder
# annotation, reserved is padding).
ACK_FIELDS = ["src", "dst", "hdr", "echo_path_id", "cum_csn", "flags",
              "pkt_index", "msg_seq", "sack0", "sack1", "echo_tx_time"]
CPL_FIELDS = ["tag", "src", "dst", "len", "pkt_index"]


def decode_hdr(w):
    """decode_header (src/wire.cpp:16-24), vectorised."""
    w = np.asarray(w, dtype=np.uint32)
    return dict(conn_id=(w >> 24) & 0xFF, msg_id=(w >> 17) & 0x7F,
                csn=(w >> 9) & 0xFF, last=(w >> 8) & 1, reserved=w & 0xFF)


def splitmix64(x):
    m = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & m
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & m
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & m
    return x ^ (x >> 31)


def ack_equal(a, b):
    """Field-wise comparison of two ACK_DTYPE arrays; returns (ok, first_bad)."""
    if len(a) != len(b):
        return False, f"len {len(a)} != {len(b)}"
    for f in ACK_FIELDS:
        bad = np.nonzero(a[f] != b[f])[0]
        if len(bad):
            i = int(bad[0])
            return False, f"ack {i} field {f}: {a[f][i]} != {b[f][i]}"
    return True, None
