"""Trace format (experiment.cpp:18-40 trace_line): the device writer
(csrc/trace.cu) renders records byte-identically to the reference's
trace.tsv (golden tests/golden/trace.npz from the reference's own
run_experiment, oracle/gen_fixtures.py)."""
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2504_17307_b200.trace import EVENTS, FLAGS, KINDS, TRACE_DTYPE, parse_tsv


def render(recs):
    """trace_line restated in Python (test checker)."""
    out = []
    for r in recs:
        line = (f"{int(r['t'])}\t{EVENTS[r['event']]}\t{int(r['link_id'])}\t{int(r['src'])}>{int(r['dst'])}:"
                f"{int(r['path_id'])}\t{int(r['csn'])}\t{KINDS[r['kind']]}")
        for name, bit in FLAGS:
            if r["flags"] & bit:
                line += "," + name
        out.append(line + "\n")
    return "".join(out).encode()


def goldens():
    z = np.load(os.path.join(GOLDEN, "trace.npz"))
    return {k[4:]: bytes(z[k]) for k in z.files if k.startswith("tsv_")}


def test_trace_golden_roundtrip_cpu():
    g = goldens()
    assert {"trim_incast", "eqds_incast", "fat_tree_loss", "ordered_loss"} <= set(g)
    seen_kinds, seen_events = set(), set()
    for name, text in g.items():
        recs = parse_tsv(text)
        assert render(recs) == text, name
        seen_kinds |= {KINDS[k] for k in recs["kind"]}
        seen_events |= {EVENTS[e] for e in recs["event"]}
    assert seen_kinds == set(KINDS)
    assert {"deliver", "drop", "trim", "loss"} <= seen_events


@pytest.mark.gpu
def test_trace_device_writer_matches_reference():
    from paper_2504_17307_b200.trace import format_tsv
    for name, text in goldens().items():
        assert format_tsv(parse_tsv(text)) == text, name


@pytest.mark.gpu
def test_trace_device_writer_extremes():
    from paper_2504_17307_b200.trace import format_tsv
    rs = np.random.RandomState(7)
    n = 20000
    r = np.zeros(n, dtype=TRACE_DTYPE)
    r["t"] = rs.randint(-2**62, 2**62, size=n, dtype=np.int64)
    r["t"][:4] = [0, -1, np.iinfo(np.int64).max, np.iinfo(np.int64).min]
    r["link_id"] = rs.randint(-2**31, 2**31 - 1, size=n)
    r["src"] = rs.randint(0, 1 << 24, size=n)
    r["dst"] = rs.randint(0, 1 << 24, size=n)
    r["path_id"] = rs.randint(0, 1024, size=n)
    r["csn"] = rs.randint(0, 256, size=n)
    r["event"] = rs.randint(0, 5, size=n)
    r["kind"] = rs.randint(0, 6, size=n)
    r["flags"] = rs.randint(0, 16, size=n)
    assert format_tsv(r) == render(r)
    assert format_tsv(r[:0]) == b""


@pytest.mark.gpu
def test_trace_from_receive_records():
    import torch

    from paper_2504_17307_b200.records import ACK_DTYPE, PKT_DTYPE
    from paper_2504_17307_b200.trace import format_tsv, from_acks, from_packets
    z = np.load(os.path.join(GOLDEN, "sender_cfg1.npz"))
    acks = np.ascontiguousarray(z["acks"], dtype=ACK_DTYPE)
    d = torch.from_numpy(acks.view(np.uint8).reshape(-1)).cuda()
    got = format_tsv(from_acks(d))
    want = np.zeros(len(acks), dtype=TRACE_DTYPE)
    want["t"], want["src"], want["dst"] = acks["aux"], acks["src"], acks["dst"]
    want["link_id"], want["kind"] = -1, KINDS.index("ack")
    want["csn"] = (acks["hdr"] >> 9) & 0xFF
    assert got == render(want)
    zc = np.load(os.path.join(GOLDEN, "cfg1.npz"))
    pk = np.ascontiguousarray(zc["data"], dtype=PKT_DTYPE)
    dp = torch.from_numpy(pk.view(np.uint8).reshape(-1)).cuda()
    times = torch.arange(len(pk), dtype=torch.int64, device="cuda") * 100
    got = format_tsv(from_packets(dp, times))
    want = np.zeros(len(pk), dtype=TRACE_DTYPE)
    want["t"] = np.arange(len(pk)) * 100
    want["link_id"], want["src"], want["dst"], want["path_id"] = -1, pk["src"], pk["dst"], pk["path_id"]
    want["csn"] = (pk["hdr"] >> 9) & 0xFF
    want["flags"] = ((pk["flags"] & 1) != 0) * 1 + ((pk["flags"] & 2) != 0) * 2 + \
        ((pk["flags"] & 4) != 0) * 4 + ((pk["hdr"] >> 8) & 1) * 8
    assert got == render(want)
