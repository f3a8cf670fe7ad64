"""The unified boundary object (cn_transport_*, TransportEndpoint) driven
like chunknet::Transport: the recorded sender scenarios through
send_message / handle_acks / advance give the reference transmit log, and
a multi-connection trim incast through one object gives every connection's
log; the receive side of the same object gives the reference ack stream."""
import glob
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden
from oracle.records import ack_equal

pytestmark = pytest.mark.gpu


def _ep(meta, n_conns=4, **kw):
    from paper_2504_17307_b200.endpoint import TransportEndpoint
    return TransportEndpoint(chunk_bytes=meta["chunk_bytes"], paths=meta["n_paths"], lb=meta["lb"],
                             rto_min=meta["rto_min"], rto_max=meta["rto_max"], commit_ahead=meta["commit_ahead"],
                             base_rtt_ns=meta["base_rtt"], seed=meta["seed"], cc=meta.get("cc", "none"),
                             swift_target_ns=meta.get("swift_target_ns", 0), max_conns=n_conns,
                             chunk_pool=1 << 18, log_cap=1 << 17, **kw)


@pytest.mark.parametrize("name", ["cfg1", "lossy_2m", "swift_closed_k8", "swift_cfg1"])
def test_endpoint_sender_replay(name):
    z = np.load(os.path.join(GOLDEN, f"sender_{name}.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    ep = _ep(meta)
    for s in z["submits"]:
        ep.send_message(meta["src"], meta["dst"], int(s["len"]), int(s["tag"]), int(s["t"]))
    ep.handle_acks(z["acks"])
    ep.advance(60_000_000_000)
    tx, conn = ep.poll_transmissions()
    want = z["tx"]
    assert len(tx) == len(want) and (conn == 0).all()
    for f in ("t", "msg_id", "chunk", "path", "is_rtx", "msg_seq"):
        assert (tx[f] == want[f]).all(), f
    st = ep.stats()
    for k in ("chunks_sent", "chunk_rtx", "fast_rtx", "rtos"):
        assert st[k] == meta["stats"][k], k


def test_endpoint_multi_connection_and_receive():
    names = sorted(glob.glob(os.path.join(GOLDEN, "sender_swift_trim_swift_f*.npz")))
    assert len(names) == 4
    zs = [np.load(p) for p in names]
    metas = [json.loads(bytes(z["meta"]).decode()) for z in zs]
    ep = _ep(metas[0])
    for z, m in zip(zs, metas):  # connections open in flow order (conn_to)
        for s in z["submits"]:
            ep.send_message(m["src"], m["dst"], int(s["len"]), int(s["tag"]), int(s["t"]))
    ep.handle_acks(np.concatenate([z["acks"] for z in zs]))
    # advance in two slices: state carries over
    ep.advance(2_000_000)
    tx1, c1 = ep.poll_transmissions()
    ep.advance(60_000_000_000)
    tx2, c2 = ep.poll_transmissions()
    tx, conn = np.concatenate([tx1, tx2]), np.concatenate([c1, c2])
    for k, (z, m) in enumerate(zip(zs, metas)):
        assert ep.conn_index(m["src"], m["dst"]) == k
        got = tx[conn == k]
        got = got[np.argsort(got["t"], kind="stable")]
        want = z["tx"]
        assert len(got) == len(want), k
        for f in ("t", "msg_id", "chunk", "path", "is_rtx", "msg_seq"):
            assert (got[f] == want[f]).all(), (k, f)
    # receive side of the same object: the trim incast's delivered packets
    import paper_2504_17307_b200 as cn
    from oracle import oracle as O
    data, acks_ref, cpls_ref, meta = load_golden("trim_swift")
    import torch
    ep.handle_data(cn.to_device_records(data), torch.from_numpy(O.fill_staging(data)).cuda())
    ok, bad = ack_equal(ep.poll_acks(), acks_ref)
    assert ok, bad
    assert len(ep.poll_completions()) == len(cpls_ref)
    st = ep.stats()
    assert st["nacks_sent"] == int(((acks_ref["flags"] & 4) != 0).sum())
    assert st["delivered_msgs"] == len(cpls_ref)


@pytest.mark.parametrize("name", ["lossy_2m", "multigen_k8", "closed_w4", "k8_4x1m"])
def test_endpoint_introspection_matches_reference(name):
    """path_inflight / window_available / outstanding_bytes / conn_credit /
    engine_* (transport.cpp:1173-1209) at times between the scenario's input
    events, the inputs handed over in time slices: the reference's values
    (oracle/gen_fixtures.py probe_<name>.npz)."""
    zp = np.load(os.path.join(GOLDEN, f"probe_{name}.npz"))
    sname = bytes(zp["sender"]).decode()
    z = np.load(os.path.join(GOLDEN, f"{sname}.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    ep = _ep(meta)
    src, dst, n = meta["src"], meta["dst"], meta["n_paths"]
    subs, acks = z["submits"], z["acks"]
    si = ai = 0
    for t, want in zip(zp["probe_t"], zp["probes"]):
        t = int(t)
        while si < len(subs) and int(subs[si]["t"]) <= t:
            ep.send_message(src, dst, int(subs[si]["len"]), int(subs[si]["tag"]), int(subs[si]["t"]))
            si += 1
        aj = ai
        while aj < len(acks) and int(acks[aj]["aux"]) <= t:
            aj += 1
        if aj > ai:
            ep.handle_acks(acks[ai:aj])
            ai = aj
        ep.advance(t)
        got = [ep.outstanding_bytes(src, dst), ep.conn_credit(src, dst), ep.engine_inflight_msgs(src),
               ep.engine_dispatched(src), ep.engine_gauge(src)]
        for p in range(n):
            got += [ep.path_inflight(src, dst, p), ep.window_available(src, dst, p)]
        assert got == [int(v) for v in want], (t, got, list(want))


@pytest.mark.parametrize("flow", range(5))
def test_endpoint_receiver_driven_replay(flow):
    """Receiver-driven mode through the boundary object: the recorded
    credits and rts_acks (EQDS incast, one connection each) give the
    reference's transmissions and RTS packets."""
    z = np.load(os.path.join(GOLDEN, f"sender_eqds_incast_f{flow}.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    ep = _ep(meta, receiver_driven=True, initial_credit=meta["initial_credit"])
    for s in z["submits"]:
        ep.send_message(meta["src"], meta["dst"], int(s["len"]), int(s["tag"]), int(s["t"]))
    ep.handle_acks(z["acks"])
    ep.advance(60_000_000_000)
    tx, conn = ep.poll_transmissions()
    want = z["tx"]
    assert len(tx) == len(want)
    rg, rw = tx["chunk"] == 0xFFFFFFFF, want["chunk"] == 0xFFFFFFFF
    assert rg.sum() == rw.sum()
    for sg, sw, srt in ((~rg, ~rw, False), (rg, rw, True)):
        g, w = tx[sg], want[sw]
        if srt:
            g, w = g[np.argsort(g["t"], kind="stable")], w[np.argsort(w["t"], kind="stable")]
        for f in ("t", "msg_id", "chunk", "path", "is_rtx", "msg_seq"):
            assert (g[f] == w[f]).all(), (srt, f)


@pytest.mark.parametrize("name", ["ordered_loss_f0", "swift_ordered_trim_f0", "swift_ordered_trim_f1"])
def test_endpoint_ordered_sender_replay(name):
    """Ordered reliability (go-back-N) through the boundary object: the
    sequence-gap NACKs in the recorded acks drive the rewinds."""
    z = np.load(os.path.join(GOLDEN, f"sender_{name}.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    ep = _ep(meta, reliability="ordered")
    for s in z["submits"]:
        ep.send_message(meta["src"], meta["dst"], int(s["len"]), int(s["tag"]), int(s["t"]))
    ep.handle_acks(z["acks"])
    ep.advance(60_000_000_000)
    tx, _ = ep.poll_transmissions()
    want = z["tx"]
    assert len(tx) == len(want)
    for f in ("t", "msg_id", "chunk", "path", "is_rtx", "msg_seq"):
        assert (tx[f] == want[f]).all(), f


@pytest.mark.parametrize("name", ["ordered_loss", "ordered_trim"])
def test_endpoint_ordered_receive(name):
    import torch

    import paper_2504_17307_b200 as cn
    from conftest import load_psn
    from oracle import oracle as O
    data, acks_ref, cpls_ref, meta = load_golden(name)
    ep = _ep({"chunk_bytes": meta["chunk_bytes"], "n_paths": 1, "lb": "oblivious", "rto_min": 100000,
              "rto_max": 0, "commit_ahead": 65536, "base_rtt": 10000, "seed": 1}, reliability="ordered")
    psn = torch.from_numpy(load_psn(name).astype(np.int64)).cuda()
    ep.handle_data(cn.to_device_records(data), torch.from_numpy(O.fill_staging(data)).cuda(), psn=psn)
    ok, bad = ack_equal(ep.poll_acks(), acks_ref)
    assert ok, bad
    assert len(ep.poll_completions()) == len(cpls_ref)


@pytest.mark.parametrize("name", ["fanout_k8_cubic", "fanout_k8_e4split", "fanout_pp_cubic_pp",
                                  "split_swift_swift_e2split", "fanout_rd_none", "engines_k8_cubic_e4"])
def test_endpoint_host_replay(name):
    """A source host with several connections through the boundary object:
    fan-out, engines / conn_split, CUBIC and per-path scope, receiver-driven
    -- the reference host's transmit log (host_<name>.npz) and the engine
    introspection after the run."""
    from test_host_gpu import compare, load
    z, meta = load(name)
    src = meta["src"]
    ep = _ep(dict(meta, n_paths=max(meta["n_paths"])), n_conns=8, engines=meta["engines"],
             conn_split=meta["conn_split"], cc_scope=["global", "per_path"][meta["cc_scope"]],
             receiver_driven=meta["receiver_driven"],
             initial_credit=meta["initial_credit"] if meta["receiver_driven"] else -1, policy=meta["policy"])
    for k, (dst, np_) in enumerate(zip(meta["conns"], meta["n_paths"])):  # conn_to order
        assert ep.open_conn(src, dst, np_) == k
    for s in z["submits"]:
        ep.send_message(src, int(s["dst"]), int(s["len"]), int(s["tag"]), int(s["t"]))
    ep.handle_acks(z["acks"])
    half = int(meta["end_time"]) // 2
    ep.advance(half)
    tx1, _ = ep.poll_transmissions()
    ep.advance(meta["end_time"])
    tx2, _ = ep.poll_transmissions(cap=7)  # a small cap: the rest stays queued
    tx3, _ = ep.poll_transmissions()
    tx = np.concatenate([tx1, tx2, tx3])
    st = ep.stats()

    class S(dict):
        def __getitem__(self, k):
            return np.array([dict.__getitem__(self, k)])
    compare(tx, z["tx"], meta, S(st))
    done = sum(ep.engine_dispatched(src, e) for e in range(meta["engines"]))
    assert done == len(z["submits"]) - st["backpressured"]
