"""Randomized parity at scale: the reference's own property suite
(test_reliability_props.cpp:126-218 -- star / fat tree, 10 or 100 Gb/s,
0-1.6% loss, chunk sizes, 1-8 paths, engines and conn_split, oblivious /
P2 load balancing, CC none / CUBIC / Swift in global or per-path scope,
receiver-driven and ordered seeds, runt and 1-byte messages), 256 seeds
drawn with its RngStream by oracle/ref_harness.cpp and recorded in the
reference DES (tests/golden/props/, oracle/gen_fixtures.py gen_props), plus
trim-mode seeds (seed % 10 == 5, the builder's extension) and the
engine-invariance case (:328-358, engines 1 / 2 / 4).

Per seed, on the device:
* the receive path on the delivered packets: the reference's ack / NACK
  stream, completions and byte-identical message buffers;
* the sender of every source host (its connections, engines, CC) on that
  host's submissions and delivered acks: the reference's transmit log."""
import glob
import json
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from oracle import oracle as O
from oracle.records import ack_equal

pytestmark = pytest.mark.gpu
PROPS = sorted(glob.glob(os.path.join(GOLDEN, "props", "*.npz")))
NAMES = [os.path.basename(p)[:-4] for p in PROPS]


def load(name):
    z = np.load(os.path.join(GOLDEN, "props", f"{name}.npz"))
    return z, json.loads(bytes(z["meta"]).decode())


def rx_check(z, meta):
    import paper_2504_17307_b200 as cn
    ordered = meta["record"]["ordered"]
    data, acks_ref, cpls_ref = z["data"], z["acks"], z["completions"]
    tr = cn.Transport(cn.TransportConfig(chunk_bytes=meta["chunk_bytes"], carry_payload=True,
                                         reliability="ordered" if ordered else "selective"),
                      arena_bytes=32 << 20, max_batch=1 << 15, chunk_pool=1 << 16, max_conns=256, max_msgs=256)
    staging = O.fill_staging(data)
    psn = torch.from_numpy(z["psn"].astype(np.int64)).cuda() if ordered else None
    out = tr.handle_packets(cn.to_device_records(data), torch.from_numpy(staging).cuda(), psn=psn)
    ok, bad = ack_equal(out.acks_np(), acks_ref)
    assert ok, bad
    got = out.completions_np()
    assert len(got) == len(cpls_ref) == len(meta["flows"])
    for f in ("tag", "src", "dst", "len"):
        assert (got[f] == cpls_ref[f]).all(), f
    arena = tr.arena()
    for c in got:
        buf = arena[int(c["buf_offset"]): int(c["buf_offset"]) + int(c["len"])].cpu().numpy()
        assert (buf == O.pattern_bytes(int(c["len"]), int(c["tag"]))).all(), int(c["tag"])
    tr.close()
    return sorted((int(c["tag"]), int(c["len"])) for c in got)


def tx_check(z, meta):
    from test_host_gpu import compare
    from paper_2504_17307_b200.sender import SUBMIT_DTYPE, TxEngine
    r = meta["record"]
    for hm in meta["hosts"]:
        h = hm["src"]
        subs_h, acks, want = z[f"h{h}_submits"], z[f"h{h}_acks"], z[f"h{h}_tx"]
        conns = hm["conns"]
        k_of = {d: k for k, d in enumerate(conns)}
        subs = np.zeros(len(subs_h), dtype=SUBMIT_DTYPE)
        for f in ("t", "len", "tag"):
            subs[f] = subs_h[f]
        ev = [(int(s["t"]), 0, k_of[int(s["dst"])], j) for j, s in enumerate(subs_h)]
        ev += [(int(a["aux"]), 1, k_of.get(int(a["src"]), 0), j) for j, a in enumerate(acks)]
        ev.sort(key=lambda e: (e[0], e[1], e[3]))
        eng = TxEngine(len(conns), chunk_bytes=r["chunk_bytes"], rto_min=hm["rto_min"], rto_max=hm["rto_max"],
                       commit_ahead=hm["commit_ahead"], base_rtt_ns=hm["base_rtt"], seed=meta["seed"], lb=r["lb"],
                       max_paths=max(hm["n_paths"]), n_paths=hm["n_paths"], src=[h] * len(conns), dst=conns,
                       chunk_pool=1 << 16, log_cap=1 << 16, cc=r["cc"],
                       cc_scope=["global", "per_path"][r["cc_scope"]], swift_target_ns=hm["swift_target_ns"],
                       receiver_driven=r["receiver_driven"],
                       initial_credit=hm["initial_credit"] if r["receiver_driven"] else 0, ordered=r["ordered"],
                       engines=r["engines"], conn_split=bool(r["conn_split"]))
        st = eng.run([(t, k, j) for _, t, k, j in ev], subs, acks, hm["end_time"])
        compare(eng.log_np(0), want, dict(meta, stats=hm["stats"]), st)
        eng.close()


@pytest.mark.parametrize("name", [n for n in NAMES if n.startswith("prop_")])
def test_property_scenario_matches_reference(name):
    z, meta = load(name)
    rx_check(z, meta)
    tx_check(z, meta)


@pytest.mark.parametrize("seed", range(12))
def test_delivered_bytes_invariant_to_engine_count(seed):
    """test_reliability_props.cpp:328-390 on the device: the same six
    messages under engines 1, 2, 4 (conn_split) -- each run's receive path
    and senders match the reference, and every engine count delivers the
    same messages with the source bytes."""
    sets = []
    for e in (1, 2, 4):
        z, meta = load(f"enginv_{seed}_e{e}")
        sets.append(rx_check(z, meta))
        tx_check(z, meta)
    assert sets[0] == sets[1] == sets[2]
