"""Device sender engine (csrc/tx.cu) vs the reference sender: the same
submissions and timed acks replayed into the unmodified reference Transport
over a blackhole (golden tests/golden/sender_*.npz, oracle/gen_fixtures.py)
must produce the identical transmit log -- every (re)transmission, in
emission order, with its time, message, chunk, path and rtx flag -- and the
same Transport::Stats.  sender_<name>: congestion control none (OpenLoop);
sender_swift_<name>: Swift with global scope, target 3 x base RTT, the
window gating egress (DRR over the path ring, retransmission queues first).
The closed_* stimuli come from Swift DES runs, so there the replay is the
DES sender itself.  sender_rr_* / sender_single_*: the policy plug-ins
(include/chunknet_policy.cuh) against the same policies installed in the
reference with Transport::set_policy_factory."""
import glob
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu
NAMES = sorted(os.path.basename(p)[7:-4] for p in glob.glob(os.path.join(GOLDEN, "sender_*.npz")))


def _events(submits, acks):
    ev = [(int(s["t"]), 0, k) for k, s in enumerate(submits)] + \
         [(int(a["aux"]), 1, k) for k, a in enumerate(acks)]
    ev.sort(key=lambda x: (x[0], x[1], x[2]))  # DES: submits scheduled before acks
    return [(typ, k) for _, typ, k in ev]


@pytest.mark.parametrize("name", NAMES)
def test_tx_engine_matches_reference_sender(name):
    _replay(name, 1 << 18)


@pytest.mark.parametrize("name,pool", [("multigen_k8", 56), ("k8_4x1m", 68), ("swift_closed_w4", 350)])
def test_tx_engine_steady_state_chunk_ring(name, pool):
    """The connection's chunk entries form a ring that finished messages
    hand back (msg_finished, transport.cpp:831-847): a pool several times
    smaller than the scenario's total chunks (about the smallest that holds
    its live set; the ring's tail is the oldest live message) gives the
    identical transmit log."""
    z = np.load(os.path.join(GOLDEN, f"sender_{name}.npz"))
    cb = json.loads(bytes(z["meta"]).decode())["chunk_bytes"]
    assert sum((int(s["len"]) + cb - 1) // cb for s in z["submits"]) > pool
    _replay(name, pool)


def _replay(name, chunk_pool):
    from paper_2504_17307_b200.sender import TxEngine
    z = np.load(os.path.join(GOLDEN, f"sender_{name}.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    eng = TxEngine(1, chunk_bytes=meta["chunk_bytes"], rto_min=meta["rto_min"],
                   rto_max=meta["rto_max"], commit_ahead=meta["commit_ahead"],
                   base_rtt_ns=meta["base_rtt"], seed=meta["seed"], lb=meta["lb"],
                   max_paths=meta["n_paths"], src=[meta["src"]], dst=[meta["dst"]],
                   chunk_pool=chunk_pool, log_cap=1 << 17, cc=meta.get("cc", "none"),
                   swift_target_ns=meta.get("swift_target_ns", 0),
                   receiver_driven=meta.get("receiver_driven", False),
                   initial_credit=meta.get("initial_credit", 0), ordered=meta.get("ordered", False),
                   policy=meta.get("policy", 0))
    st = eng.run([_events(z["submits"], z["acks"])], z["submits"], z["acks"], 60_000_000_000)[0]
    ref = meta["stats"]
    for k in ("chunks_sent", "chunk_rtx", "fast_rtx", "rtos", "msgs_completed"):
        assert int(st[k]) == ref[k], (k, int(st[k]), ref[k])
    got, want = eng.log_np(0), z["tx"]
    assert len(got) == len(want)
    # data transmissions in emission order; receiver-driven RTS records
    # (chunk = 0xFFFFFFFF; the reference logs them at delivery) by time
    rts_g, rts_w = got["chunk"] == 0xFFFFFFFF, want["chunk"] == 0xFFFFFFFF
    assert rts_g.sum() == rts_w.sum()
    for sel_g, sel_w, srt in ((~rts_g, ~rts_w, False), (rts_g, rts_w, True)):
        g, w = got[sel_g], want[sel_w]
        if srt:
            g, w = g[np.argsort(g["t"], kind="stable")], w[np.argsort(w["t"], kind="stable")]
        for f in ("t", "msg_id", "chunk", "path", "is_rtx", "msg_seq"):
            bad = np.nonzero(g[f] != w[f])[0]
            assert len(bad) == 0, (srt, f, int(bad[0]), g[bad[0]], w[bad[0]])


def test_tx_engine_eight_dup_hints_one_fast_rtx():
    """test_transport.cpp:207-261 on the device: acks for chunks 1..7 leave
    chunk 0 alone; the 8th later-chunk ack retransmits it exactly once."""
    from paper_2504_17307_b200.records import ACK_DTYPE
    from paper_2504_17307_b200.sender import TxEngine
    eng = TxEngine(1, chunk_bytes=4032, rto_min=10_000_000, commit_ahead=1 << 20,
                   base_rtt_ns=12_000, seed=2, max_paths=1, src=[0], dst=[1])
    acks = np.zeros(9, dtype=ACK_DTYPE)
    for k, c in enumerate(range(1, 10)):
        a = acks[k]
        a["src"], a["dst"], a["msg_seq"], a["aux"] = 1, 0, 1, 10_000 * c
        a["hdr"] = (c << 9)
        a["sack0"] = 1 << c
        a["echo_tx_time"] = 999
    sub = np.array([(0, 10 * 4032, 1)], dtype=[("t", "<i8"), ("len", "<u8"), ("tag", "<u8")])
    st = eng.run([[(0, 0)] + [(1, k) for k in range(9)]], sub, acks, 200_000)[0]
    assert int(st["fast_rtx"]) == 1 and int(st["chunk_rtx"]) == 1 and int(st["chunks_sent"]) == 10
    log = eng.log_np(0)
    assert [int(r["chunk"]) for r in log if r["is_rtx"]] == [0]


def test_tx_policy_contract_violation_fails_loudly():
    """test_transport.cpp:686-703: a policy path outside [0, n_paths) is a
    logic_error; the engine reports CN_E_LOGIC."""
    from paper_2504_17307_b200._lib import ChunknetError
    from paper_2504_17307_b200.records import ACK_DTYPE
    from paper_2504_17307_b200.sender import TxEngine
    eng = TxEngine(1, chunk_bytes=4032, rto_min=10_000_000, commit_ahead=1 << 20, base_rtt_ns=12_000,
                   seed=2, max_paths=4, n_paths=[4], src=[0], dst=[1], policy="test_out_of_range")
    sub = np.array([(0, 4096, 1)], dtype=[("t", "<i8"), ("len", "<u8"), ("tag", "<u8")])
    with pytest.raises(ChunknetError) as e:
        eng.run([[(0, 0)]], sub, np.zeros(1, dtype=ACK_DTYPE), 100_000)
    assert e.value.status == -2


@pytest.mark.parametrize("name,nslice", [("swift_multigen_k8", 42), ("multigen_k8", 42), ("lossy_2m", 7),
                                         ("swift_closed_w4", 25)])
def test_tx_engine_resumes_across_runs(name, nslice):
    """The input events handed over in time slices, one cn_tx_run each (how
    the endpoint drives the engine): the state persisted between launches
    gives the identical transmit log."""
    from paper_2504_17307_b200.sender import TxEngine
    z = np.load(os.path.join(GOLDEN, f"sender_{name}.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    eng = TxEngine(1, chunk_bytes=meta["chunk_bytes"], rto_min=meta["rto_min"], rto_max=meta["rto_max"],
                   commit_ahead=meta["commit_ahead"], base_rtt_ns=meta["base_rtt"], seed=meta["seed"],
                   lb=meta["lb"], max_paths=meta["n_paths"], src=[meta["src"]], dst=[meta["dst"]],
                   chunk_pool=1 << 18, log_cap=1 << 17, cc=meta.get("cc", "none"),
                   swift_target_ns=meta.get("swift_target_ns", 0))
    subs, acks = z["submits"], z["acks"]
    ev = sorted([(int(s["t"]), 0, k) for k, s in enumerate(subs)] + [(int(a["aux"]), 1, k) for k, a in enumerate(acks)])
    ts = sorted({e[0] for e in ev})
    cuts = [ts[int(len(ts) * (i + 1) / nslice) - 1] for i in range(nslice)]
    cuts[-1] = 60_000_000_000
    k = 0
    for c in cuts:
        part = []
        while k < len(ev) and ev[k][0] <= c:
            part.append(ev[k])
            k += 1
        si = [e[2] for e in part if e[1] == 0]
        ai = [e[2] for e in part if e[1] == 1]
        ms, ma = {j: i for i, j in enumerate(si)}, {j: i for i, j in enumerate(ai)}
        evs = [(0, ms[e[2]]) if e[1] == 0 else (1, ma[e[2]]) for e in part]
        eng.run([evs], subs[si] if si else subs[:1], acks[ai] if ai else acks[:1], c)
    got, want = eng.log_np(0), z["tx"]
    assert len(got) == len(want)
    for f in ("t", "msg_id", "chunk", "path", "is_rtx", "msg_seq"):
        assert (got[f] == want[f]).all(), f
