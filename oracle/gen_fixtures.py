"""Generates tests/golden/*.npz from the UNMODIFIED reference -- TEST INFRA.

Run where /root/reference is mounted, after `make -C oracle ref`:

    python -m oracle.gen_fixtures

For every scenario the reference discrete-event simulator
(Network + Transport, src/network.cpp, src/transport.cpp) is run with
carry_payload and pattern payloads (test_transport.cpp:63-71, seed = tag);
the data packets delivered at their destinations are recorded in arrival
order, then replayed into a fresh reference Transport's receive path
(Transport::handle_packet, transport.cpp:565) to capture the exact ack
stream (emission order, causing packet index) and the completions.  The
script asserts that (a) every DES completion was byte-identical to its
source, and (b) for single-connection scenarios the replay ack stream equals
the ack stream the DES delivered to the sender (replay purity, SURVEY.md
Appendix B).
"""
import json
import os
import sys

import numpy as np

from . import ref
from .records import ACK_FIELDS, ack_equal

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")

MiB = 1 << 20

# name -> (record kwargs, flows)
SCENARIOS = {
    # BASELINE.json configs[0]: 1 MiB, 4 KiB chunks, 8 paths, no loss
    "cfg1": (dict(topo="fat_tree", topo_arg=8, rate_bps=400e9, qcap_bytes=MiB,
                  loss=0.0, seed=1, chunk_bytes=4096, paths=8, lb="p2_rtt",
                  cc="cubic"), [(0, 127, MiB, 1)]),
    # BASELINE.json configs[1]: 64 MiB, 256 paths, 1% drop (32 KiB / 4 KiB chunks)
    "cfg2_32k": (dict(topo="fat_tree", topo_arg=32, rate_bps=400e9, qcap_bytes=MiB,
                      loss=0.01, seed=1, chunk_bytes=32768, paths=256, lb="p2_rtt",
                      cc="cubic"), [(0, 8191, 64 * MiB, 1)]),
    "cfg2_4k": (dict(topo="fat_tree", topo_arg=32, rate_bps=400e9, qcap_bytes=MiB,
                     loss=0.01, seed=1, chunk_bytes=4096, paths=256, lb="p2_rtt",
                     cc="cubic"), [(0, 8191, 64 * MiB, 1)]),
    # reference test "csn wrap-around: 600 chunks reassemble under loss"
    # (test_transport.cpp:330-357)
    "csn_wrap": (dict(topo="star", topo_arg=2, rate_bps=10e9, qcap_bytes=MiB,
                      loss=0.01, seed=5, chunk_bytes=4032, paths=1, lb="oblivious",
                      cc="cubic"), [(0, 1, 600 * 4032, 1)]),
    # reference test "lossy link: retransmission delivers byte-identical data"
    "lossy_2m": (dict(topo="star", topo_arg=2, rate_bps=10e9, qcap_bytes=MiB,
                      loss=0.02, seed=4, chunk_bytes=32768, paths=1, lb="oblivious",
                      cc="cubic"), [(0, 1, 2 * MiB, 1)]),
    # reference test "multipath spray with loss keeps payload integrity"
    "multipath_k4": (dict(topo="fat_tree", topo_arg=4, rate_bps=10e9, qcap_bytes=MiB,
                          loss=0.01, seed=6, chunk_bytes=16128, paths=4, lb="p2_rtt",
                          cc="cubic"), [(0, 12, MiB, 1), (5, 12, MiB, 1)]),
    # many generations per connection, msg-id reuse, 3% loss
    "multigen_k8": (dict(topo="fat_tree", topo_arg=8, rate_bps=100e9, qcap_bytes=MiB,
                         loss=0.03, seed=11, chunk_bytes=4032, paths=16, lb="p2_ecn",
                         cc="none"), [(0, 127, 64 * 1024, 32)]),
    # concurrent messages on one connection + several connections into one host
    "concurrent_k4": (dict(topo="fat_tree", topo_arg=4, rate_bps=100e9, qcap_bytes=MiB,
                           loss=0.01, seed=12, chunk_bytes=8064, paths=4, lb="p2_rtt",
                           cc="swift", window=4),
                      [(0, 12, 300_000, 6), (5, 12, 123_457, 6), (13, 2, 1, 3),
                       (7, 3, 4031, 4), (8, 3, 4033, 4)]),
    # chunk size not a multiple of 16: unaligned scatter, runt packets
    "odd_chunk": (dict(topo="star", topo_arg=6, rate_bps=100e9, qcap_bytes=MiB,
                       loss=0.02, seed=13, chunk_bytes=5000, paths=1, lb="oblivious",
                       cc="cubic", window=2),
                  [(0, 1, 77_777, 3), (2, 1, 5000, 2), (3, 4, 12_345, 3),
                   (5, 4, 7, 2)]),
    # 4 x 1 MiB, 16 paths, 1% (survey Appendix B item 10)
    "k8_4x1m": (dict(topo="fat_tree", topo_arg=8, rate_bps=400e9, qcap_bytes=MiB,
                     loss=0.01, seed=3, chunk_bytes=32768, paths=16, lb="p2_rtt",
                     cc="cubic"), [(0, 127, MiB, 4)]),
    # trim queue mode (NDP-style header trimming): incast of 4 senders into a
    # 96 KiB trimming queue; trimmed headers -> NACKs (transport.cpp:657-674)
    "trim_swift": (dict(topo="star", topo_arg=5, rate_bps=100e9, qcap_bytes=96 * 1024,
                        loss=0.0, seed=9, chunk_bytes=16384, paths=1, lb="oblivious",
                        cc="swift", queue="trim", trim_depth=4, window=2),
                   [(1, 0, MiB, 2), (2, 0, MiB, 2), (3, 0, MiB, 2), (4, 0, MiB, 2)]),
    # the same with an open window: 10,401 of 18,894 deliveries are trimmed
    "trim_storm": (dict(topo="star", topo_arg=5, rate_bps=100e9, qcap_bytes=96 * 1024,
                        loss=0.0, seed=9, chunk_bytes=16384, paths=1, lb="oblivious",
                        cc="none", queue="trim", trim_depth=4, window=2),
                   [(1, 0, MiB, 2), (2, 0, MiB, 2), (3, 0, MiB, 2), (4, 0, MiB, 2)]),
    # receiver-driven (EQDS) incast: 5 senders into one host, credit-gated
    "eqds_incast": (dict(topo="star", topo_arg=6, rate_bps=100e9, qcap_bytes=128 * 1024,
                         loss=0.0, seed=5, chunk_bytes=32768, paths=1, lb="oblivious",
                         cc="none", receiver_driven=True, window=2),
                    [(1, 0, MiB, 2), (2, 0, MiB, 2), (3, 0, MiB, 2), (4, 0, MiB, 2), (5, 0, MiB, 2)]),
    # the same with 1% loss: retransmissions owed while credit-gated
    "eqds_lossy": (dict(topo="star", topo_arg=6, rate_bps=100e9, qcap_bytes=128 * 1024,
                        loss=0.01, seed=6, chunk_bytes=16384, paths=1, lb="oblivious",
                        cc="swift", receiver_driven=True, window=2),
                   [(1, 0, MiB, 3), (2, 0, MiB, 3), (3, 0, MiB, 3), (4, 0, MiB, 3)]),
    # ordered reliability (go-back-N, transport.cpp:690-717, 966-999): one
    # lossy connection, and a trimming incast (head-of-line trims)
    "ordered_loss": (dict(topo="star", topo_arg=2, rate_bps=10e9, qcap_bytes=MiB, loss=0.02,
                          seed=4, chunk_bytes=32768, paths=1, lb="oblivious", cc="none",
                          ordered=True), [(0, 1, 2 * MiB, 1)]),
    "ordered_trim": (dict(topo="star", topo_arg=4, rate_bps=100e9, qcap_bytes=64 * 1024, loss=0.0,
                          seed=9, chunk_bytes=16384, paths=1, lb="oblivious", cc="swift",
                          ordered=True, queue="trim", trim_depth=4, window=2),
                     [(1, 0, MiB, 2), (2, 0, MiB, 2), (3, 0, MiB, 2)]),
    # closed loop under Swift: the DES sender runs Swift (target 3 x base
    # RTT), so its recorded acks answer exactly what a Swift sender sends
    "closed_k8": (dict(topo="fat_tree", topo_arg=8, rate_bps=400e9, qcap_bytes=MiB,
                       loss=0.01, seed=7, chunk_bytes=32768, paths=16, lb="p2_rtt",
                       cc="swift"), [(0, 127, MiB, 4)]),
    "closed_w4": (dict(topo="fat_tree", topo_arg=8, rate_bps=100e9, qcap_bytes=MiB,
                       loss=0.03, seed=8, chunk_bytes=8064, paths=16, lb="p2_ecn",
                       cc="swift", window=4), [(0, 127, 300_000, 12)]),
    "closed_cfg2": (dict(topo="fat_tree", topo_arg=32, rate_bps=400e9, qcap_bytes=MiB,
                         loss=0.01, seed=1, chunk_bytes=32768, paths=256, lb="p2_rtt",
                         cc="swift"), [(0, 8191, 64 * MiB, 1)]),
}


def gen(name, kw, flows):
    kw = dict(kw)
    window = kw.pop("window", 1)
    tmp = f"/tmp/cnfix_{name}"
    data, acks_des, cpl_des, st = ref.record(tmp, flows=flows, window=window, **kw)
    assert st["quiesced"] == 1, (name, st)
    assert st["bytes_ok"] == st["completions"], (name, st)
    psn = st.pop("psn")
    ordered = bool(kw.get("ordered", False))
    acks, cpls, arena = ref.rx_replay(data, st["n_hosts"], kw["chunk_bytes"], psn=psn if ordered else None,
                                      ordered=ordered)
    assert len(cpls) == st["completions"], (name, len(cpls), st)
    conns = {(int(s), int(d)) for s, d in zip(data["src"], data["dst"])}
    if len(conns) == 1:
        a2 = acks_des.copy()
        a2["pkt_index"] = acks["pkt_index"]
        ok, bad = ack_equal(acks, a2)
        assert ok, (name, bad)
    subs = st.pop("submits")
    meta = dict(name=name, n_hosts=int(st["n_hosts"]), chunk_bytes=int(kw["chunk_bytes"]),
                record=dict(kw, window=window), flows=flows,
                des_stats={k: int(v) for k, v in st.items()})
    if name in SENDER_SCENARIOS:
        gen_sender(name, kw, flows, acks_des, subs)
    if name in CLOSED_SWIFT:
        gen_sender(name, kw, flows, acks_des, subs, cc="swift")
    if name in TRIM_SENDER:
        for f in range(len(flows)):
            gen_sender(name, kw, flows, acks_des, subs, cc=kw["cc"], flow=f)
    path = os.path.join(GOLDEN, f"{name}.npz")
    extra = {"psn": psn} if ordered else {}
    np.savez_compressed(path, data=data, acks=acks, completions=cpls,
                        meta=np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8), **extra)
    print(f"{name}: pkts={len(data)} acks={len(acks)} completions={len(cpls)} "
          f"rtx={st['chunk_rtx']} fast_rtx={st['fast_rtx']} rtos={st['rtos']} "
          f"-> {os.path.getsize(path)} B")


# single-connection scenarios whose timed acks are replayed into the
# reference sender (blackhole, CC none) for the tx-engine goldens
SENDER_SCENARIOS = ["cfg1", "cfg2_32k", "cfg2_4k", "k8_4x1m", "multigen_k8", "lossy_2m",
                    "csn_wrap"]


POLICY_NAMES = {1: "rr", 2: "single", 3: "user"}  # harness ids (install_policy, ref_harness.cpp)
POLICY_ENGINE_ID = {0: 0, 1: 1, 2: 2, 3: 100}     # cn_tx_config::policy (CN_POLICY_*)


def gen_sender(name, kw, flows, acks_des, subs, cc="none", flow=None, policy=0):
    """Sender-side golden: the reference sender (OpenLoop, or Swift with
    global scope) fed the DES's submissions and the acks (and NACKs) the DES
    delivered to it, at their times.  flow: one connection of a multi-flow
    scenario (its own submissions and acks; connections are independent)."""
    src, dst = flows[flow or 0][0], flows[flow or 0][1]
    if flow is not None:
        acks_des = acks_des[(acks_des["dst"] == src) & (acks_des["src"] == dst)]
        subs = subs[(subs["src"] == src) & (subs["dst"] == dst)]
        name = f"{name}_f{flow}"
    rkw = {k: kw[k] for k in ("topo", "topo_arg", "rate_bps", "qcap_bytes", "seed", "chunk_bytes",
                              "paths", "lb", "receiver_driven", "ordered") if k in kw}
    submits = [(int(s["t"]), int(s["len"]), int(s["tag"])) for s in subs]
    tx, st = ref.sender_replay(acks_des, submits, src, dst, cc=cc, policy=policy, **rkw)
    rate = kw.get("rate_bps", 400e9)
    bdp = int(round(rate * st["base_rtt"] / 8e9))
    commit_ahead = max(2 * kw["chunk_bytes"], 2 * 32768, bdp)
    assert commit_ahead == st["commit_ahead"], (commit_ahead, st["commit_ahead"])
    meta = dict(name=name, src=src, dst=dst, chunk_bytes=kw["chunk_bytes"], lb=kw["lb"],
                seed=kw["seed"], n_paths=int(st["n_paths"]), base_rtt=int(st["base_rtt"]),
                rto_min=int(st["rto_min"]), rto_max=int(st["rto_max"]), commit_ahead=commit_ahead,
                end_time=int(st["end_time"]), stats={k: int(v) for k, v in st.items()}, cc=cc,
                receiver_driven=bool(kw.get("receiver_driven", False)), initial_credit=int(st["bdp"]),
                ordered=bool(kw.get("ordered", False)), policy=POLICY_ENGINE_ID[policy],
                # the harness resolves Swift's target to 3 x base RTT (ref_harness.cpp)
                swift_target_ns=3 * int(st["base_rtt"]) if cc == "swift" else 0)
    pre = POLICY_NAMES[policy] + "_" if policy else ""
    path = os.path.join(GOLDEN, f"sender_{pre}{name}.npz" if cc == "none" else f"sender_{pre}{cc}_{name}.npz")
    sub_arr = np.array(submits, dtype=[("t", "<i8"), ("len", "<u8"), ("tag", "<u8")])
    np.savez_compressed(path, acks=acks_des, submits=sub_arr, tx=tx,
                        meta=np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8))
    print(f"  sender[{cc}]_{name}: submits={len(submits)} acks={len(acks_des)} tx={len(tx)} "
          f"rtx={st['chunk_rtx']} fast={st['fast_rtx']} rtos={st['rtos']} done={st['msgs_completed']}")


# single-connection Swift DES runs replayed into the reference sender under
# Swift: the replay must reproduce the DES sender's own transmissions
CLOSED_SWIFT = ["closed_k8", "closed_w4", "closed_cfg2"]
# trim-mode incasts: every connection replayed with its acks and NACKs
TRIM_SENDER = ["trim_swift", "trim_storm", "eqds_incast", "eqds_lossy", "ordered_loss", "ordered_trim"]

# Swift (device-exact CC) goldens: the same stimulus as sender_<name>.npz
SWIFT_SCENARIOS = ["cfg1", "cfg2_32k", "k8_4x1m", "multigen_k8", "lossy_2m", "csn_wrap"]


def gen_sender_swift(name):
    """sender_swift_<name>.npz from the stimulus already in sender_<name>.npz."""
    z = np.load(os.path.join(GOLDEN, f"sender_{name}.npz"))
    kw, flows = SCENARIOS[name]
    gen_sender(name, kw, flows, z["acks"], z["submits"], cc="swift")


# policy plug-ins (include/chunknet_policy.cuh; the same policies as
# TransportPolicy subclasses in ref_harness.cpp): the stimulus of
# sender_<name>.npz replayed under round robin / single path
POLICY_SCENARIOS = ["cfg1", "lossy_2m", "multigen_k8", "k8_4x1m"]


# Transport introspection (path_inflight, window_available, outstanding_bytes,
# conn_credit, engine_*) of the reference sender at times between its input
# events: probe_<name>.npz for tests/test_endpoint_gpu.py
PROBE_SCENARIOS = {"lossy_2m": "none", "multigen_k8": "swift", "closed_w4": "swift", "k8_4x1m": "none"}


def gen_probes(name, cc):
    z = np.load(os.path.join(GOLDEN, f"sender_{name}.npz" if cc == "none" else f"sender_{cc}_{name}.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    kw, flows = SCENARIOS[name]
    rkw = {k: kw[k] for k in ("topo", "topo_arg", "rate_bps", "qcap_bytes", "seed", "chunk_bytes",
                              "paths", "lb") if k in kw}
    acks, sub = z["acks"], z["submits"]
    ts = np.unique(np.concatenate([acks["aux"].astype(np.int64), sub["t"].astype(np.int64)]))
    mid = ts[:-1] + (ts[1:] - ts[:-1]) // 2
    pt = mid[(ts[1:] - ts[:-1]) >= 4][:: max(1, len(mid) // 40)] + 1
    submits = [(int(s["t"]), int(s["len"]), int(s["tag"])) for s in sub]
    tx, st, pr = ref.sender_replay(acks, submits, meta["src"], meta["dst"], cc=cc, probe_t=pt,
                                   probe_paths=int(meta["n_paths"]), **rkw)
    assert len(tx) == len(z["tx"])
    path = os.path.join(GOLDEN, f"probe_{name}.npz")
    np.savez_compressed(path, probe_t=pt, probes=pr, sender=np.frombuffer(
        (f"sender_{name}" if cc == "none" else f"sender_{cc}_{name}").encode(), dtype=np.uint8))
    print(f"  probe_{name}: {len(pt)} probes x {pr.shape[1]} values")


def gen_sender_policy(name, policy):
    z = np.load(os.path.join(GOLDEN, f"sender_{name}.npz"))
    kw, flows = SCENARIOS[name]
    gen_sender(name, kw, flows, z["acks"], z["submits"], policy=policy)


# reference experiment runs with run.trace = true (experiment.cpp:18-40): the
# trace writer's golden text, covering every event / kind / flag
TRACE_SCENARIOS = {
    "trim_incast": """[topology]
kind = star
hosts = 4
[net]
rate_gbps = 100
queue = trim
qcap_bytes = 65536
trim_depth = 2
[transport]
chunk_bytes = 16384
paths = 2
[workload]
pattern = incast
fan_in = 3
bytes_per_host = 262144
msg_bytes = 65536
dst = 0
[loss]
drop_ratio = 0.01
""",
    "eqds_incast": """[topology]
kind = star
hosts = 6
[net]
rate_gbps = 100
qcap_bytes = 131072
[transport]
chunk_bytes = 32768
paths = 1
receiver_driven = true
[workload]
pattern = incast
fan_in = 5
bytes_per_host = 262144
msg_bytes = 131072
dst = 0
""",
    "fat_tree_loss": """[topology]
kind = fat_tree
k = 4
[net]
rate_gbps = 100
qcap_bytes = 32768
[transport]
chunk_bytes = 8192
paths = 4
[cc]
algo = swift
[workload]
pattern = permutation
bytes_per_host = 131072
msg_bytes = 65536
[loss]
drop_ratio = 0.02
[run]
seed = 3
""",
    "ordered_loss": """[topology]
kind = star
hosts = 2
[net]
rate_gbps = 10
[transport]
reliability = ordered
paths = 1
[workload]
pattern = fixed
src = 0
dst = 1
bytes_per_host = 524288
msg_bytes = 262144
[loss]
drop_ratio = 0.02
[run]
seed = 4
""",
}


def gen_traces():
    out = {}
    for name, ini in TRACE_SCENARIOS.items():
        t = ref.experiment_trace(ini)
        out[f"ini_{name}"] = np.frombuffer(ini.encode(), dtype=np.uint8)
        out[f"tsv_{name}"] = np.frombuffer(t, dtype=np.uint8)
        kinds = sorted({ln.split(b"\t")[5].split(b",")[0] for ln in t.splitlines()})
        events = sorted({ln.split(b"\t")[1] for ln in t.splitlines()})
        print(f"trace {name}: {len(t.splitlines())} lines, events {events}, kinds {kinds}")
    path = os.path.join(GOLDEN, "trace.npz")
    np.savez_compressed(path, **out)
    print(f"trace: -> {os.path.getsize(path)} B")


def eqds_stream(rs, n_senders, n_events, t_step, sender_base=1):
    """A random but protocol-shaped input stream for one EQDS receiver:
    RTS registrations and resyncs (some flagged rtx), chunk arrivals (some
    retransmitted), trimmed headers; ties in time included."""
    from paper_2504_17307_b200.eqds import CHUNK, EV_DTYPE, RTS, TRIM
    ev = np.zeros(n_events, dtype=EV_DTYPE)
    t = 0
    known = []
    for i in range(n_events):
        t += 0 if rs.rand() < 0.1 else int(rs.randint(1, t_step))
        s = int(rs.randint(0, n_senders)) + sender_base
        u = rs.rand()
        if s not in known or u < 0.15:
            typ, arg, flag = RTS, int(rs.randint(1, 64)) * 32768 + int(rs.randint(0, 32768)), int(rs.rand() < 0.3)
            if s not in known:
                known.append(s)
        elif u < 0.25:
            typ, arg, flag = TRIM, int(rs.choice([32768, 16384, int(rs.randint(1, 32768))])), 0
        else:
            typ, arg, flag = CHUNK, int(rs.choice([32768, 32768, int(rs.randint(1, 32768))])), int(rs.rand() < 0.1)
        ev[i] = (t, typ, s, arg, flag, 0)
    return ev


# EqdsReceiver scenarios: (params, [per-receiver event streams])
def eqds_scenarios():
    from paper_2504_17307_b200.eqds import CHUNK, EV_DTYPE, RTS, TRIM, transport_params
    P = transport_params()  # 32 KiB quantum, 100 Gb/s tick, 4-quantum bank
    basic = np.array([(0, RTS, 1, 10 * 32768, 0, 0), (0, RTS, 2, 2 * 32768, 1, 0), (100, RTS, 3, 0, 0, 0),
                      (5000, CHUNK, 1, 32768, 0, 0), (5000, TRIM, 2, 32768, 0, 0),
                      (9000, CHUNK, 2, 32768, 1, 0), (20000, RTS, 1, 3 * 32768, 0, 0)], dtype=EV_DTYPE)
    out = {"basic": (dict(P, grant_to_idle=True), [basic])}
    rs = np.random.RandomState(21)
    out["incast40"] = (dict(P, grant_to_idle=True), [eqds_stream(rs, 40, 3000, 4000)])
    out["noidle"] = (dict(P, grant_to_idle=False), [eqds_stream(rs, 10, 1000, 6000)])
    out["multi16"] = (dict(P, grant_to_idle=True),
                      [eqds_stream(rs, int(rs.randint(8, 64)), 600, int(rs.randint(1500, 8000)),
                                   sender_base=100 * r) for r in range(16)])
    return out


def gen_eqds():
    out = {}
    for name, (prm, streams) in eqds_scenarios().items():
        offs, logs, loffs, gs = [0], [], [0], []
        for ev in streams:
            lg, g = ref.eqds_replay(ev, quantum=prm["quantum"], tick_ns=prm["tick_ns"], bank_cap=prm["bank_cap"],
                                    grant_to_idle=prm["grant_to_idle"])
            offs.append(offs[-1] + len(ev))
            logs.append(lg)
            loffs.append(loffs[-1] + len(lg))
            gs.append(g)
        out[f"{name}_events"] = np.concatenate(streams)
        out[f"{name}_offsets"] = np.array(offs, dtype=np.uint32)
        out[f"{name}_log"] = np.concatenate(logs)
        out[f"{name}_log_offsets"] = np.array(loffs, dtype=np.uint64)
        out[f"{name}_grants_sent"] = np.array(gs, dtype=np.uint64)
        out[f"{name}_params"] = np.frombuffer(json.dumps(prm).encode(), dtype=np.uint8)
        print(f"eqds {name}: receivers={len(streams)} events={offs[-1]} log={loffs[-1]} grants={sum(gs)}")
    path = os.path.join(GOLDEN, "eqds.npz")
    np.savez_compressed(path, **out)
    print(f"eqds: -> {os.path.getsize(path)} B")


# ------------------------------------------------------------ host-level
# One source host with several connections (fan-out), engines, conn_split,
# CUBIC and per-path CC scope: the host's submissions and the acks the DES
# delivered to it, replayed into a fresh reference Transport per config
# (ref_harness.cpp cnref_host_replay).  The per-host engine state
# (commit_ahead, factory rotation, DRR ring, max_inflight_msgs, pumps of
# every engine after an ack, transport.cpp:198-431, 941) couples the
# connections; only a host-level replay pins it.
HOST_DES = {
    # 1 -> 3 destinations on a k=8 fat tree (two inter-pod, one intra-pod),
    # CUBIC DES sender, 1% loss, two messages outstanding per connection
    "fanout_k8": (dict(topo="fat_tree", topo_arg=8, rate_bps=100e9, qcap_bytes=256 * 1024, loss=0.01,
                       seed=21, chunk_bytes=16384, paths=16, lb="p2_rtt", cc="cubic", window=2),
                  [(0, 127, 400_000, 4), (0, 64, 300_000, 4), (0, 9, 250_000, 4)], 0),
    # the same under Swift in the DES (its acks answer a Swift sender)
    "fanout_swift": (dict(topo="fat_tree", topo_arg=8, rate_bps=100e9, qcap_bytes=256 * 1024, loss=0.01,
                          seed=22, chunk_bytes=16384, paths=16, lb="p2_rtt", cc="swift", window=2),
                     [(0, 127, 400_000, 4), (0, 64, 300_000, 4), (0, 9, 250_000, 4)], 0),
    # receiver-driven (EQDS): one sender to three receivers, credit-gated
    "fanout_rd": (dict(topo="star", topo_arg=5, rate_bps=100e9, qcap_bytes=128 * 1024, loss=0.01, seed=23,
                       chunk_bytes=16384, paths=1, lb="oblivious", cc="none", receiver_driven=True, window=2),
                  [(0, 1, 512 * 1024, 3), (0, 2, 256 * 1024, 3), (0, 3, 300_000, 3)], 0),
    # multiple engines in the DES itself (home engines by load, conn_split)
    # per-path CC scope in the DES (closed loop for the per-path replays)
    "fanout_pp": (dict(topo="fat_tree", topo_arg=8, rate_bps=100e9, qcap_bytes=256 * 1024, loss=0.01,
                       seed=26, chunk_bytes=16384, paths=16, lb="p2_rtt", cc="cubic", cc_scope=1, window=2),
                  [(0, 127, 400_000, 4), (0, 64, 300_000, 4), (0, 9, 250_000, 4)], 0),
    "fanout_swift_pp": (dict(topo="fat_tree", topo_arg=8, rate_bps=100e9, qcap_bytes=256 * 1024, loss=0.01,
                             seed=27, chunk_bytes=16384, paths=16, lb="p2_ecn", cc="swift", cc_scope=1, window=2),
                        [(0, 127, 400_000, 4), (0, 64, 300_000, 4), (0, 9, 250_000, 4)], 0),
    "rd_swift": (dict(topo="star", topo_arg=5, rate_bps=100e9, qcap_bytes=128 * 1024, loss=0.01, seed=28,
                      chunk_bytes=16384, paths=1, lb="oblivious", cc="swift", receiver_driven=True, window=2),
                 [(0, 1, 512 * 1024, 3), (0, 2, 256 * 1024, 3), (0, 3, 300_000, 3)], 0),
    "split_swift": (dict(topo="fat_tree", topo_arg=8, rate_bps=100e9, qcap_bytes=256 * 1024, loss=0.02,
                         seed=29, chunk_bytes=8064, paths=16, lb="p2_rtt", cc="swift", engines=2, conn_split=1,
                         window=3), [(0, 127, 300_000, 5), (0, 64, 200_000, 5), (0, 9, 100_000, 4)], 0),
    "engines_k8": (dict(topo="fat_tree", topo_arg=8, rate_bps=100e9, qcap_bytes=256 * 1024, loss=0.02,
                        seed=24, chunk_bytes=8064, paths=16, lb="p2_rtt", cc="cubic", engines=4, window=3),
                   [(0, 127, 300_000, 5), (0, 64, 200_000, 5), (0, 100, 150_000, 5), (0, 9, 120_000, 5)], 0),
    "split_k8": (dict(topo="fat_tree", topo_arg=8, rate_bps=100e9, qcap_bytes=256 * 1024, loss=0.02,
                      seed=25, chunk_bytes=8064, paths=16, lb="p2_rtt", cc="cubic", engines=3, conn_split=1,
                      window=3), [(0, 127, 300_000, 5), (0, 64, 200_000, 5)], 0),
    # BASELINE configs[0] / [1] under CUBIC, the reference default: the DES
    # sender ran CUBIC, so the CUBIC replay is the DES sender itself
    "cfg1": (None, None, 0),
    "cfg2_32k": (None, None, 0),
    "k8_4x1m": (None, None, 0),
    "lossy_2m": (None, None, 0),
    "csn_wrap": (None, None, 0),
}
# name -> list of (tag, replay overrides)
HOST_REPLAYS = {
    "fanout_k8": [("none", dict(cc="none")), ("cubic", dict(cc="cubic")), ("swift", dict(cc="swift")),
                  ("cubic_pp", dict(cc="cubic", cc_scope=1)), ("swift_pp", dict(cc="swift", cc_scope=1)),
                  ("e2", dict(cc="cubic", engines=2)), ("e4split", dict(cc="cubic", engines=4, conn_split=True)),
                  ("swift_e3split", dict(cc="swift", engines=3, conn_split=True)),
                  ("inflight2", dict(cc="none", max_inflight_msgs=2)),
                  ("rr", dict(cc="swift", policy=1)), ("single", dict(cc="none", policy=2))],
    "fanout_swift": [("swift", dict(cc="swift")), ("swift_pp", dict(cc="swift", cc_scope=1)),
                     ("cubic", dict(cc="cubic")), ("swift_e2", dict(cc="swift", engines=2))],
    "fanout_rd": [("none", dict(cc="none")), ("swift", dict(cc="swift")), ("cubic", dict(cc="cubic"))],
    "fanout_pp": [("cubic_pp", dict(cc="cubic", cc_scope=1)), ("cubic", dict(cc="cubic")),
                  ("swift_pp_e2", dict(cc="swift", cc_scope=1, engines=2))],
    "fanout_swift_pp": [("swift_pp", dict(cc="swift", cc_scope=1)),
                        ("swift_pp_e4split", dict(cc="swift", cc_scope=1, engines=4, conn_split=True))],
    "rd_swift": [("swift", dict(cc="swift")), ("swift_pp", dict(cc="swift", cc_scope=1))],
    "split_swift": [("swift_e2split", dict(cc="swift", engines=2, conn_split=True)),
                    ("cubic_e2split", dict(cc="cubic", engines=2, conn_split=True))],
    "engines_k8": [("cubic_e4", dict(cc="cubic", engines=4)), ("cubic_e4split", dict(cc="cubic", engines=4,
                                                                                      conn_split=True)),
                   ("swift_e2", dict(cc="swift", engines=2)), ("cubic_pp_e4", dict(cc="cubic", engines=4,
                                                                                   cc_scope=1))],
    "split_k8": [("cubic_e3split", dict(cc="cubic", engines=3, conn_split=True)),
                 ("none_e3split", dict(cc="none", engines=3, conn_split=True)),
                 ("swift_pp_e2split", dict(cc="swift", engines=2, conn_split=True, cc_scope=1))],
    "cfg1": [("cubic", dict(cc="cubic")), ("cubic_pp", dict(cc="cubic", cc_scope=1))],
    "cfg2_32k": [("cubic", dict(cc="cubic"))],
    "k8_4x1m": [("cubic", dict(cc="cubic")), ("cubic_e2split", dict(cc="cubic", engines=2, conn_split=True))],
    "lossy_2m": [("cubic", dict(cc="cubic"))],
    "csn_wrap": [("cubic", dict(cc="cubic"))],
}


def gen_host(name):
    kw, flows, src = HOST_DES[name]
    if kw is None:  # a single-connection scenario recorded above: reuse its sender stimulus
        kw, flows = SCENARIOS[name]
        z = np.load(os.path.join(GOLDEN, f"sender_{name}.npz"))
        acks_des = z["acks"]
        subs = np.zeros(len(z["submits"]), dtype=ref.HOST_SUBMIT_DTYPE)
        for f in ("t", "len", "tag"):
            subs[f] = z["submits"][f]
        subs["dst"] = flows[0][1]
        src = flows[0][0]
        des_cc = kw["cc"]
    else:
        kw = dict(kw)
        window = kw.pop("window", 1)
        tmp = f"/tmp/cnfix_host_{name}"
        _, acks_all, _, st = ref.record(tmp, flows=flows, window=window, **kw)
        assert st["quiesced"] == 1, (name, st)
        assert st["bytes_ok"] == st["completions"], (name, st)
        sl = st["submits"]
        sl = sl[sl["src"] == src]
        acks_des = acks_all[acks_all["dst"] == src]
        subs = np.zeros(len(sl), dtype=ref.HOST_SUBMIT_DTYPE)
        for f in ("t", "len", "tag", "dst"):
            subs[f] = sl[f]
        des_cc = kw["cc"]
    rkw = {k: kw[k] for k in ("topo", "topo_arg", "rate_bps", "qcap_bytes", "seed", "chunk_bytes", "paths", "lb",
                              "receiver_driven", "ordered") if k in kw}
    # an open-loop replay (the DES ran another sender) can end in an RTO
    # storm once the recorded acks run out: stop 20 ms after the last input
    t_last = max(int(subs["t"].max()), int(acks_des["aux"].max()) if len(acks_des) else 0)
    rkw["cutoff_ns"] = t_last + 20_000_000
    for tag, over in HOST_REPLAYS[name]:
        r = dict(rkw)
        r.update(over)
        tx, stt, conns = ref.host_replay(acks_des, subs, src, **r)
        rate = kw.get("rate_bps", 400e9)
        bdp = int(round(rate * stt["base_rtt"] / 8e9))
        commit_ahead = max(2 * kw["chunk_bytes"], 2 * 32768, bdp)
        assert commit_ahead == stt["commit_ahead"], (commit_ahead, stt["commit_ahead"])
        cc = r.get("cc", "none")
        meta = dict(name=f"{name}_{tag}", src=int(src), conns=[int(c) for c in conns], chunk_bytes=kw["chunk_bytes"],
                    lb=r["lb"], seed=kw["seed"], paths=int(r["paths"]), base_rtt=int(stt["base_rtt"]),
                    rto_min=int(stt["rto_min"]), rto_max=int(stt["rto_max"]), commit_ahead=commit_ahead,
                    end_time=int(stt["end_time"]), stats={k: int(v) for k, v in stt.items()}, cc=cc,
                    cc_scope=int(r.get("cc_scope", 0)), engines=int(r.get("engines", 1)),
                    conn_split=bool(r.get("conn_split", False)), des_cc=des_cc,
                    receiver_driven=bool(r.get("receiver_driven", False)), initial_credit=int(stt["bdp"]),
                    policy=POLICY_ENGINE_ID[r.get("policy", 0)],
                    max_inflight_msgs=int(r.get("max_inflight_msgs", 0)) or 128,
                    swift_target_ns=3 * int(stt["base_rtt"]) if cc == "swift" else 0,
                    topo=kw.get("topo"), topo_arg=kw.get("topo_arg"), rate_bps=kw.get("rate_bps", 400e9),
                    qcap_bytes=kw.get("qcap_bytes", 1 << 20), cutoff_ns=int(rkw["cutoff_ns"]))
        # the reference's path count per connection: min(paths, path_count(src, dst))
        meta["n_paths"] = [int(x) for x in _path_counts(kw, src, conns)]
        path = os.path.join(GOLDEN, f"host_{name}_{tag}.npz")
        np.savez_compressed(path, acks=acks_des, submits=subs, tx=tx,
                            meta=np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8))
        print(f"  host_{name}_{tag}: conns={len(conns)} submits={len(subs)} acks={len(acks_des)} tx={len(tx)} "
              f"rtx={stt['chunk_rtx']} fast={stt['fast_rtx']} rtos={stt['rtos']} done={stt['msgs_completed']}"
              f" rts={stt['rts_sent']}")


def _path_counts(kw, src, conns):
    """min(paths, topo.path_count(src, dst)) per connection (conn_to,
    transport.cpp:97-99): fat tree k -- same edge switch 1, same pod k/2,
    other pod k^2/4 (topology.cpp:47-56); star 1."""
    out = []
    for dst in conns:
        if kw.get("topo") == "star":
            pc = 1
        else:
            k = kw["topo_arg"]
            per_edge, per_pod = k // 2, (k // 2) * (k // 2)
            if src // per_edge == dst // per_edge:
                pc = 1
            elif src // per_pod == dst // per_pod:
                pc = k // 2
            else:
                pc = per_pod
        out.append(min(kw["paths"], pc) if src != dst else 1)
    return out


# ------------------------------------------------------ randomized suite
# The reference's own property suite (test_reliability_props.cpp:126-218):
# seed -> topology (star 8 / fat tree k=4), rate, delay, drop, chunk size,
# paths, engines, conn_split, LB, CC algo and scope, receiver-driven /
# ordered modes and 3-5 messages, drawn over its RngStream by the harness
# (cnref_prop_spec_draw).  Every seed is recorded in the reference DES, the
# delivered packets replayed into its receive path (rx parity) and each
# source host's submissions and acks into a host-level sender replay
# (sender parity).  Builder's extension: seeds with seed % 10 == 5 run the
# switch queues in trim mode (64 KiB) so trimmed headers and NACKs appear.
# kind 1: the engine-invariance case (:328-358), engines 1 / 2 / 4.
LB_NAMES = ["oblivious", "p2_rtt", "p2_ecn"]
CC_NAMES = ["none", "cubic", "swift"]
PROPS_DIR = os.path.join(GOLDEN, "props")


def gen_prop(seed, kind=0, engines=None):
    sp = ref.prop_spec(seed, kind)
    kw = dict(topo="star" if sp["star"] else "fat_tree", topo_arg=sp["topo_arg"], rate_bps=sp["rate_bps"],
              link_delay_ns=sp["link_delay_ns"], qcap_bytes=0, loss=sp["drop"], seed=seed,
              chunk_bytes=sp["chunk_bytes"], paths=sp["paths"], lb=LB_NAMES[sp["lb"]], cc=CC_NAMES[sp["cc"]],
              cc_scope=sp["cc_scope"], engines=sp["engines"], conn_split=sp["conn_split"],
              receiver_driven=bool(sp["receiver_driven"]), ordered=bool(sp["ordered"]))
    if kind == 1:
        kw.update(engines=engines, conn_split=1 if engines > 1 else 0)
    trim = kind == 0 and seed % 10 == 5
    if trim:
        kw.update(queue="trim", qcap_bytes=64 * 1024, trim_depth=8)
    flows = [(s_, d_, ln, 1) for s_, d_, ln, _ in sp["msgs"]]
    tmp = f"/tmp/cnprop_{kind}_{seed}_{engines}"
    data, acks_des, _, st = ref.record(tmp, flows=flows, window=1, cutoff_ns=2_000_000_000, **kw)
    assert st["quiesced"] == 1 and st["bytes_ok"] == st["completions"] == len(flows), (seed, st)
    psn = st.pop("psn")
    ordered = kw["ordered"]
    acks, cpls, _ = ref.rx_replay(data, st["n_hosts"], kw["chunk_bytes"], psn=psn if ordered else None,
                                  ordered=ordered)
    out = {"data": data, "acks": acks, "completions": cpls}
    if ordered:
        out["psn"] = psn
    sl = st.pop("submits")
    hosts = []
    for s_ in [m[0] for m in sp["msgs"]]:
        if s_ not in hosts:
            hosts.append(s_)
    host_meta = []
    for h in hosts:
        sub = sl[sl["src"] == h]
        subs = np.zeros(len(sub), dtype=ref.HOST_SUBMIT_DTYPE)
        for f in ("t", "len", "tag", "dst"):
            subs[f] = sub[f]
        ah = acks_des[acks_des["dst"] == h]
        t_last = max(int(subs["t"].max()), int(ah["aux"].max()) if len(ah) else 0)
        rkw = dict(topo=kw["topo"], topo_arg=kw["topo_arg"], rate_bps=kw["rate_bps"],
                   link_delay_ns=kw["link_delay_ns"], qcap_bytes=0, seed=seed, chunk_bytes=kw["chunk_bytes"],
                   paths=kw["paths"], lb=kw["lb"], cc=kw["cc"], cc_scope=kw["cc_scope"], engines=kw["engines"],
                   conn_split=bool(kw["conn_split"]), receiver_driven=kw["receiver_driven"], ordered=ordered,
                   cutoff_ns=t_last + 20_000_000)
        tx, stt, conns = ref.host_replay(ah, subs, h, **rkw)
        swift_t = 3 * int(stt["base_rtt"]) if kw["cc"] == "swift" else 0
        host_meta.append(dict(src=int(h), conns=[int(c) for c in conns],
                              n_paths=[int(x) for x in _path_counts(kw, h, conns)],
                              base_rtt=int(stt["base_rtt"]), rto_min=int(stt["rto_min"]),
                              rto_max=int(stt["rto_max"]), commit_ahead=int(stt["commit_ahead"]),
                              initial_credit=int(stt["bdp"]), end_time=int(stt["end_time"]),
                              swift_target_ns=swift_t, stats={k: int(v) for k, v in stt.items()}))
        out[f"h{h}_acks"] = ah
        out[f"h{h}_submits"] = subs
        out[f"h{h}_tx"] = tx
    meta = dict(seed=seed, kind=kind, trim=trim, record=kw, flows=flows, n_hosts=int(st["n_hosts"]),
                chunk_bytes=kw["chunk_bytes"], des_stats={k: int(v) for k, v in st.items()}, hosts=host_meta)
    os.makedirs(PROPS_DIR, exist_ok=True)
    name = f"prop_{seed}" if kind == 0 else f"enginv_{seed}_e{engines}"
    np.savez_compressed(os.path.join(PROPS_DIR, f"{name}.npz"),
                        meta=np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8), **out)
    return meta


def gen_props(n_seeds=256):
    tally = dict(star=0, ordered=0, rd=0, trim=0, multi_engine=0, split=0, rtx=0, rtos=0, fast=0, cubic=0,
                 per_path=0)
    for seed in range(n_seeds):
        m = gen_prop(seed)
        r = m["record"]
        tally["star"] += r["topo"] == "star"
        tally["ordered"] += r["ordered"]
        tally["rd"] += r["receiver_driven"]
        tally["trim"] += m["trim"]
        tally["multi_engine"] += r["engines"] > 1
        tally["split"] += bool(r["conn_split"])
        tally["cubic"] += r["cc"] == "cubic"
        tally["per_path"] += r["cc_scope"] == 1
        tally["rtx"] += m["des_stats"]["chunk_rtx"]
        tally["rtos"] += m["des_stats"]["rtos"]
        tally["fast"] += m["des_stats"]["fast_rtx"]
    for seed in range(12):
        for e in (1, 2, 4):
            gen_prop(seed, kind=1, engines=e)
    print("props:", tally)


def gen_rng():
    """RngStream / select_path draw sequences (rng.hpp:29-60, lb.cpp:7-27).

    The reference tests pin only statistics here (test_lb.cpp:34-108), so
    the literal sequences come from running the compiled reference."""
    out = {}
    # raw mt19937_64 outputs of per-connection streams (transport.cpp:101)
    for idx in (0, 1, 2, 255, 1023):
        out[f"u64_conn{idx}"] = ref.rng_u64(1, "transport.conn", idx, 1000)
    out["u64_named_loss7"] = ref.rng_u64(42, "loss", 7, 1000)
    out["u64_unindexed"] = ref.rng_u64(9, "workload", -1, 1000)
    # next_below over assorted ranges incl. non powers of two (Lemire rejection)
    rs = np.random.RandomState(5)
    ns = np.concatenate([np.array([1, 2, 3, 7, 8, 255, 256, 1000, 2**33 + 5,
                                   2**63 + 1, 2**64 - 1], dtype=np.uint64),
                         rs.randint(1, 1 << 30, size=4000).astype(np.uint64)])
    out["below_ns"] = ns
    out["below_vals"] = ref.next_below(3, "transport.conn", 17, ns)
    out["double_vals"] = ref.next_double(3, "loss", 2, 1000)
    # select_path on fixed boards
    for n_paths in (1, 2, 7, 8, 256):
        rtt = 10000.0 + rs.randint(0, 5000, size=n_paths).astype(np.float64)
        rtt[rs.randint(0, n_paths, size=max(1, n_paths // 4))] = 12345.0  # ties
        ecn = rs.randint(0, 9, size=n_paths) / 8.0
        out[f"board{n_paths}_rtt"] = rtt
        out[f"board{n_paths}_ecn"] = ecn
        for pol in ("oblivious", "p2_rtt", "p2_ecn"):
            for idx in (0, 5):
                out[f"sel_{pol}_{n_paths}_{idx}"] = ref.select_paths(
                    pol, rtt, ecn, 1, "transport.conn", idx, 2000)
    path = os.path.join(GOLDEN, "rng.npz")
    np.savez_compressed(path, **out)
    print(f"rng: {len(out)} arrays -> {os.path.getsize(path)} B")


def main(argv):
    os.makedirs(GOLDEN, exist_ok=True)
    names = argv or list(SCENARIOS) + ["rng", "swift", "trace", "eqds", "policy", "probe"]
    for n in names:
        if n == "probe":
            for m, cc in PROBE_SCENARIOS.items():
                gen_probes(m, cc)
            continue
        if n == "policy":
            for m in POLICY_SCENARIOS:
                for pol in POLICY_NAMES:
                    gen_sender_policy(m, pol)
            continue
        if n == "rng":
            gen_rng()
            continue
        if n == "props":
            gen_props()
            continue
        if n == "host":
            for m in HOST_DES:
                gen_host(m)
            continue
        if n.startswith("host_"):
            gen_host(n[5:])
            continue
        if n == "eqds":
            gen_eqds()
            continue
        if n == "trace":
            gen_traces()
            continue
        if n == "swift":
            for m in SWIFT_SCENARIOS:
                gen_sender_swift(m)
            continue
        kw, flows = SCENARIOS[n]
        gen(n, kw, flows)


if __name__ == "__main__":
    main(sys.argv[1:])
