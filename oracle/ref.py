"""ctypes wrapper of oracle/_ref/libcnref.so -- TEST INFRASTRUCTURE ONLY.

libcnref.so is the UNMODIFIED reference chunknet library compiled from
/root/reference/proj/src by oracle/Makefile, plus oracle/ref_harness.cpp.
Only tests/, __graft_entry__.smoke() and bench.py's cpu-baseline /
--impl reference legs may import this module.
"""
import ctypes
import os

import numpy as np

from .records import ACK_DTYPE, CPL_DTYPE, PKT_DTYPE

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libcnref.so")

LB = {"oblivious": 0, "p2_rtt": 1, "p2_ecn": 2}
CC = {"none": 0, "cubic": 1, "swift": 2}


class Scenario(ctypes.Structure):
    _fields_ = [
        ("topo_kind", ctypes.c_int32), ("topo_arg", ctypes.c_int32),
        ("rate_bps", ctypes.c_double), ("link_delay_ns", ctypes.c_int64),
        ("qcap_bytes", ctypes.c_int64), ("loss", ctypes.c_double),
        ("seed", ctypes.c_uint64), ("chunk_bytes", ctypes.c_uint32),
        ("paths", ctypes.c_int32), ("lb", ctypes.c_int32), ("cc", ctypes.c_int32),
        ("cc_scope", ctypes.c_int32), ("engines", ctypes.c_int32),
        ("conn_split", ctypes.c_int32), ("dupack_threshold", ctypes.c_int32),
        ("rto_min", ctypes.c_int64), ("n_flows", ctypes.c_int32),
        ("window", ctypes.c_int32), ("cutoff_ns", ctypes.c_int64),
        ("queue_mode", ctypes.c_int32), ("trim_depth", ctypes.c_int32),
        ("receiver_driven", ctypes.c_int32), ("ordered", ctypes.c_int32),
        ("policy", ctypes.c_int32), ("pad_policy", ctypes.c_int32),
    ]


QUEUE = {"drop_tail": 0, "trim": 1, "pause": 2}


class Flow(ctypes.Structure):
    _fields_ = [("src", ctypes.c_int32), ("dst", ctypes.c_int32),
                ("len", ctypes.c_uint64), ("count", ctypes.c_int32),
                ("pad", ctypes.c_int32)]


class RecordStats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "data_pkts", "acks_at_sender", "completions", "chunks_sent", "chunk_rtx",
        "fast_rtx", "rtos", "acks_sent", "loss_dropped")] + [
        ("end_time", ctypes.c_int64), ("quiesced", ctypes.c_int32),
        ("n_hosts", ctypes.c_int32), ("bytes_ok", ctypes.c_uint64)]


class RxOut(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "n_acks", "n_completions", "arena_used", "acks_sent_stat")]


class TxRec(ctypes.Structure):
    _fields_ = [("t", ctypes.c_int64), ("msg_id", ctypes.c_uint32), ("chunk", ctypes.c_uint32),
                ("path", ctypes.c_int32), ("is_rtx", ctypes.c_int32), ("msg_seq", ctypes.c_uint64)]


class SenderStats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "chunks_sent", "chunk_rtx", "fast_rtx", "rtos", "msgs_completed", "n_tx")] + [
        (n, ctypes.c_int64) for n in ("base_rtt", "rto_min", "rto_max", "end_time")] + [
        ("n_paths", ctypes.c_int32), ("pad", ctypes.c_int32),
        ("bdp", ctypes.c_int64), ("commit_ahead", ctypes.c_int64), ("rts_sent", ctypes.c_uint64)]


class PropSpec(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("star", "topo_arg", "ordered", "receiver_driven", "zero_loss",
                                               "engines", "conn_split", "paths", "lb", "cc", "cc_scope",
                                               "n_msgs")] + [
        ("chunk_bytes", ctypes.c_uint32), ("pad", ctypes.c_uint32), ("rate_bps", ctypes.c_double),
        ("drop", ctypes.c_double), ("link_delay_ns", ctypes.c_int64), ("src", ctypes.c_int32 * 8),
        ("dst", ctypes.c_int32 * 8), ("len", ctypes.c_uint64 * 8), ("tag", ctypes.c_uint64 * 8)]


def prop_spec(seed, kind=0):
    """The reference property suite's scenario draws for `seed`
    (test_reliability_props.cpp: kind 0 run_scenario, kind 1 the
    engine-invariance case), as a dict."""
    o = PropSpec()
    lib().cnref_prop_spec_draw(seed, kind, ctypes.byref(o))
    d = {k: getattr(o, k) for k, _ in PropSpec._fields_ if k not in ("src", "dst", "len", "tag", "pad")}
    n = o.n_msgs
    d["msgs"] = [(o.src[i], o.dst[i], int(o.len[i]), int(o.tag[i])) for i in range(n)]
    return d


class Submit(ctypes.Structure):
    _fields_ = [("t", ctypes.c_int64), ("len", ctypes.c_uint64), ("tag", ctypes.c_uint64)]


SUBMIT_LOG_DTYPE = np.dtype([("t", "<i8"), ("len", "<u8"), ("tag", "<u8"), ("src", "<i4"),
                             ("dst", "<i4")])
TX_DTYPE = np.dtype([("t", "<i8"), ("msg_id", "<u4"), ("chunk", "<u4"), ("path", "<i4"),
                     ("is_rtx", "<i4"), ("msg_seq", "<u8")])
HOST_TX_DTYPE = np.dtype([("t", "<i8"), ("msg_id", "<u4"), ("chunk", "<u4"), ("path", "<i4"),
                          ("is_rtx", "<i4"), ("msg_seq", "<u8"), ("conn", "<u4"), ("dst", "<i4")])
HOST_SUBMIT_DTYPE = np.dtype([("t", "<i8"), ("len", "<u8"), ("tag", "<u8"), ("dst", "<i4"), ("pad", "<i4")])

_lib = None


def available():
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"{LIB_PATH} missing: run `make -C oracle ref` "
                               "where /root/reference is mounted")
        L = ctypes.CDLL(LIB_PATH)
        vp, u64, i64, i32, u32 = (ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64,
                                  ctypes.c_int, ctypes.c_uint32)
        L.cnref_last_error.restype = ctypes.c_char_p
        L.cnref_record.argtypes = [ctypes.POINTER(Scenario), ctypes.POINTER(Flow),
                                   ctypes.c_char_p, ctypes.POINTER(RecordStats)]
        L.cnref_rx_replay.argtypes = [vp, u64, i32, u32, i32, vp, u64, vp, u64, vp,
                                      u64, ctypes.POINTER(RxOut), vp, i32]
        L.cnref_rx_replay_bench.argtypes = [vp, u64, i32, u32, i32, i32]
        L.cnref_rx_replay_bench.restype = ctypes.c_double
        L.cnref_sender_replay.argtypes = [ctypes.POINTER(Scenario), i32, i32, vp, u64, vp, u64,
                                          vp, u64, ctypes.POINTER(SenderStats)]
        L.cnref_sender_replay_bench.argtypes = [ctypes.POINTER(Scenario), i32, i32, vp, u64, vp,
                                                u64, i32, i32]
        L.cnref_sender_replay_bench.restype = ctypes.c_double
        L.cnref_set_probes.argtypes = [vp, u32, vp, u32]
        L.cnref_set_probes.restype = None
        L.cnref_host_replay.argtypes = [ctypes.POINTER(Scenario), i32, vp, u64, vp, u64, vp, u64,
                                        ctypes.POINTER(SenderStats), vp, u32, i32, i32]
        L.cnref_set_host_probes.argtypes = [vp, u32, vp, u32, u32]
        L.cnref_prop_spec_draw.argtypes = [u64, i32, vp]
        L.cnref_set_host_probes.restype = None
        L.cnref_rng_u64.argtypes = [u64, ctypes.c_char_p, i64, u64, vp]
        L.cnref_next_below.argtypes = [u64, ctypes.c_char_p, i64, vp, u64, vp]
        L.cnref_next_double.argtypes = [u64, ctypes.c_char_p, i64, u64, vp]
        L.cnref_select_paths.argtypes = [i32, i32, vp, vp, u64, ctypes.c_char_p, i64,
                                         u64, vp]
        L.cnref_select_paths_bench.argtypes = [i32, i32, i32, u64, i32, vp]
        L.cnref_select_paths_bench.restype = ctypes.c_double
        L.cnref_encode_header.argtypes = [ctypes.c_uint8] * 3 + [i32, ctypes.c_uint8,
                                                                 ctypes.POINTER(u32)]
        L.cnref_csn_before.argtypes = [ctypes.c_uint8] * 3 + [i32, ctypes.POINTER(i32)]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def record(outdir, *, topo="fat_tree", topo_arg=8, rate_bps=400e9,
           link_delay_ns=1000, qcap_bytes=1 << 20, loss=0.0, seed=1,
           chunk_bytes=32768, paths=8, lb="p2_rtt", cc="cubic", cc_scope=0,
           engines=1, conn_split=0, dupack_threshold=8, rto_min=0, flows=(),
           window=1, cutoff_ns=60_000_000_000, queue="drop_tail", trim_depth=0, receiver_driven=False,
           ordered=False):
    """Runs the reference DES and writes data.bin / acks_des.bin /
    completions_des.bin into outdir.  flows: [(src, dst, len, count)]."""
    sc = Scenario(0 if topo == "star" else 1, topo_arg, rate_bps, link_delay_ns,
                  qcap_bytes, loss, seed, chunk_bytes, paths, LB[lb], CC[cc],
                  cc_scope, engines, conn_split, dupack_threshold, rto_min,
                  len(flows), window, cutoff_ns, QUEUE[queue], trim_depth, 1 if receiver_driven else 0,
                  1 if ordered else 0)
    fl = (Flow * max(1, len(flows)))(*[Flow(s, d, l, c, 0) for (s, d, l, c) in flows])
    st = RecordStats()
    os.makedirs(outdir, exist_ok=True)
    rc = lib().cnref_record(ctypes.byref(sc), fl, outdir.encode(), ctypes.byref(st))
    if rc != 0:
        raise RuntimeError(lib().cnref_last_error().decode())
    data = np.fromfile(os.path.join(outdir, "data.bin"), dtype=PKT_DTYPE)
    psn = np.fromfile(os.path.join(outdir, "psn.bin"), dtype=np.uint64)
    acks = np.fromfile(os.path.join(outdir, "acks_des.bin"), dtype=ACK_DTYPE)
    cpls = np.fromfile(os.path.join(outdir, "completions_des.bin"), dtype=CPL_DTYPE)
    subs = np.fromfile(os.path.join(outdir, "submits.bin"), dtype=SUBMIT_LOG_DTYPE)
    st_d = {k: getattr(st, k) for k, _ in RecordStats._fields_}
    st_d["submits"] = subs
    st_d["psn"] = psn
    return data, acks, cpls, st_d


def sender_replay(acks, submits, src, dst, *, topo="fat_tree", topo_arg=8, rate_bps=400e9,
                  link_delay_ns=1000, qcap_bytes=1 << 20, seed=1, chunk_bytes=32768, paths=8,
                  lb="p2_rtt", cc="none", cc_scope=0, dupack_threshold=8, rto_min=0,
                  cutoff_ns=60_000_000_000, max_out=1 << 20, receiver_driven=False, ordered=False,
                  policy=0, probe_t=None, probe_paths=0):
    """Reference sender over a blackhole: submits [(t, len, tag)] and acks
    (ACK_DTYPE, aux = delivery time at the sender; also NACK / credit /
    rts_ack records) -> (tx log, stats).  Receiver-driven: RTS packets are
    logged as records with chunk = 0xFFFFFFFF, msg_seq = demand.  policy:
    0 DefaultPolicy, 1 round robin, 2 single path, 3 the example plug-in
    (TransportPolicy subclasses installed with set_policy_factory,
    ref_harness.cpp)."""
    sc = Scenario(0 if topo == "star" else 1, topo_arg, rate_bps, link_delay_ns, qcap_bytes, 0.0,
                  seed, chunk_bytes, paths, LB[lb], CC[cc], cc_scope, 1, 0, dupack_threshold,
                  rto_min, 0, 1, cutoff_ns, 0, 0, 1 if receiver_driven else 0, 1 if ordered else 0,
                  policy, 0)
    sb = (Submit * max(1, len(submits)))(*[Submit(int(t), int(l), int(g)) for t, l, g in submits])
    acks = np.ascontiguousarray(acks, dtype=ACK_DTYPE)
    out = np.zeros(max_out, dtype=TX_DTYPE)
    st = SenderStats()
    probes = None
    if probe_t is not None:  # Transport introspection at these times (cnref_set_probes)
        pt = np.ascontiguousarray(probe_t, dtype=np.int64)
        probes = np.zeros((len(pt), 5 + 2 * probe_paths), dtype=np.int64)
        lib().cnref_set_probes(_ptr(pt), len(pt), _ptr(probes), probes.shape[1])
    try:
        rc = lib().cnref_sender_replay(ctypes.byref(sc), src, dst, ctypes.cast(sb, ctypes.c_void_p),
                                       len(submits), _ptr(acks), len(acks), _ptr(out), max_out,
                                       ctypes.byref(st))
    finally:
        if probe_t is not None:
            lib().cnref_set_probes(None, 0, None, 0)
    if rc != 0:
        raise RuntimeError(lib().cnref_last_error().decode())
    res = out[: min(st.n_tx, max_out)].copy(), {k: getattr(st, k) for k, _ in SenderStats._fields_}
    return res + (probes,) if probe_t is not None else res


def host_replay(acks, submits, src, *, topo="fat_tree", topo_arg=8, rate_bps=400e9, link_delay_ns=1000,
                qcap_bytes=1 << 20, seed=1, chunk_bytes=32768, paths=8, lb="p2_rtt", cc="none", cc_scope=0,
                engines=1, conn_split=False, dupack_threshold=8, rto_min=0, cutoff_ns=60_000_000_000,
                max_out=1 << 21, receiver_driven=False, ordered=False, policy=0, ecn_as_loss=False,
                max_inflight_msgs=0, probe_t=None, probe_conns=0, probe_paths=0):
    """The reference sender of one source host (ref_harness.cpp
    cnref_host_replay): submits HOST_SUBMIT_DTYPE (t, len, tag, dst), acks
    delivered at `src` -> (tx log HOST_TX_DTYPE in emission order, stats,
    dst per connection index in creation order[, probes])."""
    sc = Scenario(0 if topo == "star" else 1, topo_arg, rate_bps, link_delay_ns, qcap_bytes, 0.0,
                  seed, chunk_bytes, paths, LB[lb], CC[cc], cc_scope, engines, 1 if conn_split else 0,
                  dupack_threshold, rto_min, 0, 1, cutoff_ns, 0, 0, 1 if receiver_driven else 0,
                  1 if ordered else 0, policy, 0)
    sb = np.ascontiguousarray(submits, dtype=HOST_SUBMIT_DTYPE)
    acks = np.ascontiguousarray(acks, dtype=ACK_DTYPE)
    out = np.zeros(max_out, dtype=HOST_TX_DTYPE)
    conns = np.full(4096, -1, dtype=np.int32)
    st = SenderStats()
    probes = None
    if probe_t is not None:
        pt = np.ascontiguousarray(probe_t, dtype=np.int64)
        probes = np.zeros((len(pt), 3 * engines + probe_conns * (2 + 2 * probe_paths)), dtype=np.int64)
        lib().cnref_set_host_probes(_ptr(pt), len(pt), _ptr(probes), probe_conns, probe_paths)
    try:
        rc = lib().cnref_host_replay(ctypes.byref(sc), src, _ptr(sb), len(sb), _ptr(acks), len(acks), _ptr(out),
                                     max_out, ctypes.byref(st), _ptr(conns), len(conns), 1 if ecn_as_loss else 0,
                                     max_inflight_msgs)
    finally:
        if probe_t is not None:
            lib().cnref_set_host_probes(None, 0, None, 0, 0)
    if rc != 0:
        raise RuntimeError(lib().cnref_last_error().decode())
    n_conns = int(st.n_paths)
    res = (out[: min(st.n_tx, max_out)].copy(), {k: getattr(st, k) for k, _ in SenderStats._fields_},
           conns[:n_conns].copy())
    return res + (probes,) if probe_t is not None else res


def sender_replay_bench(acks, submits, src, dst, threads=1, reps=1, *, topo="fat_tree",
                        topo_arg=8, rate_bps=400e9, link_delay_ns=1000, qcap_bytes=1 << 20, seed=1,
                        chunk_bytes=32768, paths=8, lb="p2_rtt", dupack_threshold=8,
                        cutoff_ns=60_000_000_000):
    sc = Scenario(0 if topo == "star" else 1, topo_arg, rate_bps, link_delay_ns, qcap_bytes, 0.0,
                  seed, chunk_bytes, paths, LB[lb], CC["none"], 0, 1, 0, dupack_threshold, 0, 0, 1,
                  cutoff_ns)
    sb = (Submit * max(1, len(submits)))(*[Submit(int(t), int(l), int(g)) for t, l, g in submits])
    acks = np.ascontiguousarray(acks, dtype=ACK_DTYPE)
    return lib().cnref_sender_replay_bench(ctypes.byref(sc), src, dst, ctypes.cast(sb, ctypes.c_void_p),
                                           len(submits), _ptr(acks), len(acks), threads, reps)


def rx_replay(recs, n_hosts, chunk_bytes, carry_payload=True, arena_bytes=None, psn=None, ordered=False):
    """Reference receive path over recorded packets -> (acks, completions, arena)."""
    recs = np.ascontiguousarray(recs, dtype=PKT_DTYPE)
    n = len(recs)
    max_acks = n + 16
    acks = np.zeros(max_acks, dtype=ACK_DTYPE)
    cpls = np.zeros(n + 16, dtype=CPL_DTYPE)
    if arena_bytes is None:
        lens = {}
        for t, l in zip(recs["msg_tag"], recs["msg_len"]):
            lens[(int(t), int(l))] = int(l)
        arena_bytes = sum(((l + 15) // 16) * 16 for l in lens.values()) * 2 + 64
    arena = np.zeros(arena_bytes if carry_payload else 1, dtype=np.uint8)
    out = RxOut()
    rc = lib().cnref_rx_replay(_ptr(recs), n, n_hosts, chunk_bytes,
                               1 if carry_payload else 0, _ptr(acks), max_acks,
                               _ptr(cpls), len(cpls), _ptr(arena),
                               arena.nbytes if carry_payload else 0, ctypes.byref(out),
                               _ptr(np.ascontiguousarray(psn, dtype=np.uint64)) if psn is not None else None,
                               1 if ordered else 0)
    if rc != 0:
        raise RuntimeError(lib().cnref_last_error().decode())
    return acks[: out.n_acks].copy(), cpls[: out.n_completions].copy(), arena[: out.arena_used]


def rx_replay_bench(recs, n_hosts, chunk_bytes, threads=1, reps=1):
    recs = np.ascontiguousarray(recs, dtype=PKT_DTYPE)
    return lib().cnref_rx_replay_bench(_ptr(recs), len(recs), n_hosts, chunk_bytes,
                                       threads, reps)


def rng_u64(seed, name, index, count):
    out = np.zeros(count, dtype=np.uint64)
    lib().cnref_rng_u64(seed, name.encode(), index, count, _ptr(out))
    return out


def next_below(seed, name, index, ns):
    ns = np.ascontiguousarray(ns, dtype=np.uint64)
    out = np.zeros(len(ns), dtype=np.uint64)
    lib().cnref_next_below(seed, name.encode(), index, _ptr(ns), len(ns), _ptr(out))
    return out


def next_double(seed, name, index, count):
    out = np.zeros(count, dtype=np.float64)
    lib().cnref_next_double(seed, name.encode(), index, count, _ptr(out))
    return out


def select_paths(policy, rtt, ecn, seed, name, index, count):
    rtt = np.ascontiguousarray(rtt, dtype=np.float64)
    ecn = np.ascontiguousarray(ecn, dtype=np.float64)
    out = np.zeros(count, dtype=np.int32)
    lib().cnref_select_paths(LB[policy], len(rtt), _ptr(rtt), _ptr(ecn), seed,
                             name.encode(), index, count, _ptr(out))
    return out


def select_paths_bench(policy, n_paths, conns, count, threads=1):
    cs = np.zeros(1, dtype=np.uint64)
    t = lib().cnref_select_paths_bench(LB[policy], n_paths, conns, count, threads, _ptr(cs))
    return t, int(cs[0])


def encode_header(conn, msg, csn, last, rsvd):
    out = ctypes.c_uint32()
    rc = lib().cnref_encode_header(conn, msg, csn, int(last), rsvd, ctypes.byref(out))
    return rc, out.value


def csn_before(a, b, base, width):
    out = ctypes.c_int()
    rc = lib().cnref_csn_before(a, b, base, width, ctypes.byref(out))
    return rc, out.value


def experiment_trace(ini):
    """The reference's run_experiment on an ExperimentSpec INI text with
    run.trace = true -> its trace.tsv text (experiment.cpp trace_line)."""
    L = lib()
    L.cnref_experiment_trace.restype = ctypes.c_int64
    L.cnref_experiment_trace.argtypes = [ctypes.c_char_p, ctypes.c_void_p, ctypes.c_uint64]
    b = ini.encode()
    n = L.cnref_experiment_trace(b, None, 0)
    if n < 0:
        raise RuntimeError(L.cnref_last_error().decode())
    buf = ctypes.create_string_buffer(max(1, n))
    L.cnref_experiment_trace(b, buf, n)
    return buf.raw[:n]


def eqds_replay(events, *, quantum, tick_ns, bank_cap, grant_to_idle=True, cutoff=1 << 62, max_out=1 << 20):
    """The reference EqdsReceiver (eqds.cpp) over scripted events
    (paper_2504_17307_b200.eqds.EV_DTYPE) -> (log LOG_DTYPE, grants_sent)."""
    from paper_2504_17307_b200.eqds import EV_DTYPE, LOG_DTYPE
    L = lib()
    L.cnref_eqds_replay.restype = ctypes.c_int
    L.cnref_eqds_replay.argtypes = [ctypes.c_uint32, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                    ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p,
                                    ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64),
                                    ctypes.POINTER(ctypes.c_uint64)]
    ev = np.ascontiguousarray(events, dtype=EV_DTYPE)
    out = np.zeros(max_out, dtype=LOG_DTYPE)
    n, gs = ctypes.c_uint64(), ctypes.c_uint64()
    rc = L.cnref_eqds_replay(quantum, tick_ns, bank_cap, 1 if grant_to_idle else 0, _ptr(ev), len(ev), cutoff,
                             _ptr(out), max_out, ctypes.byref(n), ctypes.byref(gs))
    if rc != 0:
        raise RuntimeError(L.cnref_last_error().decode())
    return out[: min(n.value, max_out)].copy(), gs.value
