"""Device sender engine (C ABI cn_tx_*): message dispatch over each host's
engines, chunk commit and DRR egress, ack processing, duplicate-hint fast
retransmit, RTO backoff and congestion control (OpenLoop, CUBIC, Swift;
global or per-path scope) of chunknet::Transport (src/transport.cpp:84-542,
807-1169; cc.cpp), one warp per source host.

Inputs are each host's event stream: message submissions
(Transport::send_message at time t on a connection) and acks / NACKs /
credits / rts_acks delivered at the host (the cn_ack_rec records the
receive path emits, `aux` = delivery time).  Output is each host's transmit
log (one record per send_chunk, emission order) and per-connection
Transport::Stats.
"""
import ctypes

import numpy as np
import torch

from . import _lib
from .records import ACK_DTYPE

LB = {"oblivious": 0, "p2_rtt": 1, "p2_ecn": 2}
TX_DTYPE = np.dtype([("t", "<i8"), ("msg_id", "<u4"), ("chunk", "<u4"), ("path", "<i4"),
                     ("is_rtx", "<i4"), ("msg_seq", "<u8"), ("conn", "<u4"), ("dst", "<i4")])
SUBMIT_DTYPE = np.dtype([("t", "<i8"), ("len", "<u8"), ("tag", "<u8")])
STATS_DTYPE = np.dtype([(n, "<u8") for n in ("chunks_sent", "chunk_rtx", "fast_rtx", "rtos",
                                             "msgs_sent", "msgs_completed", "backpressured",
                                             "n_log")] +
                       [("srtt", "<i8"), ("rttvar", "<i8"), ("backoff", "<i4"), ("live_msgs", "<i4"),
                        ("cwnd_bytes", "<i8"), ("inflight", "<i8"), ("cwnd_pkts", "<f8"),
                        ("rts_sent", "<u8"), ("decreases", "<u8")])
CC = {"none": 0, "cubic": 1, "swift": 2}
SCOPE = {"global": 0, "per_path": 1}
# transport policy plug-ins (include/chunknet_policy.cuh; cn_tx_config::policy)
POLICY = {"default": 0, "round_robin": 1, "single_path": 2, "test_out_of_range": 3, "user": 100}


class TxEngine:
    """n_conns connections in the reference's creation order (connection c
    draws from RngStream("transport.conn", stream_index0 + c)); src[c] names
    its host -- connections with the same src share the host's engines."""

    def __init__(self, n_conns, *, chunk_bytes, rto_min, commit_ahead, base_rtt_ns, seed,
                 lb="oblivious", max_paths=1, n_paths=None, src=None, dst=None, rto_max=0,
                 dupack_threshold=8, rtx_avoid_prev_path=True, stream_index0=0,
                 chunk_pool=1 << 20, log_cap=1 << 16, cc="none", swift_target_ns=0,
                 drr_quantum=32768, mss=4032, cap_bytes=0, init_cwnd_pkts=2.0, receiver_driven=False,
                 initial_credit=0, credit_quantum=32768, credit_bank_quanta=4, ordered=False,
                 policy="default", engines=1, conn_split=False, cc_scope="global", ecn_as_loss=False,
                 max_inflight_msgs=128, device="cuda"):
        # CN_POLICY_USER lives in the library built with the plug-in
        pol = POLICY[policy] if isinstance(policy, str) else int(policy)
        self._L = L = _lib.user_lib() if pol == POLICY["user"] else _lib.lib()
        c = _lib.TxConfig()
        L.cn_tx_config_default(ctypes.byref(c))
        c.chunk_bytes, c.dupack_threshold = chunk_bytes, dupack_threshold
        c.rtx_avoid_prev_path = 1 if rtx_avoid_prev_path else 0
        c.lb_policy, c.max_paths, c.log_cap = LB[lb], max_paths, log_cap
        c.rto_min, c.rto_max, c.commit_ahead = rto_min, rto_max, commit_ahead
        c.base_rtt_ns, c.seed, c.stream_index0, c.chunk_pool = float(base_rtt_ns), seed, stream_index0, chunk_pool
        c.cc_algo, c.swift_target_ns, c.drr_quantum = CC[cc], swift_target_ns, drr_quantum
        c.mss, c.cap_bytes, c.init_cwnd_pkts = mss, cap_bytes, float(init_cwnd_pkts)
        c.receiver_driven, c.initial_credit = (1 if receiver_driven else 0), initial_credit
        c.credit_quantum, c.credit_bank_quanta = credit_quantum, credit_bank_quanta
        c.ordered = 1 if ordered else 0
        c.policy = pol
        c.engines, c.conn_split = engines, 1 if conn_split else 0
        c.cc_scope, c.ecn_as_loss = SCOPE[cc_scope], 1 if ecn_as_loss else 0
        c.max_inflight_msgs = max_inflight_msgs
        self.device = torch.device(device)
        self.n, self.log_cap = n_conns, log_cap
        arr = lambda v: (ctypes.c_int32 * n_conns)(*[int(x) for x in v]) if v is not None else None  # noqa: E731
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(L.cn_tx_create(ctypes.byref(c), n_conns, arr(src), arr(dst), arr(n_paths),
                                      ctypes.byref(h)), "cn_tx_create", L)
        self._h = h
        self.n_hosts = int(L.cn_tx_n_hosts(h))
        self.host_of = [int(L.cn_tx_conn_host(h, k)) for k in range(n_conns)]
        self.log = torch.zeros(self.n_hosts * log_cap * TX_DTYPE.itemsize, dtype=torch.uint8, device=self.device)
        self.stats = torch.zeros(n_conns * STATS_DTYPE.itemsize, dtype=torch.uint8, device=self.device)

    def close(self):
        if getattr(self, "_h", None):
            self._L.cn_tx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def prepare(self, events, submits, acks):
        """Device copies of the event streams.  events: a flat, time-ordered
        list of (type, conn, index) -- type 0 = submits[index] on connection
        conn, 1 = acks[index] for connection conn -- or the legacy form, a
        list per connection of (type, index) pairs (one connection per
        host)."""
        per_host = [[] for _ in range(self.n_hosts)]
        if events and isinstance(events[0], list):
            for c, evs in enumerate(events):
                per_host[self.host_of[c]].extend((t, c, i) for t, i in evs)
        else:
            for t, c, i in events:
                per_host[self.host_of[c]].append((t, c, i))
        off = np.zeros(self.n_hosts + 1, dtype=np.uint32)
        ev = []
        for h, evs in enumerate(per_host):
            off[h + 1] = off[h] + len(evs)
            ev.extend((int(t) << 62) | (int(c) << 40) | int(i) for t, c, i in evs)
        dev = self.device
        t_off = torch.from_numpy(off.view(np.int32)).to(dev)
        t_ev = torch.from_numpy(np.array(ev if ev else [0], dtype=np.uint64).view(np.int64)).to(dev)
        sub = np.ascontiguousarray(submits, dtype=SUBMIT_DTYPE)
        t_sub = torch.from_numpy(sub.view(np.uint8).copy() if len(sub) else np.zeros(24, np.uint8)).to(dev)
        ak = np.ascontiguousarray(acks, dtype=ACK_DTYPE)
        t_ack = torch.from_numpy(ak.view(np.uint8).copy() if len(ak) else np.zeros(64, np.uint8)).to(dev)
        return (t_off, t_ev, t_sub, t_ack)

    def launch(self, prepared, end_time, stream=None):
        """Enqueue cn_tx_run on prepared device events (no synchronisation)."""
        t_off, t_ev, t_sub, t_ack = prepared
        s = stream or torch.cuda.current_stream(self.device)
        _lib.check(self._L.cn_tx_run(self._h, t_off.data_ptr(), t_ev.data_ptr(), t_sub.data_ptr(),
                                        t_ack.data_ptr(), int(end_time), self.log.data_ptr(),
                                        self.stats.data_ptr(), ctypes.c_void_p(s.cuda_stream)),
                   "cn_tx_run", self._L)

    def run(self, events, submits, acks, end_time, stream=None):
        s = stream or torch.cuda.current_stream(self.device)
        self.launch(self.prepare(events, submits, acks), end_time, s)
        s.synchronize()
        self.check_status()
        return self.stats_np()

    def check_status(self):
        st = ctypes.c_uint()
        self._L.cn_tx_status(self._h, ctypes.byref(st))
        if st.value:
            # 64 = policy contract violation: the reference's logic_error
            raise _lib.ChunknetError(-2 if st.value & 64 else -6, f"tx engine status 0x{st.value:x}")

    def stats_np(self):
        return self.stats.cpu().numpy().view(STATS_DTYPE)

    def log_counts(self):
        out = (ctypes.c_uint32 * self.n_hosts)()
        _lib.check(self._L.cn_tx_log_counts(self._h, out), "cn_tx_log_counts", self._L)
        return list(out)

    def log_np(self, host=0):
        """Host `host`'s transmissions in emission order (connection 0's host
        is host 0)."""
        n = self.log_counts()[host]
        w = self.log_cap * TX_DTYPE.itemsize
        raw = self.log.view(self.n_hosts, w)[host, : min(n, self.log_cap) * TX_DTYPE.itemsize]
        return raw.cpu().numpy().view(TX_DTYPE)

    def conn_state(self, conn):
        cs = _lib.TxConnState()
        _lib.check(self._L.cn_tx_get_conn_state(self._h, conn, ctypes.byref(cs), None, 0), "conn_state", self._L)
        return cs

    def engine_state(self, conn, engine):
        es = _lib.TxEngineState()
        _lib.check(self._L.cn_tx_get_engine_state(self._h, conn, engine, ctypes.byref(es)), "engine_state",
                   self._L)
        return es
