"""The drop-in boundary in the shape of chunknet::Transport (C ABI
cn_transport_*, csrc/transport_api.cu; transport.hpp:53-107): one object
owning the device sender engine for every connection it opens and the
device receive path, driven by the caller's clock.

    ep = TransportEndpoint(chunk_bytes=32768, paths=8, lb="p2_rtt", rto_min=..., max_conns=64)
    ep.send_message(src, dst, len, tag, t)      # Transport::send_message at time t
    ep.handle_acks(ack_records)                 # acks / NACKs delivered at the senders (aux = time)
    ep.advance(until)                           # run the sender up to `until`
    tx, conn = ep.poll_transmissions()          # every send_chunk since the last poll
    ep.handle_data(hdrs_dev, payload_dev)       # Transport::handle_packet for a batch of data packets
    acks = ep.poll_acks(); cpls = ep.poll_completions(); st = ep.stats()
"""
import ctypes

import numpy as np
import torch

from . import _lib
from .records import ACK_DTYPE, CPL_DTYPE
from .sender import LB, TX_DTYPE

CC = {"none": 0, "cubic": 1, "swift": 2}


class TransportConfigC(ctypes.Structure):
    i32, u32, i64, u64, f64 = ctypes.c_int32, ctypes.c_uint32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
    _fields_ = [("engines", i32), ("conn_split", i32), ("paths", i32), ("chunk_bytes", u32),
                ("lb", i32), ("reliability", i32), ("receiver_driven", i32), ("max_inflight_msgs", i32),
                ("rto_min", i64), ("rto_max", i64), ("drr_quantum", u32), ("rtx_avoid_prev_path", i32),
                ("dupack_threshold", i32), ("carry_payload", i32), ("initial_credit", i64),
                ("credit_quantum", u32), ("credit_bank_quanta", i32), ("cc_algo", i32), ("cc_scope", i32),
                ("mss", i64), ("cap_bytes", i64), ("ecn_as_loss", i32), ("pad0", i32),
                ("swift_target_ns", i64), ("init_cwnd_pkts", f64), ("base_rtt_ns", f64),
                ("commit_ahead", i64), ("max_conns", u32), ("max_batch", u32), ("log_cap", u32),
                ("policy", i32), ("chunk_pool", u64), ("arena_bytes", u64), ("max_conns_per_host", u32),
                ("pad_mcph", u32)]


STATS_FIELDS = ["msgs_sent", "msgs_completed", "backpressured", "chunks_sent", "chunk_rtx", "fast_rtx", "rtos",
                "acks_sent", "nacks_sent", "rts_sent", "credit_pkts", "delivered_msgs"]


class StatsC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in STATS_FIELDS]


def _setup(L):
    vp, i32, i64, u32, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64
    L.cn_transport_config_default.argtypes = [vp]
    L.cn_transport_config_default.restype = None
    L.cn_transport_create.argtypes = [vp, u64, ctypes.POINTER(vp)]
    L.cn_transport_destroy.argtypes = [vp]
    L.cn_transport_destroy.restype = None
    L.cn_transport_send_message.argtypes = [vp, i32, i32, u64, u64, i64]
    L.cn_transport_handle_acks.argtypes = [vp, vp, u32]
    L.cn_transport_advance.argtypes = [vp, i64, vp]
    L.cn_transport_poll_transmissions.argtypes = [vp, vp, u64, vp]
    L.cn_transport_poll_transmissions.restype = i64
    L.cn_transport_handle_data.argtypes = [vp, vp, vp, u64, u32, vp]
    L.cn_transport_handle_data_psn.argtypes = [vp, vp, vp, vp, u64, u32, vp]
    L.cn_transport_handle_data_msgdata.argtypes = [vp, vp, vp, vp, u32, vp]
    L.cn_transport_poll_acks.argtypes = [vp, vp, u64]
    L.cn_transport_poll_acks.restype = i64
    L.cn_transport_poll_completions.argtypes = [vp, vp, u64]
    L.cn_transport_poll_completions.restype = i64
    L.cn_transport_stats.argtypes = [vp, vp]
    L.cn_transport_conn_index.argtypes = [vp, i32, i32]
    L.cn_transport_open_conn.argtypes = [vp, i32, i32, i32]
    L.cn_transport_outstanding_bytes.argtypes = [vp, i32, i32]
    L.cn_transport_outstanding_bytes.restype = i64
    for f, rt in (("path_inflight", i64), ("window_available", i64)):
        getattr(L, f"cn_transport_{f}").argtypes = [vp, i32, i32, i32]
        getattr(L, f"cn_transport_{f}").restype = rt
    L.cn_transport_conn_credit.argtypes = [vp, i32, i32]
    L.cn_transport_conn_credit.restype = i64
    for f, rt in (("engine_inflight_msgs", i32), ("engine_dispatched", u64), ("engine_gauge", i64)):
        getattr(L, f"cn_transport_{f}").argtypes = [vp, i32, i32]
        getattr(L, f"cn_transport_{f}").restype = rt


class TransportEndpoint:
    def __init__(self, *, chunk_bytes=32768, paths=1, lb="oblivious", rto_min, rto_max=0, seed=1,
                 commit_ahead=0, base_rtt_ns=10000.0, cc="none", swift_target_ns=0, dupack_threshold=8,
                 rtx_avoid_prev_path=True, carry_payload=True, max_conns=64, max_batch=1 << 16,
                 log_cap=1 << 16, chunk_pool=1 << 20, arena_bytes=64 << 20, receiver_driven=False,
                 initial_credit=-1, credit_quantum=32768, credit_bank_quanta=4, policy=0,
                 reliability="selective", engines=1, conn_split=False, cc_scope="global", ecn_as_loss=False,
                 cap_bytes=0, max_conns_per_host=0, device="cuda"):
        L = _lib.lib()
        _setup(L)
        c = TransportConfigC()
        L.cn_transport_config_default(ctypes.byref(c))
        c.chunk_bytes, c.paths, c.lb = chunk_bytes, paths, LB[lb]
        c.rto_min, c.rto_max, c.commit_ahead, c.base_rtt_ns = rto_min, rto_max, commit_ahead, float(base_rtt_ns)
        c.cc_algo, c.swift_target_ns = CC[cc], swift_target_ns
        c.dupack_threshold, c.rtx_avoid_prev_path = dupack_threshold, 1 if rtx_avoid_prev_path else 0
        c.carry_payload = 1 if carry_payload else 0
        c.max_conns, c.max_batch, c.log_cap = max_conns, max_batch, log_cap
        c.chunk_pool, c.arena_bytes = chunk_pool, arena_bytes
        c.receiver_driven, c.initial_credit = (1 if receiver_driven else 0), initial_credit
        c.credit_quantum, c.credit_bank_quanta, c.policy = credit_quantum, credit_bank_quanta, policy
        c.reliability = {"selective": 0, "ordered": 1}[reliability]
        c.engines, c.conn_split = engines, 1 if conn_split else 0
        c.cc_scope = {"global": 0, "per_path": 1}[cc_scope]
        c.ecn_as_loss, c.cap_bytes, c.max_conns_per_host = 1 if ecn_as_loss else 0, cap_bytes, max_conns_per_host
        self.device = torch.device(device)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(L.cn_transport_create(ctypes.byref(c), seed, ctypes.byref(h)), "cn_transport_create")
        self._h = h
        self._L = L

    def close(self):
        if getattr(self, "_h", None):
            self._L.cn_transport_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def send_message(self, src, dst, length, tag, t):
        rc = self._L.cn_transport_send_message(self._h, src, dst, length, tag, t)
        _lib.check(rc if rc < 0 else 0, "send_message")
        return rc == 1

    def handle_acks(self, acks):
        a = np.ascontiguousarray(acks, dtype=ACK_DTYPE)
        _lib.check(self._L.cn_transport_handle_acks(self._h, a.ctypes.data_as(ctypes.c_void_p), len(a)),
                   "handle_acks")

    def advance(self, until, stream=None):
        s = stream or torch.cuda.current_stream(self.device)
        _lib.check(self._L.cn_transport_advance(self._h, until, ctypes.c_void_p(s.cuda_stream)), "advance")

    def poll_transmissions(self, cap=1 << 20):
        """(TX_DTYPE records, connection index per record) since the last poll."""
        out = np.zeros(cap, dtype=TX_DTYPE)
        conn = np.zeros(cap, dtype=np.int32)
        n = self._L.cn_transport_poll_transmissions(self._h, out.ctypes.data_as(ctypes.c_void_p), cap,
                                                    conn.ctypes.data_as(ctypes.c_void_p))
        _lib.check(n if n < 0 else 0, "poll_transmissions")
        return out[: min(n, cap)], conn[: min(n, cap)]

    def handle_data(self, hdrs, payload=None, stride=4032, stream=None, psn=None, msg_data=None):
        """psn: device int64 conn_psn per packet (ordered reliability);
        msg_data: device int64 message-data pointer per packet (Packet::msg_data,
        the send_message_data path) instead of a payload buffer."""
        s = stream or torch.cuda.current_stream(self.device)
        n = hdrs.numel() // 64
        if msg_data is not None:
            _lib.check(self._L.cn_transport_handle_data_msgdata(
                self._h, hdrs.data_ptr(), psn.data_ptr() if psn is not None else None, msg_data.data_ptr(), n,
                ctypes.c_void_p(s.cuda_stream)), "handle_data_msgdata")
            return
        pl = payload.data_ptr() if payload is not None else None
        _lib.check(self._L.cn_transport_handle_data_psn(self._h, hdrs.data_ptr(),
                                                         psn.data_ptr() if psn is not None else None, pl,
                                                         stride, n, ctypes.c_void_p(s.cuda_stream)),
                   "handle_data")

    def poll_acks(self):
        n = self._L.cn_transport_poll_acks(self._h, None, 0)
        out = np.zeros(max(n, 1), dtype=ACK_DTYPE)
        self._L.cn_transport_poll_acks(self._h, out.ctypes.data_as(ctypes.c_void_p), n)
        return out[:n]

    def poll_completions(self):
        n = self._L.cn_transport_poll_completions(self._h, None, 0)
        out = np.zeros(max(n, 1), dtype=CPL_DTYPE)
        self._L.cn_transport_poll_completions(self._h, out.ctypes.data_as(ctypes.c_void_p), n)
        return out[:n]

    def stats(self):
        st = StatsC()
        _lib.check(self._L.cn_transport_stats(self._h, ctypes.byref(st)), "stats")
        return {n: int(getattr(st, n)) for n in STATS_FIELDS}

    def open_conn(self, src, dst, n_paths):
        """conn_to with min(paths, path_count(src, dst)) from the caller's topology."""
        k = int(self._L.cn_transport_open_conn(self._h, src, dst, n_paths))
        _lib.check(k if k < 0 else 0, "open_conn")
        return k

    def conn_index(self, src, dst):
        return int(self._L.cn_transport_conn_index(self._h, src, dst))

    def outstanding_bytes(self, src, dst):
        return int(self._L.cn_transport_outstanding_bytes(self._h, src, dst))

    # the rest of Transport's introspection (transport.hpp:101-107)
    def path_inflight(self, src, dst, path):
        return int(self._L.cn_transport_path_inflight(self._h, src, dst, path))

    def window_available(self, src, dst, path):
        return int(self._L.cn_transport_window_available(self._h, src, dst, path))

    def conn_credit(self, src, dst):
        return int(self._L.cn_transport_conn_credit(self._h, src, dst))

    def engine_inflight_msgs(self, host, engine=0):
        return int(self._L.cn_transport_engine_inflight_msgs(self._h, host, engine))

    def engine_dispatched(self, host, engine=0):
        return int(self._L.cn_transport_engine_dispatched(self._h, host, engine))

    def engine_gauge(self, host, engine=0):
        return int(self._L.cn_transport_engine_gauge(self._h, host, engine))
