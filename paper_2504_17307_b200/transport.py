"""Host-side mirror of the reference transport interface over the C ABI.

The reference (/root/reference/proj/include/chunknet/transport.hpp:60-107)
is one `Transport` object managing every host endpoint, driven by packet
delivery (`handle_packet`, transport.cpp:565) and reporting delivered
messages through `set_on_complete(CompleteFn)` (transport.hpp:77-79).
This module keeps those names.  Packets arrive in batches of 64-byte
header records (cn_pkt_hdr) plus a payload staging buffer, both resident
in device memory; the receive path runs entirely in the sm_100a kernels of
libchunknet_b200.so (csrc/rx.cu).  There is no CPU fallback.
"""
import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .records import ACK_DTYPE, CPL_DTYPE, PKT_DTYPE

MAX_PAYLOAD = 4032  # NetParams mtu 4096 - hdr_overhead 64 (network.hpp:25-26)


@dataclass
class TransportConfig:
    """chunknet::TransportConfig (transport.hpp:23-51); same names/defaults."""
    engines: int = 1
    conn_split: bool = False
    paths: int = 1
    chunk_bytes: int = 32768
    lb: str = "oblivious"
    reliability: str = "selective"
    receiver_driven: bool = False
    rto_min: int = 0
    rto_max: int = 0
    max_inflight_msgs: int = 128
    drr_quantum: int = 32768
    rtx_avoid_prev_path: bool = True
    dupack_threshold: int = 8
    carry_payload: bool = False
    initial_credit: int = -1
    credit_quantum: int = 32768
    credit_bank_quanta: int = 4


@dataclass
class Stats:
    """Receive-side subset of Transport::Stats (transport.hpp:62-75)."""
    msgs_completed: int = 0
    acks_sent: int = 0
    nacks_sent: int = 0
    pkts_accepted: int = 0
    bytes_accepted: int = 0


class RxBatch:
    """Device outputs of one cn_rx_batch call."""

    def __init__(self, acks, completions, result):
        self.acks = acks                # torch.uint8 [n_acks, 64] on device
        self.completions = completions  # torch.uint8 [n_cpl, 64] on device
        self.result = result            # _lib.RxResult (host copy)

    def acks_np(self):
        return self.acks.cpu().numpy().reshape(-1).view(ACK_DTYPE)

    def completions_np(self):
        return self.completions.cpu().numpy().reshape(-1).view(CPL_DTYPE)


class Transport:
    """Receive side of chunknet::Transport on one B200 (selective mode,
    fixed-size chunking as DefaultPolicy, policy.hpp:70-97)."""

    REDUCE = {None: 0, "none": 0, "sum_f32": 1, "sum_bf16": 2}

    def __init__(self, cfg=None, seed=0, *, device="cuda", max_conns=1024, max_msgs=4096,
                 chunk_pool=1 << 22, arena_bytes=1 << 30, max_batch=1 << 20, reduce=None,
                 max_posts=0, pipeline=False):
        self.cfg = cfg or TransportConfig()
        if self.cfg.reliability not in ("selective", "ordered"):
            raise _lib.ChunknetError(-1, "reliability is 'selective' or 'ordered'")
        if self.cfg.receiver_driven:
            raise _lib.ChunknetError(-6, "receiver-driven (EQDS) pacing is host-side")
        self.seed = seed
        self.device = torch.device(device)
        if self.device.type != "cuda":
            raise _lib.ChunknetError(-1, "the transport runs on a CUDA device only")
        L = _lib.lib()
        rc = _lib.RxConfig()
        L.cn_rx_config_default(ctypes.byref(rc))
        rc.chunk_bytes = self.cfg.chunk_bytes
        rc.max_payload = MAX_PAYLOAD
        rc.max_conns = max_conns
        rc.max_msgs = max_msgs
        rc.chunk_pool = chunk_pool
        rc.arena_bytes = arena_bytes if self.cfg.carry_payload else 0
        rc.max_batch = max_batch
        rc.carry_payload = 1 if self.cfg.carry_payload else 0
        rc.reduce_op = self.REDUCE[reduce]
        rc.max_posts = max_posts
        rc.ordered = 1 if self.cfg.reliability == "ordered" else 0
        rc.pipeline = 1 if pipeline else 0
        self.pipeline = bool(pipeline)
        self._rxcfg = rc
        with torch.cuda.device(self.device):
            h = ctypes.c_void_p()
            _lib.check(L.cn_rx_create(ctypes.byref(rc), ctypes.byref(h)), "cn_rx_create")
        self._h = h
        self._on_complete = None
        self._stats = Stats()
        self._result = torch.zeros(24, dtype=torch.uint8, device=self.device)
        self._pinned = torch.zeros(24, dtype=torch.uint8).pin_memory()
        self._acks = torch.empty(0, dtype=torch.uint8, device=self.device)
        self._cpls = torch.empty(0, dtype=torch.uint8, device=self.device)
        self._index_base = 0

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().cn_rx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- reference API names -------------------------------------------
    def set_on_complete(self, fn):
        """fn(tag, src, dst, len, pkt_index, data) -- data is a device uint8
        view of the reassembled message (None unless carry_payload), valid
        during the callback like the reference's (transport.cpp:797-802)."""
        self._on_complete = fn

    def stats(self):
        return self._stats

    def config(self):
        return self.cfg

    def reset(self, stream=None):
        s = stream or torch.cuda.current_stream(self.device)
        _lib.check(_lib.lib().cn_rx_reset(self._h, ctypes.c_void_p(s.cuda_stream)), "reset")
        self._index_base = 0

    def _ensure(self, n):
        need = (n + 16) * 64
        if self._acks.numel() < need:
            self._acks = torch.empty(need, dtype=torch.uint8, device=self.device)
        if self._cpls.numel() < need:
            self._cpls = torch.empty(need, dtype=torch.uint8, device=self.device)

    def rx_batch_async(self, hdrs, payload, stride=MAX_PAYLOAD, stream=None, n=None, psn=None, msg_data=None,
                       offsets=None):
        """Enqueue the receive path for a batch; no host synchronisation.
        A pipelined receiver (pipeline=True) leaves this batch's payload
        scatter running beside the next batch (flush() joins it).
        hdrs: device uint8 [n*64] (cn_pkt_hdr records, arrival order);
        payload: device buffer, packet i's payload at i*stride; psn: device
        uint64 conn_psn per packet (ordered reliability only); offsets: device
        int64 per packet -- packed payloads, packet i at payload + offsets[i];
        msg_data: device
        int64 per packet, its message's data pointer (Packet::msg_data, the
        send_message_data path) -- replaces payload / stride."""
        n = hdrs.numel() // 64 if n is None else n
        self._ensure(n)
        s = stream or torch.cuda.current_stream(self.device)
        if offsets is not None:  # packed payloads: packet i at payload + offsets[i]
            _lib.check(_lib.lib().cn_rx_batch_packed(
                self._h, hdrs.data_ptr(), psn.data_ptr() if psn is not None else None,
                payload.data_ptr() if payload is not None else None, offsets.data_ptr(), n,
                self._acks.data_ptr(), n + 16, self._cpls.data_ptr(), n + 16, self._result.data_ptr(),
                ctypes.c_void_p(s.cuda_stream)), "cn_rx_batch_packed")
            return n
        if msg_data is not None:
            _lib.check(_lib.lib().cn_rx_batch_msgdata(
                self._h, hdrs.data_ptr(), psn.data_ptr() if psn is not None else None, msg_data.data_ptr(), n,
                self._acks.data_ptr(), n + 16, self._cpls.data_ptr(), n + 16, self._result.data_ptr(),
                ctypes.c_void_p(s.cuda_stream)), "cn_rx_batch_msgdata")
            return n
        pl = payload.data_ptr() if payload is not None else None
        if payload is not None and stride == 0 and not self.cfg.carry_payload:
            pl = None
        if self.cfg.reliability == "ordered":
            _lib.check(_lib.lib().cn_rx_batch_psn(
                self._h, hdrs.data_ptr(), psn.data_ptr() if psn is not None else None, pl, stride, n,
                self._acks.data_ptr(), n + 16, self._cpls.data_ptr(), n + 16, self._result.data_ptr(),
                ctypes.c_void_p(s.cuda_stream)), "cn_rx_batch_psn")
            return n
        _lib.check(_lib.lib().cn_rx_batch(
            self._h, hdrs.data_ptr(), pl, stride, n, self._acks.data_ptr(), n + 16,
            self._cpls.data_ptr(), n + 16, self._result.data_ptr(),
            ctypes.c_void_p(s.cuda_stream)), "cn_rx_batch")
        return n

    def handle_packets(self, hdrs, payload=None, stride=MAX_PAYLOAD, stream=None, psn=None, msg_data=None,
                       offsets=None):
        """Batched Transport::handle_packet for data packets: runs the device
        receive path, returns the ack records in emission order, and fires
        the completion callback for every delivered message."""
        s = stream or torch.cuda.current_stream(self.device)
        n = self.rx_batch_async(hdrs, payload, stride, s, psn=psn, msg_data=msg_data, offsets=offsets)
        if self.pipeline:  # this call's contract: the delivered bytes are final
            self.flush(s)
        self._pinned.copy_(self._result, non_blocking=True)
        s.synchronize()
        res = _lib.RxResult.from_buffer_copy(bytes(self._pinned.numpy()))
        if res.status:
            raise _lib.ChunknetError(-6 if res.status & 3 else -7,
                                     f"rx batch status flags 0x{res.status:x}")
        acks = self._acks[: res.n_acks * 64].view(res.n_acks, 64)
        cpls = self._cpls[: res.n_completions * 64].view(res.n_completions, 64)
        n_nacks = 0
        if res.n_acks:  # NACK records (trimmed headers) share the ack stream
            fo = ACK_DTYPE.fields["flags"][1]
            n_nacks = int(((acks[:, fo] & 4) != 0).sum().item())
        self._stats.acks_sent += res.n_acks - n_nacks
        self._stats.nacks_sent += n_nacks
        self._stats.msgs_completed += res.n_completions
        self._stats.pkts_accepted += res.n_copied
        self._stats.bytes_accepted += res.bytes_copied
        out = RxBatch(acks, cpls, res)
        if self._on_complete is not None and res.n_completions:
            arena = self.arena()
            for c in out.completions_np():
                data = None
                if self.cfg.carry_payload and arena is not None:
                    off = int(c["buf_offset"])
                    data = arena[off: off + int(c["len"])]
                self._on_complete(int(c["tag"]), int(c["src"]), int(c["dst"]), int(c["len"]),
                                  self._index_base + int(c["pkt_index"]), data)
        self._index_base += n
        return out

    def flush(self, stream=None):
        """Pipelined receivers: join the outstanding payload scatter (cn_rx_flush)."""
        s = stream or torch.cuda.current_stream(self.device)
        _lib.check(_lib.lib().cn_rx_flush(self._h, ctypes.c_void_p(s.cuda_stream)), "cn_rx_flush")

    def post(self, tag, buf, stream=None):
        """Scatter (or, in reduce mode, accumulate) the message with caller
        tag `tag` into the device tensor `buf` instead of the arena."""
        s = stream or torch.cuda.current_stream(self.device)
        _lib.check(_lib.lib().cn_rx_post(self._h, tag, buf.data_ptr(), buf.numel() * buf.element_size(),
                                          ctypes.c_void_p(s.cuda_stream)), "cn_rx_post")

    def completions_np(self, n):
        """The first n completion records of the last batch (host copy)."""
        return self._cpls[: n * 64].cpu().numpy().view(CPL_DTYPE)

    def set_profiling(self, enable=True):
        _lib.lib().cn_rx_set_profiling(self._h, 1 if enable else 0)

    def kernel_profile(self, reset=True):
        """{kernel name: accumulated ms}, batches -- CUDA events on the launch stream."""
        L = _lib.lib()
        ms = (ctypes.c_double * 16)()
        nb = ctypes.c_uint64()
        k = L.cn_rx_profile(self._h, ms, 16, ctypes.byref(nb), 1 if reset else 0)
        return {L.cn_rx_kernel_name(i).decode(): ms[i] for i in range(k)}, nb.value

    def last_launches(self):
        return _lib.lib().cn_rx_last_launches(self._h)

    def usage(self):
        """Ring occupancy (cn_rx_get_usage): chunk-pool entries and arena
        blocks held by undelivered messages, capacities, totals allocated."""
        u = _lib.RxUsage()
        _lib.check(_lib.lib().cn_rx_get_usage(self._h, ctypes.byref(u)), "cn_rx_get_usage")
        return {k: getattr(u, k) for k, _ in u._fields_}

    def arena(self):
        """Device uint8 view of the reassembly arena (cn_rx_arena)."""
        ptr = _lib.lib().cn_rx_arena(self._h)
        if not ptr:
            return None
        nbytes = _lib.lib().cn_rx_arena_bytes(self._h)
        return _device_u8_view(ptr, nbytes, self.device)


def _device_u8_view(ptr, nbytes, device):
    """Zero-copy torch view of device memory owned by the C library."""
    class _Holder:
        pass
    h = _Holder()
    h.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                  "data": (int(ptr), False), "version": 3}
    return torch.as_tensor(h, device=device)


def encode_header(conn_id, msg_id, csn, last_chunk=False, reserved=0):
    """encode_header (src/wire.cpp:5-14); raises on msg_id > 127."""
    h = _lib.ControlHeader(conn_id, msg_id, csn, 1 if last_chunk else 0, reserved)
    out = ctypes.c_uint32()
    _lib.check(_lib.lib().cn_encode_header(ctypes.byref(h), ctypes.byref(out)),
               "encode_header")
    return out.value


def decode_header(word):
    """decode_header (src/wire.cpp:16-24) -> (conn_id, msg_id, csn, last, reserved)."""
    h = _lib.ControlHeader()
    _lib.lib().cn_decode_header(word, ctypes.byref(h))
    return (h.conn_id, h.msg_id, h.csn, bool(h.last_chunk), h.reserved)


def csn_before(a, b, base, width):
    """csn_before (src/wire.cpp:26-40) over SeqWindow{base, width}."""
    out = ctypes.c_int()
    _lib.check(_lib.lib().cn_csn_before(a, b, base, width, ctypes.byref(out)), "csn_before")
    return bool(out.value)


def to_device_records(arr, device="cuda"):
    """numpy structured records -> flat device uint8 tensor."""
    raw = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
    return torch.from_numpy(raw.copy()).to(device)


__all__ = ["TransportConfig", "Transport", "Stats", "RxBatch", "encode_header",
           "decode_header", "csn_before", "to_device_records", "PKT_DTYPE", "ACK_DTYPE",
           "CPL_DTYPE", "MAX_PAYLOAD"]
