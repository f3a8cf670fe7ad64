"""The reference's packet trace format (experiment.cpp:18-40 trace_line over
network.hpp:30-35 TraceEvent) on the device: receive-path records become
trace records, and a batch of records is rendered to TSV text in parallel
(csrc/trace.cu), byte-identical to the reference's trace.tsv.

    t \\t event \\t link_id \\t src>dst:path_id \\t csn \\t kind[,rtx][,ecn][,trim][,last]
"""
import ctypes

import numpy as np
import torch

from . import _lib

TRACE_DTYPE = np.dtype([("t", "<i8"), ("link_id", "<i4"), ("src", "<i4"), ("dst", "<i4"),
                        ("path_id", "<i4"), ("csn", "u1"), ("event", "u1"), ("kind", "u1"),
                        ("flags", "u1"), ("reserved", "<u4")])
EVENTS = ["deliver", "drop", "trim", "loss", "hdr_drop"]
KINDS = ["data", "ack", "nack", "credit", "rts", "rts_ack"]
FLAGS = [("rtx", 1), ("ecn", 2), ("trim", 4), ("last", 8)]


def parse_tsv(text):
    """trace.tsv text -> TRACE_DTYPE records (the inverse of the writer)."""
    lines = text.splitlines() if isinstance(text, str) else text.decode().splitlines()
    out = np.zeros(len(lines), dtype=TRACE_DTYPE)
    for i, ln in enumerate(lines):
        t, ev, link, ends, csn, kf = ln.split("\t")
        sd, path = ends.split(":")
        src, dst = sd.split(">")
        parts = kf.split(",")
        fl = 0
        for name, bit in FLAGS:
            if name in parts[1:]:
                fl |= bit
        out[i] = (int(t), int(link), int(src), int(dst), int(path), int(csn), EVENTS.index(ev),
                  KINDS.index(parts[0]), fl, 0)
    return out


def _dev(x, device):
    if isinstance(x, torch.Tensor):
        return x.to(device).contiguous()
    a = np.ascontiguousarray(x)
    return torch.from_numpy(a.view(np.uint8).reshape(-1)).to(device)


def format_tsv(recs, device="cuda", stream=None):
    """Render trace records (TRACE_DTYPE array or device uint8 tensor of
    32-B records) -> bytes, on the device."""
    L = _lib.lib()
    d = _dev(recs, device)
    n = d.numel() // TRACE_DTYPE.itemsize
    cap = L.cn_trace_tsv_bound(n)
    out = torch.empty(max(1, cap), dtype=torch.uint8, device=device)
    scratch = torch.empty(max(8, L.cn_trace_scratch_bytes(n)), dtype=torch.uint8, device=device)
    ln = torch.zeros(1, dtype=torch.int64, device=device)
    s = stream or torch.cuda.current_stream(device)
    _lib.check(L.cn_trace_format(d.data_ptr() if n else None, n, out.data_ptr(), cap, ln.data_ptr(),
                                 scratch.data_ptr(), ctypes.c_void_p(s.cuda_stream)), "cn_trace_format")
    k = int(ln.item())
    return bytes(out[:k].cpu().numpy())


def from_packets(hdrs, times=None, event="deliver", link_id=-1, device="cuda", stream=None):
    """cn_pkt_hdr records (device uint8 [n*64]) -> device trace records."""
    L = _lib.lib()
    n = hdrs.numel() // 64
    out = torch.empty(max(1, n) * TRACE_DTYPE.itemsize, dtype=torch.uint8, device=device)
    s = stream or torch.cuda.current_stream(device)
    tp = times.data_ptr() if times is not None else None
    _lib.check(L.cn_trace_from_packets(hdrs.data_ptr(), tp, n, EVENTS.index(event), link_id, out.data_ptr(),
                                       ctypes.c_void_p(s.cuda_stream)), "cn_trace_from_packets")
    return out[: n * TRACE_DTYPE.itemsize]


def from_acks(acks, event="deliver", link_id=-1, device="cuda", stream=None):
    """cn_ack_rec records (device uint8 [n*64], aux = delivery time) -> device trace records."""
    L = _lib.lib()
    n = acks.numel() // 64
    out = torch.empty(max(1, n) * TRACE_DTYPE.itemsize, dtype=torch.uint8, device=device)
    s = stream or torch.cuda.current_stream(device)
    _lib.check(L.cn_trace_from_acks(acks.data_ptr(), n, EVENTS.index(event), link_id, out.data_ptr(),
                                    ctypes.c_void_p(s.cuda_stream)), "cn_trace_from_acks")
    return out[: n * TRACE_DTYPE.itemsize]
