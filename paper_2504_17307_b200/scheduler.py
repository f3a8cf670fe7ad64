"""Multipath chunk scheduler on the device (C ABI cn_sched_*).

Mirrors the reference's path-choice interface: `PathScoreboard`
(include/chunknet/lb.hpp:15-36), `select_path(LbPolicy, board, rng)`
(src/lb.cpp:7-27) and the per-connection `RngStream(seed,
"transport.conn", idx)` (transport.cpp:101), batched: one call produces the
next decisions of many connections at once, bit-identical to calling the
reference sequentially per connection.
"""
import ctypes

import torch

from . import _lib

LB = {"oblivious": 0, "p2_rtt": 1, "p2_ecn": 2}


class PathScheduler:
    def __init__(self, n_conns, max_paths, seed, *, n_paths=None, base_rtt_ns=0.0,
                 stream_name="transport.conn", index0=0, device="cuda"):
        self.device = torch.device(device)
        self.n_conns, self.max_paths = n_conns, max_paths
        np_arr = None
        if n_paths is not None:
            np_arr = (ctypes.c_int32 * n_conns)(*[int(x) for x in n_paths])
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib().cn_sched_create(n_conns, max_paths, np_arr, float(base_rtt_ns),
                                                  seed, stream_name.encode(), index0,
                                                  ctypes.byref(h)), "cn_sched_create")
        self._h = h
        r, e = ctypes.c_void_p(), ctypes.c_void_p()
        _lib.lib().cn_sched_boards(h, ctypes.byref(r), ctypes.byref(e))
        self._rtt_ptr, self._ecn_ptr = r.value, e.value

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().cn_sched_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _board(self, ptr):
        class _H:
            pass
        h = _H()
        h.__cuda_array_interface__ = {"shape": (self.n_conns, self.max_paths), "typestr": "<f8",
                                      "data": (int(ptr), False), "version": 3}
        return torch.as_tensor(h, device=self.device)

    def rtt_scores(self):
        """Device view [n_conns, max_paths] of PathScoreboard::rtt_."""
        return self._board(self._rtt_ptr)

    def ecn_scores(self):
        return self._board(self._ecn_ptr)

    def select(self, policy, count=None, *, conns=None, offsets=None, prev_paths=None,
               rtx_avoid_prev_path=True, out=None, stream=None):
        """Next decisions.  Uniform: `count` per connection -> [n, count].
        Grouped: conns (device u32), offsets (device u32, len+1) -> flat."""
        s = stream or torch.cuda.current_stream(self.device)
        if offsets is None:
            n = self.n_conns if conns is None else conns.numel()
            if out is None:
                out = torch.empty((n, count), dtype=torch.int32, device=self.device)
            ng, uc = n, count
        else:
            ng, uc = offsets.numel() - 1, 0
            if out is None:
                out = torch.empty(int(offsets[-1].item()), dtype=torch.int32, device=self.device)
        ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
        _lib.check(_lib.lib().cn_sched_select(
            self._h, LB[policy] if isinstance(policy, str) else policy,
            1 if rtx_avoid_prev_path else 0, ptr(conns), ptr(offsets), ptr(prev_paths), ng, uc,
            out.data_ptr(), ctypes.c_void_p(s.cuda_stream)), "cn_sched_select")
        return out

    def draws(self, conn, count=None, ns=None, stream=None):
        """RngStream::next_u64 (ns None) or next_below(ns[i]) of one connection."""
        s = stream or torch.cuda.current_stream(self.device)
        if ns is not None:
            ns = ns.to(self.device)
            count = ns.numel()
        out = torch.empty(count, dtype=torch.int64, device=self.device)
        _lib.check(_lib.lib().cn_sched_draws(self._h, conn, ns.data_ptr() if ns is not None else None,
                                             count, out.data_ptr(), ctypes.c_void_p(s.cuda_stream)),
                   "cn_sched_draws")
        return out

    def record(self, conn, path, rtt, ecn, offsets, stream=None):
        """PathScoreboard::record_rtt/record_ecn for grouped samples."""
        s = stream or torch.cuda.current_stream(self.device)
        _lib.check(_lib.lib().cn_sched_record(
            self._h, conn.data_ptr(), path.data_ptr(), rtt.data_ptr(), ecn.data_ptr(),
            offsets.data_ptr(), offsets.numel() - 1, ctypes.c_void_p(s.cuda_stream)), "record")
