"""EQDS receiver-driven pull pacer on the device (C ABI cn_eqds_*): the
reference's EqdsReceiver (src/eqds.cpp:7-104), one per receiving host, run
over each receiver's time-ordered input stream (RTS, chunk arrivals, trimmed
headers); outputs the credit grants and RTS acknowledgements in the order
the reference's callbacks fire them."""
import ctypes

import numpy as np
import torch

from . import _lib

EV_DTYPE = np.dtype([("t", "<i8"), ("type", "<i4"), ("sender", "<i4"), ("arg", "<u8"), ("flag", "<i4"),
                     ("pad", "<i4")])
LOG_DTYPE = np.dtype([("t", "<i8"), ("sender", "<i4"), ("bytes", "<u4"), ("kind", "<i4"), ("pad", "<i4")])
RTS, CHUNK, TRIM = 0, 1, 2


class EqdsConfig(ctypes.Structure):
    _fields_ = [("quantum", ctypes.c_uint32), ("grant_to_idle", ctypes.c_int32), ("tick_ns", ctypes.c_int64),
                ("bank_cap", ctypes.c_int64), ("max_senders", ctypes.c_uint32), ("queue_cap", ctypes.c_uint32),
                ("log_cap", ctypes.c_uint32), ("reserved", ctypes.c_uint32)]


def transport_params(credit_quantum=32768, credit_bank_quanta=4, rate_gbps=100.0, hdr_overhead=64,
                     max_payload=4032):
    """EqdsParams as Transport builds them (transport.cpp:45-73)."""
    pkts = (credit_quantum + max_payload - 1) // max_payload
    tick = int(round((credit_quantum + pkts * hdr_overhead) * 8.0 / rate_gbps))  # Network::ser_ns
    return dict(quantum=credit_quantum, tick_ns=tick, bank_cap=credit_bank_quanta * credit_quantum)


class EqdsPacers:
    def __init__(self, n_receivers, *, quantum=32768, tick_ns=0, bank_cap=0, grant_to_idle=True,
                 max_senders=1024, queue_cap=1 << 14, log_cap=1 << 16, device="cuda"):
        L = _lib.lib()
        c = EqdsConfig()
        L.cn_eqds_config_default(ctypes.byref(c))
        c.quantum, c.tick_ns, c.bank_cap = quantum, tick_ns, bank_cap
        c.grant_to_idle = 1 if grant_to_idle else 0
        c.max_senders, c.queue_cap, c.log_cap = max_senders, queue_cap, log_cap
        self.device = torch.device(device)
        self.n, self.log_cap = n_receivers, log_cap
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(L.cn_eqds_create(ctypes.byref(c), n_receivers, ctypes.byref(h)), "cn_eqds_create")
        self._h = h
        self.log = torch.zeros(n_receivers * log_cap * LOG_DTYPE.itemsize, dtype=torch.uint8, device=self.device)
        self.log_n = torch.zeros(n_receivers, dtype=torch.int32, device=self.device)

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().cn_eqds_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def prepare(self, events, offsets):
        """events: EV_DTYPE grouped by receiver; offsets: n+1 (host arrays)."""
        ev = torch.from_numpy(np.ascontiguousarray(events, dtype=EV_DTYPE).view(np.uint8).reshape(-1)).to(self.device)
        off = torch.from_numpy(np.ascontiguousarray(offsets, dtype=np.uint32).view(np.int32)).to(self.device)
        return ev, off

    def launch(self, prepared, end_time, stream=None):
        ev, off = prepared
        s = stream or torch.cuda.current_stream(self.device)
        _lib.check(_lib.lib().cn_eqds_run(self._h, off.data_ptr(), ev.data_ptr() if ev.numel() else None,
                                          end_time, self.log.data_ptr(), self.log_n.data_ptr(),
                                          ctypes.c_void_p(s.cuda_stream)), "cn_eqds_run")

    def run(self, events, offsets, end_time, stream=None):
        self.launch(self.prepare(events, offsets), end_time, stream)

    def log_np(self, r):
        n = min(int(self.log_n[r].item()), self.log_cap)
        b = self.log[r * self.log_cap * LOG_DTYPE.itemsize:(r * self.log_cap + n) * LOG_DTYPE.itemsize]
        return b.cpu().numpy().view(LOG_DTYPE)

    def status(self, r):
        st, gs = ctypes.c_uint32(), ctypes.c_uint64()
        _lib.check(_lib.lib().cn_eqds_status(self._h, r, ctypes.byref(st), ctypes.byref(gs)), "cn_eqds_status")
        return st.value, gs.value
