"""ctypes wrapper of oracle/liboracle.so (the C restatement) -- TEST INFRA.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this module; the product path (paper_2504_17307_b200) never does.
"""
import ctypes
import os
import subprocess

import numpy as np

from .records import ACK_DTYPE, CPL_DTYPE, PKT_DTYPE

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

_lib = None


class RxCounts(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "n_acks", "n_completions", "n_nacks", "arena_used", "pkts_accepted",
        "bytes_accepted")]


def build():
    subprocess.run(["make", "-C", HERE, "oracle"], check=True,
                   stdout=subprocess.DEVNULL)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        vp, u64, i64, i32, u32 = (ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64,
                                  ctypes.c_int, ctypes.c_uint32)
        L.orc_rx_create.restype = vp
        L.orc_rx_create.argtypes = [u32, i32]
        L.orc_rx_destroy.argtypes = [vp]
        L.orc_rx_set_ordered.argtypes = [vp, i32, vp]
        L.orc_rx_set_ordered.restype = None
        L.orc_rx_batch.argtypes = [vp, vp, vp, u64, u64, u32, vp, u64, vp, u64, vp, u64,
                                   ctypes.POINTER(RxCounts)]
        L.orc_pattern_bytes.argtypes = [u64, u64, vp]
        L.orc_fill_staging.argtypes = [vp, u64, u32, vp, u64]
        L.orc_select_paths.argtypes = [i32, i32, vp, vp, u64, ctypes.c_char_p, i64, u64, vp]
        L.orc_ring_allreduce.argtypes = [i32, i32, u64, vp, vp]
        L.orc_ring_allreduce_q.argtypes = [i32, i32, u64, vp, vp, u64]
        L.orc_rng_u64_seq.argtypes = [u64, ctypes.c_char_p, i64, u64, vp]
        L.orc_next_below_seq.argtypes = [u64, ctypes.c_char_p, i64, vp, u64, vp]
        L.orc_next_double_seq.argtypes = [u64, ctypes.c_char_p, i64, u64, vp]
        L.orc_fnv1a64.restype = u64
        L.orc_libm.argtypes = [i32, i32, vp, vp, u64]
        L.orc_libm.restype = None
        L.orc_fnv1a64.argtypes = [ctypes.c_char_p]
        L.orc_splitmix64.restype = u64
        L.orc_splitmix64.argtypes = [u64]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class OracleRx:
    """Sequential restatement of the reference receive path."""

    def __init__(self, max_payload=4032, carry_payload=True, ordered=False):
        self.h = lib().orc_rx_create(max_payload, 1 if carry_payload else 0)
        self.carry = carry_payload
        self.ordered = ordered

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_rx_destroy(self.h)
            self.h = None

    def batch(self, hdrs, payload=None, stride=4032, index_base=0, arena_bytes=None, psn=None):
        hdrs = np.ascontiguousarray(hdrs, dtype=PKT_DTYPE)
        n = len(hdrs)
        psn_a = np.ascontiguousarray(psn if psn is not None else np.zeros(n), dtype=np.uint64)
        lib().orc_rx_set_ordered(self.h, 1 if self.ordered else 0, _ptr(psn_a) if self.ordered else None)
        acks = np.zeros(n + 16, dtype=ACK_DTYPE)
        cpls = np.zeros(n + 16, dtype=CPL_DTYPE)
        if arena_bytes is None:
            lens = {(int(t), int(l)) for t, l in zip(hdrs["msg_tag"], hdrs["msg_len"])}
            arena_bytes = 2 * sum(((l + 15) // 16) * 16 for _, l in lens) + 64
        arena = np.zeros(max(arena_bytes, 1), dtype=np.uint8)
        c = RxCounts()
        pl = _ptr(payload) if payload is not None else None
        rc = lib().orc_rx_batch(self.h, _ptr(hdrs), pl, stride, n, index_base,
                                _ptr(acks), len(acks), _ptr(cpls), len(cpls),
                                _ptr(arena), arena.nbytes, ctypes.byref(c))
        if rc != 0:
            raise RuntimeError(f"oracle rx status {rc}")
        return (acks[: c.n_acks].copy(), cpls[: c.n_completions].copy(),
                arena[: c.arena_used], c)


def pattern_bytes(n, seed):
    out = np.zeros(max(n, 1), dtype=np.uint8)
    lib().orc_pattern_bytes(n, seed, _ptr(out))
    return out[:n]


def fill_staging(hdrs, max_pl=4032, stride=4032):
    hdrs = np.ascontiguousarray(hdrs, dtype=PKT_DTYPE)
    st = np.zeros(len(hdrs) * stride + 16, dtype=np.uint8)
    lib().orc_fill_staging(_ptr(hdrs), len(hdrs), max_pl, _ptr(st), stride)
    return st


def select_paths(policy, rtt, ecn, seed, name, index, count):
    pol = {"oblivious": 0, "p2_rtt": 1, "p2_ecn": 2}[policy]
    rtt = np.ascontiguousarray(rtt, dtype=np.float64)
    ecn = np.ascontiguousarray(ecn, dtype=np.float64)
    out = np.zeros(count, dtype=np.int32)
    lib().orc_select_paths(pol, len(rtt), _ptr(rtt), _ptr(ecn), seed, name.encode(),
                           index, count, _ptr(out))
    return out


def ring_allreduce(x, quantum=1):
    """x: [n_ranks, count] float32 or uint16 (bf16 bits) -> allreduced [count].
    Segment boundaries are rounded down to multiples of `quantum` elements."""
    x = np.ascontiguousarray(x)
    dtype = 0 if x.dtype == np.float32 else 1
    assert x.dtype in (np.float32, np.uint16)
    out = np.zeros(x.shape[1], dtype=x.dtype)
    lib().orc_ring_allreduce_q(dtype, x.shape[0], x.shape[1], _ptr(x), _ptr(out), quantum)
    return out


def fnv1a64(s):
    return lib().orc_fnv1a64(s.encode())


def splitmix64(x):
    return lib().orc_splitmix64(x)


def rng_u64(seed, name, index, count):
    out = np.zeros(count, dtype=np.uint64)
    lib().orc_rng_u64_seq(seed, name.encode(), index, count, _ptr(out))
    return out


def next_below(seed, name, index, ns):
    ns = np.ascontiguousarray(ns, dtype=np.uint64)
    out = np.zeros(len(ns), dtype=np.uint64)
    lib().orc_next_below_seq(seed, name.encode(), index, _ptr(ns), len(ns), _ptr(out))
    return out


def next_double(seed, name, index, count):
    out = np.zeros(count, dtype=np.float64)
    lib().orc_next_double_seq(seed, name.encode(), index, count, _ptr(out))
    return out


def libm(mode, x, restated=False):
    """mode 0 cbrt / 1 pow(x, 3.0) over a float64 array: the host libm the
    reference links (restated=False) or the C restatement (libm_restate.c)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    lib().orc_libm(mode, 1 if restated else 0, x.ctypes.data_as(ctypes.c_void_p),
                   out.ctypes.data_as(ctypes.c_void_p), len(x))
    return out


def libm_test_inputs(n, seed=0):
    """Doubles over CUBIC's argument ranges (t - K in [-200, 200], cube-root
    arguments w_max * 0.3 / 0.4 up to 1e7) plus every exponent, both signs."""
    rs = np.random.default_rng(seed)
    q = n // 4
    a = (rs.random(q) - 0.5) * 400.0
    b = rs.random(q) * 1e7
    c = rs.random(q) * 1e-3
    bits = rs.integers(0, 0x7FEFFFFFFFFFFFFF, size=n - 3 * q, dtype=np.int64)
    d = bits.view(np.float64) * np.where(rs.random(n - 3 * q) < 0.5, -1.0, 1.0)
    return np.concatenate([a, b, c, d, [0.0, -0.0, 1.0, -1.0, 8.0, 27.0, 0.75, 1e-300, 5e-324]])
