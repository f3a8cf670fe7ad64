"""Ring all-reduce / reduce-scatter over NVLink built on the transport.

SURVEY.md 8(a) row X1 and 8(e): one rank per B200.  Reduce-scatter step s
(s = 0..N-2): rank r's message for rank r+1 is its segment (r-s) mod N; rank
r receives segment (r-s-1) mod N from r-1 and reduces it into its own copy
(acc = acc + recv).  All-gather step s: rank r receives segment (r-s) mod N
(complete on r-1) and overwrites.  Segment j therefore folds as
x[j-1] + (... + (x[j+1] + x[j])) and the result is bit-identical to the
same-order CPU fold (oracle/chunknet_oracle.c: orc_ring_allreduce).

Data movement is B200-native: every segment message is packetized by its
sender (cn_packetize = Transport::send_chunk, transport.cpp:433-494) into a
header ring in the sender's HBM, and the receiver runs the transport's
receive path (csrc/rx.cu) with the fused reduce scatter reading both the
headers and the payload straight out of the peer's memory over NVLink
(CUDA IPC mapping, zero copy, payload_stride 0).  Neighbours synchronise
with device-side progress flags (cn_flag_*), never the host.
"""
import ctypes

import torch
import torch.distributed as dist

from . import _lib
from .transport import MAX_PAYLOAD, Transport, TransportConfig

ELEM = {torch.float32: 4, torch.bfloat16: 2}


def seg_bounds(count, n, j, q=1):
    """Segment j of a count-element buffer split over n ranks (elements),
    boundaries rounded down to multiples of q (16-byte aligned segments)."""
    lo = count * j // n // q * q
    hi = count if j + 1 >= n else count * (j + 1) // n // q * q
    return lo, hi


def ring_schedule(n, rank):
    """Per-iteration steps of rank `rank`: (k, phase, s, send_seg, recv_seg, tag).

    k = 0 is the local init (acc <- input); k = 1..n-1 reduce-scatter steps;
    k = n..2n-2 all-gather steps.  `tag` identifies the segment message of
    step (phase, s) on every connection (the reference's per-message tag)."""
    steps = [(0, "init", -1, -1, -1, -1)]
    for s in range(n - 1):
        steps.append((1 + s, "rs", s, (rank - s) % n, (rank - s - 1) % n, s))
    for s in range(n - 1):
        steps.append((n + s, "ag", s, (rank - s + 1) % n, (rank - s) % n, n + s))
    return steps


def packetize(length, chunk_bytes, *, src, dst, conn_id=0, msg_id=0, msg_seq=1, tag=0, tx_time=0,
              chunk_paths=None, path=0, is_rtx=False, out=None, stream=None, device="cuda"):
    """Transport::send_chunk packetization of a whole message -> device
    cn_pkt_hdr records (uint8 [n*64]) in chunk order."""
    L = _lib.lib()
    n = L.cn_packet_count(length, chunk_bytes, MAX_PAYLOAD)
    if out is None:
        out = torch.empty(n * 64, dtype=torch.uint8, device=device)
    a = _lib.PacketizeArgs(length, chunk_bytes, MAX_PAYLOAD, src, dst, conn_id, msg_id, msg_seq, tag,
                           tx_time, chunk_paths.data_ptr() if chunk_paths is not None else None,
                           path, 1 if is_rtx else 0)
    s = stream or torch.cuda.current_stream()
    _lib.check(L.cn_packetize(ctypes.byref(a), out.data_ptr(), ctypes.c_void_p(s.cuda_stream)),
               "cn_packetize")
    return out


class DeviceBuffer:
    """A whole cudaMalloc allocation (cn_dev_alloc): IPC handles of a torch
    caching-allocator tensor would name the enclosing segment, not the tensor."""

    def __init__(self, nbytes, device):
        p = ctypes.c_void_p()
        _lib.check(_lib.lib().cn_dev_alloc(nbytes, ctypes.byref(p)), "cn_dev_alloc")
        self.ptr, self.nbytes, self.device = p.value, nbytes, device

    def data_ptr(self):
        return self.ptr

    def tensor(self, dtype=torch.uint8, count=None):
        class _H:
            pass
        h = _H()
        es = torch.tensor([], dtype=dtype).element_size()
        n = count if count is not None else self.nbytes // es
        typestr = {torch.uint8: "|u1", torch.int64: "<i8", torch.float32: "<f4",
                   torch.int16: "<i2"}[dtype if dtype != torch.bfloat16 else torch.int16]
        h.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                      "data": (int(self.ptr), False), "version": 3}
        t = torch.as_tensor(h, device=self.device)
        return t.view(torch.bfloat16) if dtype == torch.bfloat16 else t

    def free(self):
        if self.ptr:
            _lib.lib().cn_dev_free(ctypes.c_void_p(self.ptr))
            self.ptr = None


def _ipc_handle(t):
    buf = ctypes.create_string_buffer(64)
    _lib.check(_lib.lib().cn_ipc_get_handle(t.data_ptr(), buf), "cn_ipc_get_handle")
    return bytes(buf.raw)


def _ipc_open(h):
    p = ctypes.c_void_p()
    _lib.check(_lib.lib().cn_ipc_open(ctypes.create_string_buffer(h, 64), ctypes.byref(p)),
               "cn_ipc_open")
    return p.value


class RingAllreduce:
    """In-place ring all-reduce of a `count`-element buffer, one rank per GPU.

    Construct collectively (every rank of the default process group); then
    `run(x)` returns the all-reduced buffer (a view of the internal
    accumulator) on every rank."""

    def __init__(self, count, dtype=torch.float32, *, chunk_bytes=32768, paths=8, seed=1,
                 group=None, max_spins=1 << 26):
        self.group = group
        self.n = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.dtype = dtype
        self.count = count
        self.elem = ELEM[dtype]
        self.cb = chunk_bytes
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.max_spins = max_spins
        n, r = self.n, self.rank
        if n < 2:
            raise ValueError("RingAllreduce needs >= 2 ranks")
        self._acc_buf = DeviceBuffer(count * self.elem, self.dev)
        self.acc = self._acc_buf.tensor(dtype, count)
        self.steps = ring_schedule(n, r)
        self.quantum = 16 // self.elem
        segb = [seg_bounds(count, n, j, self.quantum) for j in range(n)]
        self.seg_bytes = [(b - a) * self.elem for a, b in segb]
        self.seg_off = [a * self.elem for a, b in segb]
        if min(self.seg_bytes) == 0:
            raise ValueError("count too small for the ring")
        # outgoing header rings, one per step (read by rank r+1 over NVLink)
        self.n_pkts = [_lib.lib().cn_packet_count(self.seg_bytes[st[3]], chunk_bytes, MAX_PAYLOAD)
                       if st[1] != "init" else 0 for st in self.steps]
        self._hdr_bufs = [DeviceBuffer(max(1, k) * 64, self.dev) for k in self.n_pkts]
        self.hdrs = [b.tensor() for b in self._hdr_bufs]
        # per-chunk path choices for the outgoing messages (S3 scheduler)
        # one virtual connection (RngStream) per step's message, so the path
        # choices of all messages of an iteration are drawn in one launch
        from .scheduler import PathScheduler
        n_msgs = len(self.steps) - 1
        self.sched = PathScheduler(n_msgs, paths, seed, base_rtt_ns=10000.0, index0=r * n_msgs)
        self.max_chunks = max((b + chunk_bytes - 1) // chunk_bytes for b in self.seg_bytes)
        nchs = [(self.seg_bytes[st[3]] + chunk_bytes - 1) // chunk_bytes for st in self.steps[1:]]
        offs = [0]
        for c in nchs:
            offs.append(offs[-1] + c)
        self.path_offs = torch.tensor(offs, dtype=torch.int32, device=self.dev)
        self.paths_all = torch.empty(max(1, offs[-1]), dtype=torch.int32, device=self.dev)
        self.path_slices = [(offs[i], offs[i + 1]) for i in range(n_msgs)]
        # flags: [from_prev, from_next, err]
        self._flag_buf = DeviceBuffer(64, self.dev)
        self.flags = self._flag_buf.tensor(torch.int64, 4)
        # exchange IPC handles: acc, headers, flags
        mine = {"acc": _ipc_handle(self._acc_buf), "flags": _ipc_handle(self._flag_buf),
                "hdrs": [_ipc_handle(b) for b in self._hdr_bufs]}
        allh = [None] * n
        dist.all_gather_object(allh, mine, group=group)
        prev, nxt = (r - 1) % n, (r + 1) % n
        self._opened = []
        self.prev_acc = self._open(allh[prev]["acc"])
        self.prev_hdrs = [self._open(h) for h in allh[prev]["hdrs"]]
        self.prev_flags = self._open(allh[prev]["flags"])
        self.next_flags = self._open(allh[nxt]["flags"]) if nxt != prev else self.prev_flags
        self.prev_n_pkts = []
        for st in ring_schedule(n, prev):
            self.prev_n_pkts.append(_lib.lib().cn_packet_count(self.seg_bytes[st[3]], chunk_bytes,
                                                               MAX_PAYLOAD) if st[1] != "init" else 0)
        # receive paths: reduce-scatter (fused reduce) and all-gather (copy)
        red = "sum_f32" if dtype == torch.float32 else "sum_bf16"
        maxp = max(self.prev_n_pkts)
        kw = dict(device=self.dev, max_conns=4, max_msgs=4 * n, chunk_pool=4 * n * self.max_chunks + 64,
                  arena_bytes=0, max_batch=maxp + 16, max_posts=4 * n)
        cfg = TransportConfig(chunk_bytes=chunk_bytes, paths=paths, lb="p2_rtt", carry_payload=True)
        self.rx_rs = Transport(cfg, reduce=red, **kw)
        self.rx_ag = Transport(cfg, **kw)
        accb = self.acc.view(torch.uint8)
        for (k, ph, s, snd, rcv, tag) in self.steps:
            if ph == "rs":
                self.rx_rs.post(tag, accb[self.seg_off[rcv]: self.seg_off[rcv] + self.seg_bytes[rcv]])
            elif ph == "ag":
                self.rx_ag.post(tag, accb[self.seg_off[rcv]: self.seg_off[rcv] + self.seg_bytes[rcv]])
        self.g = 0  # global step counter (across iterations)
        torch.cuda.synchronize()
        dist.barrier(group)

    def _open(self, h):
        p = _ipc_open(h)
        self._opened.append(p)
        return p

    def close(self):
        torch.cuda.synchronize()
        for p in getattr(self, "_opened", []):
            _lib.lib().cn_ipc_close(ctypes.c_void_p(p))
        self._opened = []
        for b in [getattr(self, "_acc_buf", None), getattr(self, "_flag_buf", None)] + \
                list(getattr(self, "_hdr_bufs", [])):
            if b is not None:
                b.free()

    def _wait(self, g, s):
        fp = self.flags.data_ptr()
        _lib.check(_lib.lib().cn_flag_wait(fp, fp + 8, g, self.max_spins, fp + 16,
                                           ctypes.c_void_p(s.cuda_stream)), "cn_flag_wait")

    def _signal(self, g, s):
        # next rank's from_prev, previous rank's from_next
        a = self.next_flags
        b = self.prev_flags + 8
        _lib.check(_lib.lib().cn_flag_signal(a, b, g, ctypes.c_void_p(s.cuda_stream)),
                   "cn_flag_signal")

    def buffer(self):
        """The accumulator: write the input here and call run() for an
        in-place all-reduce (no init copy, like an in-place ncclAllReduce)."""
        return self.acc

    def run(self, x=None, stream=None):
        """All-reduce x (count elements, this rank's contribution), or the
        accumulator in place when x is None."""
        s = stream or torch.cuda.current_stream(self.dev)
        n, r = self.n, self.rank
        for (k, ph, st, snd, rcv, tag) in self.steps:
            g = self.g
            self._wait(g, s)  # neighbours finished global step g-1
            if ph == "init":
                if x is not None:
                    self.acc.copy_(x)
                self.rx_rs.reset(s)
                self.rx_ag.reset(s)
                self.sched.select("p2_rtt", offsets=self.path_offs, out=self.paths_all, stream=s)
                for (k2, ph2, st2, snd2, rcv2, tag2) in self.steps[1:]:
                    a, b = self.path_slices[k2 - 1]
                    packetize(self.seg_bytes[snd2], self.cb, src=r, dst=(r + 1) % n, conn_id=0,
                              msg_id=k2 % 128, msg_seq=k2, tag=tag2, chunk_paths=self.paths_all[a:b],
                              out=self.hdrs[k2], stream=s, device=self.dev)
            else:
                rx = self.rx_rs if ph == "rs" else self.rx_ag
                npk = self.prev_n_pkts[k]
                hd = _PeerView(self.prev_hdrs[k], npk * 64)
                src = _PeerView(self.prev_acc + self.seg_off[rcv], self.seg_bytes[rcv])
                rx.rx_batch_async(hd, src, 0, s, n=npk)
            self._signal(g + 1, s)
            self.g += 1
        return self.acc

    def check(self):
        """Host check after run(): device flag timeouts and transport status."""
        if int(self.flags[2].item()) != 0:
            raise _lib.ChunknetError(-5, "ring flag wait timed out")
        for rx in (self.rx_rs, self.rx_ag):
            res = _lib.RxResult.from_buffer_copy(bytes(rx._result.cpu().numpy()))
            if res.status:
                raise _lib.ChunknetError(-6, f"ring receive status 0x{res.status:x}")


class _PeerView:
    """Duck-typed stand-in for a device tensor at a raw (peer) address."""

    def __init__(self, ptr, nbytes):
        self._p = int(ptr)
        self._n = int(nbytes)

    def data_ptr(self):
        return self._p

    def numel(self):
        return self._n


def busbw(nbytes, seconds, n):
    """NCCL-tests convention: (S/t) * 2(n-1)/n."""
    return nbytes / seconds * 2 * (n - 1) / n / 1e9
