"""Ring all-reduce / reduce-scatter over NVLink built on the transport.

SURVEY.md 8(a) row X1 and 8(e): one rank per B200.  Reduce-scatter step s
(s = 0..N-2): rank r's message for rank r+1 is its segment (r-s) mod N; rank
r receives segment (r-s-1) mod N from r-1 and reduces it into its own copy
(acc = acc + recv).  All-gather step s: rank r receives segment (r-s) mod N
(complete on r-1) and overwrites.  Segment j therefore folds as
x[j-1] + (... + (x[j+1] + x[j])) and the result is bit-identical to the
same-order CPU fold (oracle/chunknet_oracle.c: orc_ring_allreduce).

Data movement is B200-native: every segment message is
packetized by its sender (cn_packetize = Transport::send_chunk,
transport.cpp:433-494) and pushed in chunk-aligned pieces by the copy
engines over NVLink (CUDA IPC peer mappings).  Reduce-scatter pieces land in
a staging slot of the receiver's HBM and the receiver's transport receive
path (csrc/rx.cu) reduces them into its accumulator (fused scatter-reduce);
all-gather pieces land directly in the receiver's accumulator segment and
its receive path runs on the headers only (bookkeeping, no payload pass).
Neighbours synchronise with device-side progress counters (cn_ctr_*),
never the host.  The scheduler's per-chunk paths travel in the headers and
drive the receive bookkeeping; NVLink gives one physical path per peer
pair, so the bytes move on two copy-engine lanes by piece.
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
    accumulator) on every rank.

    Pipelined push design.  Every segment message of a step is cut into
    `pieces` chunk-aligned pieces.  The sender's "wire" is a copy-engine
    transfer of a piece over NVLink into a staging slot in the receiver's
    HBM (cn_copy_async), followed by a system-scope release of a progress
    counter; a step's 64-B packet headers (cn_packetize, with the S3
    scheduler's per-chunk paths, packetized once per iteration) travel with
    its first piece into the receiver's header buffer.  The receiver runs the transport's receive path
    (csrc/rx.cu: ingest, fused reduce-scatter or copy, SACK/cum bookkeeping,
    completion) on each piece from local memory as soon as it lands, then
    frees the slot.  Piece p of step k+1 leaves as soon as piece p of step k
    has been reduced, so NVLink stays busy across steps (the pipelining NCCL
    does with its chunked ring), and the copy engines move the bytes while
    the SMs reduce.  Counters are relative to a device iteration counter, so
    one iteration can be captured in a CUDA graph (capture()/replay())."""

    def __init__(self, count, dtype=torch.float32, *, chunk_bytes=32768, paths=8, seed=1,
                 group=None, piece_bytes=32 << 20, max_spins=1 << 26):
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
        L = _lib.lib()
        self._acc_buf = DeviceBuffer(count * self.elem, self.dev)
        self.acc = self._acc_buf.tensor(dtype, count)
        self.steps = ring_schedule(n, r)
        self.quantum = 16 // self.elem
        segb = [seg_bounds(count, n, j, self.quantum) for j in range(n)]
        self.seg_bytes = [(b - a) * self.elem for a, b in segb]
        self.seg_off = [a * self.elem for a, b in segb]
        if min(self.seg_bytes) < chunk_bytes:
            raise ValueError("count too small for the ring (a segment must hold a chunk)")
        # pieces per step (the same on every rank and step), chunk-aligned; an
        # even count feeds two push lanes (copy streams) alternately
        P = max(1, min(-(-max(self.seg_bytes) // piece_bytes), min(self.seg_bytes) // chunk_bytes))
        if P > 1 and P % 2:
            P = P + 1 if P + 1 <= min(self.seg_bytes) // chunk_bytes else P - 1
        self.pieces = P
        self.lanes = 2 if P % 2 == 0 else 1
        self.bounds = [[0 if p == 0 else (sb if p == P else sb * p // P // chunk_bytes * chunk_bytes)
                        for p in range(P + 1)] for sb in self.seg_bytes]
        self.slot_bytes = max(b[p + 1] - b[p] for b in self.bounds for p in range(P))
        self.ppi = (2 * n - 2) * P  # pieces per iteration
        ppc = -(-chunk_bytes // MAX_PAYLOAD)
        self.n_pkts = [L.cn_packet_count(sb, chunk_bytes, MAX_PAYLOAD) for sb in self.seg_bytes]

        def pkt_range(j, p):
            lo, hi = self.bounds[j][p], self.bounds[j][p + 1]
            return lo // chunk_bytes * ppc, (self.n_pkts[j] if hi == self.seg_bytes[j] else hi // chunk_bytes * ppc)
        self.pkt_range = pkt_range
        # receive side: staging slots and one header buffer per step (written by prev)
        self._stage = DeviceBuffer(P * self.slot_bytes, self.dev)
        self._hdr_bufs = [DeviceBuffer(max(1, self.n_pkts[st[4]]) * 64, self.dev) if st[1] != "init" else None
                          for st in self.steps]
        # flags: ready[2] (from prev), freed[2] (from next), err, iteration;
        # one ready/freed counter pair per push lane (monotone within a lane)
        self._flag_buf = DeviceBuffer(64, self.dev)
        self.flags = self._flag_buf.tensor(torch.int64, 8)
        fp = self._flag_buf.data_ptr()
        self.f_ready, self.f_freed, self.f_err, self.f_it = fp, fp + 16, fp + 32, fp + 40
        # per-chunk path choices of the outgoing messages (S3 scheduler): one
        # virtual connection (RngStream) per piece of each step's message, so
        # all of an iteration's choices come from one launch of many streams
        from .scheduler import PathScheduler
        n_msgs = len(self.steps) - 1
        self.sched = PathScheduler(n_msgs * P, paths, seed, base_rtt_ns=10000.0, index0=r * n_msgs * P)
        offs, self.path_slices = [0], []
        for st in self.steps[1:]:
            b = self.bounds[st[3]]
            start = offs[-1]
            for p in range(P):
                offs.append(start + -(-b[p + 1] // chunk_bytes))
            self.path_slices.append((start, offs[-1]))
        self.path_offs = torch.tensor(offs, dtype=torch.int32, device=self.dev)
        self.paths_all = torch.empty(max(1, offs[-1]), dtype=torch.int32, device=self.dev)
        # my outgoing headers (packetized locally, copied per piece with the payload)
        self._out_hdrs = [DeviceBuffer(max(1, self.n_pkts[st[3]]) * 64, self.dev) if st[1] != "init" else None
                          for st in self.steps]
        # exchange IPC handles: staging, header buffers, flags
        mine = {"stage": _ipc_handle(self._stage), "flags": _ipc_handle(self._flag_buf),
                "acc": _ipc_handle(self._acc_buf),
                "hdrs": [_ipc_handle(b) if b is not None else None for b in self._hdr_bufs]}
        allh = [None] * n
        dist.all_gather_object(allh, mine, group=group)
        prev, nxt = (r - 1) % n, (r + 1) % n
        self._opened = []
        self.next_stage = self._open(allh[nxt]["stage"])
        self.next_acc = self._open(allh[nxt]["acc"])
        self.next_hdrs = [self._open(h) if h is not None else None for h in allh[nxt]["hdrs"]]
        self.next_flags = self._open(allh[nxt]["flags"])
        self.prev_flags = self._open(allh[prev]["flags"]) if prev != nxt else self.next_flags
        # receive paths: reduce-scatter (fused reduce) and all-gather (copy)
        red = "sum_f32" if dtype == torch.float32 else "sum_bf16"
        maxp = max(pkt_range(j, p)[1] - pkt_range(j, p)[0] for j in range(n) for p in range(P))
        max_chunks = max(-(-sb // chunk_bytes) for sb in self.seg_bytes)
        kw = dict(device=self.dev, max_conns=4, max_msgs=4 * n, chunk_pool=4 * n * max_chunks + 64,
                  arena_bytes=0, max_batch=maxp + 16, max_posts=4 * n)
        cfg = TransportConfig(chunk_bytes=chunk_bytes, paths=paths, lb="p2_rtt", carry_payload=True)
        self.rx_rs = Transport(cfg, reduce=red, **kw)
        # all-gather: the payload lands in place, the receive path keeps the books
        self.rx_ag = Transport(TransportConfig(chunk_bytes=chunk_bytes, paths=paths, lb="p2_rtt",
                                               carry_payload=False), **kw)
        accb = self.acc.view(torch.uint8)
        for (k, ph, s, snd, rcv, tag) in self.steps:
            if ph == "rs":
                self.rx_rs.post(tag, accb[self.seg_off[rcv]: self.seg_off[rcv] + self.seg_bytes[rcv]])
        self.push_streams = [torch.cuda.Stream(self.dev) for _ in range(self.lanes)]
        self.hdr_stream = torch.cuda.Stream(self.dev)
        self.rx_done = [[torch.cuda.Event() for _ in range(P)] for _ in self.steps]
        self.ev_init = torch.cuda.Event()
        self.ev_hdrs = torch.cuda.Event()
        self._graph = None
        torch.cuda.synchronize()
        dist.barrier(group)

    def _open(self, h):
        p = _ipc_open(h)
        self._opened.append(p)
        return p

    def close(self):
        torch.cuda.synchronize()
        self._graph = None
        for p in getattr(self, "_opened", []):
            _lib.lib().cn_ipc_close(ctypes.c_void_p(p))
        self._opened = []
        for b in [getattr(self, "_acc_buf", None), getattr(self, "_flag_buf", None),
                  getattr(self, "_stage", None)] + list(getattr(self, "_hdr_bufs", [])) + \
                list(getattr(self, "_out_hdrs", [])):
            if b is not None:
                b.free()

    def _wait(self, flag, off, s):
        _lib.check(_lib.lib().cn_ctr_wait(flag, self.f_it, self.ppi // self.lanes, off, self.max_spins,
                                          self.f_err, ctypes.c_void_p(s.cuda_stream)), "cn_ctr_wait")

    def _signal(self, flag, off, s):
        _lib.check(_lib.lib().cn_ctr_signal(flag, self.f_it, self.ppi // self.lanes, off,
                                            ctypes.c_void_p(s.cuda_stream)), "cn_ctr_signal")

    def buffer(self):
        """The accumulator: write the input here and call run() for an
        in-place all-reduce (no init copy, like an in-place ncclAllReduce)."""
        return self.acc

    def _enqueue(self, x, s):
        L = _lib.lib()
        n, r, P, NL = self.n, self.rank, self.pieces, self.lanes
        sp = self.push_streams[0]
        # init: the accumulator and fresh receive state (main stream); this
        # iteration's paths and packet headers, packetized locally (push stream)
        if x is not None:
            self.acc.copy_(x)
        self.rx_rs.reset(s)
        self.rx_ag.reset(s)
        self.ev_init.record(s)
        sh = self.hdr_stream  # paths + headers, beside the first payload transfers
        sh.wait_event(self.ev_init)
        self.sched.select("p2_rtt", offsets=self.path_offs, out=self.paths_all, stream=sh)
        for (k, ph, st, snd, rcv, tag) in self.steps[1:]:
            a, b = self.path_slices[k - 1]
            out = _PeerView(self._out_hdrs[k].data_ptr(), self.n_pkts[snd] * 64)
            packetize(self.seg_bytes[snd], self.cb, src=r, dst=(r + 1) % n, conn_id=0, msg_id=k % 128,
                      msg_seq=k, tag=tag, chunk_paths=self.paths_all[a:b], out=out, stream=sh, device=self.dev)
        self.ev_hdrs.record(sh)
        for sl in self.push_streams:
            sl.wait_event(self.ev_init)
        acc = self._acc_buf.data_ptr()
        for (k, ph, st, snd, rcv, tag) in self.steps[1:]:
            rx = self.rx_rs if ph == "rs" else self.rx_ag
            for p in range(P):
                gp = (k - 1) * P + p
                ln, q = p % NL, gp // NL  # push lane, index within the lane
                sp = self.push_streams[ln]
                # push piece p of my message (segment snd) into next's slot p
                if k > 1:
                    sp.wait_event(self.rx_done[k - 1][p])  # its bytes were reduced here
                # next consumed the slot's last piece (for p = 0 that also
                # means it is done with this step's headers of the last iteration:
                # its receive path runs pieces in order)
                self._wait(self.f_freed + 8 * ln, q + 1 - P // NL, sp)
                lo, hi = self.bounds[snd][p], self.bounds[snd][p + 1]
                # reduce-scatter: into next's staging slot; all-gather: the
                # final bytes straight into next's accumulator segment
                dst = self.next_stage + p * self.slot_bytes if ph == "rs" else self.next_acc + self.seg_off[snd] + lo
                _lib.check(L.cn_copy_async(dst, acc + self.seg_off[snd] + lo, hi - lo,
                                           ctypes.c_void_p(sp.cuda_stream)), "cn_copy_async")
                if p == 0:  # the whole step's headers ride with its first piece
                    if k == 1:
                        sp.wait_event(self.ev_hdrs)
                    _lib.check(L.cn_copy_async(self.next_hdrs[k], self._out_hdrs[k].data_ptr(),
                                               self.n_pkts[snd] * 64, ctypes.c_void_p(sp.cuda_stream)),
                               "cn_copy_async")
                self._signal(self.next_flags + 8 * ln, q + 1, sp)  # next's ready counter
                # receive piece p of prev's message (segment rcv) from my slot p
                self._wait(self.f_ready + 8 * ln, q + 1, s)
                rlo = self.bounds[rcv][p]
                a, b = self.pkt_range(rcv, p)
                hd = _PeerView(self._hdr_bufs[k].data_ptr() + a * 64, (b - a) * 64)
                if ph == "rs":
                    src = _PeerView(self._stage.data_ptr() + p * self.slot_bytes - rlo, self.slot_bytes)
                    rx.rx_batch_async(hd, src, 0, s, n=b - a)
                else:  # headers only: the bytes already sit in the accumulator
                    rx.rx_batch_async(hd, None, 0, s, n=b - a)
                self.rx_done[k][p].record(s)
                self._signal(self.prev_flags + 16 + 8 * ln, q + 1, s)  # prev's freed counter
        for sl in self.push_streams + [self.hdr_stream]:
            s.wait_stream(sl)
        _lib.check(L.cn_ctr_advance(self.f_it, ctypes.c_void_p(s.cuda_stream)), "cn_ctr_advance")

    def run(self, x=None, stream=None):
        """All-reduce x (count elements, this rank's contribution), or the
        accumulator in place when x is None."""
        s = stream or torch.cuda.current_stream(self.dev)
        if self._graph is not None and x is None:
            self._graph.replay()
        else:
            self._enqueue(x, s)
        return self.acc

    def capture(self):
        """Capture one in-place iteration in a CUDA graph; later run() calls
        without x replay it (host launch cost independent of the pieces)."""
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(self.dev)
        s.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.graph(g, stream=s):
            self._enqueue(None, torch.cuda.current_stream(self.dev))
        torch.cuda.synchronize()
        self._graph = g
        return g

    def check(self):
        """Host check after run(): device flag timeouts and transport status."""
        if int(self.flags[4].item()) != 0:
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
