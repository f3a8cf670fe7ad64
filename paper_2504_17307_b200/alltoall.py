"""Variable-size all-to-all over NVLink through the transport: the MoE
dispatch / combine of BASELINE configs[3] (SURVEY.md 8(d) cfg 4, 8(e):
"all-to-all = N-1 peer connections per rank").

Each rank holds one connection to every peer.  Per call, rank r's message
to peer d (`send_counts[d]` bytes of its send buffer) is packetized
(cn_packetize = Transport::send_chunk, per-chunk paths from the S3
scheduler) and moved by a copy engine over NVLink, its headers alongside,
followed by a system-scope release of d's ready counter for r (the NIC DMA
+ doorbell of the paper's transport).  Direct mode (the default): the bytes
land straight in d's receive slot for r -- RDMA-write semantics into a
posted buffer, armed by d at the start of each call -- and d's receive
path keeps the books on the headers alone (SACK / cum / completion, no
payload pass); staged mode lands them in a staging slot and d's receive
path scatters them into the slot (accept_payload).  Either way d releases
r's freed counter per piece, after which r may reuse the header slot.  Messages to different
peers leave on two lanes in a staggered order (r+1, r+2, ...), so a
hot receiver (incast) sees all its senders at once -- its NVLink ingress is
the bottleneck, which is the point of the workload.  Messages move in
chunk-aligned pieces, each releasing a per-pair monotone counter, so the
receive path runs on early pieces while later ones are still in flight.
"""
import ctypes
import os

import torch
import torch.distributed as dist

from . import _lib
from .collective import DeviceBuffer, _ipc_handle, _ipc_open, _PeerView, packetize
from .transport import MAX_PAYLOAD, Transport, TransportConfig


class AllToAll:
    def __init__(self, max_bytes_per_peer, *, chunk_bytes=32768, paths=8, seed=7, group=None,
                 piece_bytes=128 << 20, max_spins=1 << 26, direct=True, tail=0, push=None, early=None):
        self.group = group
        self.n = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        n, r = self.n, self.rank
        if n < 2:
            raise ValueError("AllToAll needs >= 2 ranks")
        self.cap = (max_bytes_per_peer + 15) // 16 * 16
        self.cb = chunk_bytes
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.max_spins = max_spins
        self.direct = direct
        self.tail = tail
        # direct mode: a source's headers lead its first piece, and the bytes
        # never pass through the receive path, so the path runs on the whole
        # message once the headers land, beside the remaining pieces; the
        # call still returns only after every piece's flag (else: a piece's
        # headers after that piece lands, the last one's path exposed)
        if early is None:
            early = os.environ.get("CN_A2A_EARLY", "1") == "1"
        self.early = bool(early) and direct
        # the wire: SM stores over NVLink ("sm:<blocks>", default 64 blocks per
        # piece: N = 2 / 4 1.307 / 3.388 ms vs 1.325 / 3.422 with 32; no per-copy
        # cost, and unaffected by a source the previous phase just wrote) or
        # the copy engines ("ce"; ~4.4 us per copy)
        self.push = push or os.environ.get("CN_A2A_PUSH", "sm:64")
        # push lanes (streams): two hide the gap between consecutive pieces (one
        # lane measured no better with SM push: 1.56 vs 1.54 ms, N = 2)
        self.nl = int(os.environ.get("CN_A2A_LANES", "2"))
        self.calls = 0
        self._rx_clean = False  # the receive state was reset after the previous call's last batch
        L = _lib.lib()
        self.max_pkts = L.cn_packet_count(self.cap, chunk_bytes, MAX_PAYLOAD)
        # receive side: posted destination slot, staging slot and header slot per source
        self._recv = DeviceBuffer(n * self.cap, self.dev)
        self._stage = None if direct else DeviceBuffer(n * self.cap, self.dev)
        self._hdrs = DeviceBuffer(n * self.max_pkts * 64, self.dev)
        self._out_hdrs = DeviceBuffer(n * self.max_pkts * 64, self.dev)  # my outgoing headers
        # flags: ready[n][2] (written by sources, per copy lane), freed[n][2]
        # (written by destinations), err, spare, armed[n] (written by
        # destinations: my receive slot for you is free for call k)
        self._flags = DeviceBuffer((5 * n + 2) * 8, self.dev)
        self._ctr = DeviceBuffer(64, self.dev)  # per push lane: the signalling copy's block counter
        self.flags = self._flags.tensor(torch.int64, 5 * n + 2)
        fp = self._flags.data_ptr()
        self.f_ready, self.f_freed = fp, fp + 16 * n
        self.f_err = fp + 32 * n
        self.o_armed = (4 * n + 2) * 8
        self.f_armed = fp + self.o_armed
        land = self._recv if direct else self._stage
        mine = {"land": _ipc_handle(land), "hdrs": _ipc_handle(self._hdrs),
                "flags": _ipc_handle(self._flags)}
        allh = [None] * n
        dist.all_gather_object(allh, mine, group=group)
        self._opened = []
        self.peer = {}
        for d in range(n):
            if d == r:
                continue
            self.peer[d] = {k: self._open(allh[d][k]) for k in ("land", "hdrs", "flags")}
        # path choices: one RngStream per block of 2048 chunks of each peer
        # connection's message (the sequential Mersenne draws of one stream
        # would otherwise sit in front of every transfer)
        from .scheduler import PathScheduler
        self.max_chunks = -(-self.cap // chunk_bytes)
        self.blk = 2048
        self.sp = -(-self.max_chunks // self.blk)
        self.sched = PathScheduler(n * self.sp, paths, seed, base_rtt_ns=10000.0, index0=r * n * self.sp)
        self.paths_all = torch.empty(n * self.max_chunks, dtype=torch.int32, device=self.dev)
        self.rx = Transport(TransportConfig(chunk_bytes=chunk_bytes, paths=paths, lb="p2_rtt",
                                            carry_payload=not direct),
                            device=self.dev, max_conns=2 * n, max_msgs=4 * n,
                            chunk_pool=2 * n * self.max_chunks + 64, arena_bytes=0,
                            max_batch=self.max_pkts + 16, max_posts=4 * n)
        if not direct:  # the receive path scatters staged bytes into the posted slots
            rb = self.recv_buffer()
            for s in range(n):
                if s != r:
                    self.rx.post(s, rb[s * self.cap:(s + 1) * self.cap])
        self.lanes = [torch.cuda.Stream(self.dev) for _ in range(2)]
        self.hdr_stream = torch.cuda.Stream(self.dev)
        self.ev_hdrs = torch.cuda.Event()
        self.piece_bytes = max(chunk_bytes, piece_bytes // chunk_bytes * chunk_bytes)
        self.sent = [[0, 0] for _ in range(n)]   # pieces sent to each peer, per lane
        self.recvd = [[0, 0] for _ in range(n)]  # pieces consumed from each peer, per lane
        self.ev_init = torch.cuda.Event()
        # the copy lanes' last work of the previous call: the next call's headers
        # may be built as soon as those copies have read the header buffer
        self.ev_lanes = [torch.cuda.Event() for _ in range(2)]
        torch.cuda.synchronize()
        dist.barrier(group)

    def _open(self, h):
        p = _ipc_open(h)
        self._opened.append(p)
        return p

    def recv_buffer(self):
        """uint8 view of the receive slots: source s's message at [s*cap, s*cap + recv_counts[s])."""
        return self._recv.tensor()

    def close(self):
        torch.cuda.synchronize()
        for p in self._opened:
            _lib.lib().cn_ipc_close(ctypes.c_void_p(p))
        self._opened = []
        for b in (self._recv, self._stage, self._hdrs, self._out_hdrs, self._flags, self._ctr):
            if b is not None:
                b.free()

    def _wait(self, flag, off, s):
        _lib.check(_lib.lib().cn_ctr_wait(flag, self.f_it, 1, off, self.max_spins, self.f_err,
                                          ctypes.c_void_p(s.cuda_stream)), "cn_ctr_wait")

    def _signal(self, flag, off, s):
        _lib.check(_lib.lib().cn_ctr_signal(flag, self.f_it, 1, off, ctypes.c_void_p(s.cuda_stream)),
                   "cn_ctr_signal")

    def _pieces(self, cnt):
        """Chunk-aligned piece bounds of a cnt-byte message.  With tail
        pieces: one large head piece (a copy-engine transfer runs at the
        link's rate only when large, ~4 us of fixed cost per copy), then
        `tail` pieces of piece_bytes whose transfers hide the receive path
        of the head; else equal pieces of at most piece_bytes."""
        if cnt == 0:
            return []
        tb = self.tail * self.piece_bytes
        if self.tail and cnt > tb + self.piece_bytes:
            h = (cnt - tb) // self.cb * self.cb
            b = [0, h] + [h + k * self.piece_bytes for k in range(1, self.tail)] + [cnt]
            return [(b[p], b[p + 1]) for p in range(len(b) - 1) if b[p + 1] > b[p]]
        P = max(1, min(-(-cnt // self.piece_bytes), -(-cnt // self.cb)))
        b = [0] + [cnt * p // P // self.cb * self.cb for p in range(1, P)] + [cnt]
        return [(b[p], b[p + 1]) for p in range(P) if b[p + 1] > b[p]]

    def run(self, send, send_counts, recv_counts, send_offsets=None, stream=None):
        """send: device uint8 tensor; send_counts[d] bytes for peer d starting at
        send_offsets[d] (default: packed in peer order); recv_counts[s] bytes
        expected from each source.  Returns the receive slots view.

        Messages travel in chunk-aligned pieces (piece_bytes), interleaved
        across sources.  Direct mode (early): a source's headers land with
        its first piece and the receive path runs on the whole message then,
        beside the remaining pieces; otherwise the path runs on each piece as
        it lands.  Either way a hot receiver's processing overlaps its
        ingress, and the call returns after every piece has landed."""
        L = _lib.lib()
        n, r = self.n, self.rank
        s = stream or torch.cuda.current_stream(self.dev)
        send_counts = [int(x) for x in send_counts]
        recv_counts = [int(x) for x in recv_counts]
        if send_offsets is not None:
            send_offsets = [int(x) for x in send_offsets]
        if send_offsets is None:
            send_offsets, o = [], 0
            for d in range(n):
                send_offsets.append(o)
                o += send_counts[d]
        assert max(send_counts) <= self.cap and max(recv_counts) <= self.cap
        ppc = -(-self.cb // MAX_PAYLOAD)
        self.calls += 1
        if not self._rx_clean:
            self.rx.reset(s)
        self._rx_clean = False
        if self.direct:  # my receive slots are free (stream order): arm every source
            for src in range(n):
                if src != r:
                    _lib.check(L.cn_flag_post(self.peer[src]["flags"] + self.o_armed + 8 * r, self.calls,
                                              ctypes.c_void_p(s.cuda_stream)), "cn_flag_post")
        self.ev_init.record(s)
        for ln in self.lanes:
            ln.wait_event(self.ev_init)
        # paths and headers of every outgoing message on a side stream, beside
        # the first transfers (headers ride with a message's first piece)
        # built ahead: the header stream waits only for the previous call's
        # copies of the header buffer, not for this rank's earlier work on s
        # (the combine's headers are ready while the dispatch still runs)
        sh = self.hdr_stream
        for ev in self.ev_lanes:
            sh.wait_event(ev)
        nch = [-(-send_counts[d] // self.cb) if d != r else 0 for d in range(n)]
        offs, goffs = [0], [0]
        for d in range(n):
            start = offs[-1]
            for b_ in range(self.sp):
                goffs.append(start + min(nch[d], (b_ + 1) * self.blk))
            offs.append(start + nch[d])
        with torch.cuda.stream(sh):
            po = torch.tensor(goffs, dtype=torch.int32).to(self.dev, non_blocking=True)
        self.sched.select("p2_rtt", offsets=po, out=self.paths_all, stream=sh)
        for d in range(n):
            if d != r and send_counts[d]:
                npk = L.cn_packet_count(send_counts[d], self.cb, MAX_PAYLOAD)
                oh = _PeerView(self._out_hdrs.data_ptr() + d * self.max_pkts * 64, npk * 64)
                packetize(send_counts[d], self.cb, src=r, dst=d, conn_id=0, msg_id=1, msg_seq=1, tag=r,
                          chunk_paths=self.paths_all[offs[d]:offs[d + 1]], out=oh, stream=sh, device=self.dev)
        self.ev_hdrs.record(sh)
        sb = send.data_ptr()
        cs = lambda st: ctypes.c_void_p(st.cuda_stream)  # noqa: E731
        for k in range(1, n):  # staggered: r+1, r+2, ...
            d = (r + k) % n
            if not send_counts[d]:
                continue
            pe = self.peer[d]
            # d consumed every piece of my previous message (slot and header reuse)
            # (direct mode: and d armed its receive slot for me this call) -- one wait kernel
            for ln in range(self.nl):
                _lib.check(L.cn_flag_wait_signal(self.f_freed + 16 * d + 8 * ln, self.sent[d][ln],
                                                 self.f_armed + 8 * d if self.direct else None, self.calls,
                                                 None, 0, self.max_spins, self.f_err, cs(self.lanes[ln])),
                           "cn_flag_wait_signal")
            npk = L.cn_packet_count(send_counts[d], self.cb, MAX_PAYLOAD)
            oh = self._out_hdrs.data_ptr() + d * self.max_pkts * 64
            for p, (lo, hi) in enumerate(self._pieces(send_counts[d])):
                ln = (k + p) % self.nl  # consecutive pieces alternate push lanes
                sp = self.lanes[ln]
                if p == 0:  # the message's headers lead its first piece (a copy beside it on its
                    # own stream measured slower: 1.38 vs 1.36 ms, N = 2)
                    sp.wait_event(self.ev_hdrs)
                    _lib.check(L.cn_copy_async(pe["hdrs"] + r * self.max_pkts * 64, oh, npk * 64, cs(sp)),
                               "cn_copy_async")
                dst_p, src_p = pe["land"] + r * self.cap + lo, sb + send_offsets[d] + lo
                self.sent[d][ln] += 1
                ready = pe["flags"] + 16 * r + 8 * ln
                if self.push.startswith("sm") and not ((dst_p | src_p | (hi - lo)) & 15):
                    # the copy's last block raises d's ready flag
                    nb = int(self.push.split(":")[1]) if ":" in self.push else 64
                    _lib.check(L.cn_copy_sm_signal(dst_p, src_p, hi - lo, nb, ready, self.sent[d][ln],
                                                   self._ctr.data_ptr() + 4 * ln, cs(sp)), "cn_copy_sm_signal")
                else:  # the copy engines (or a piece not 16-byte aligned, which SM vectors cannot move)
                    _lib.check(L.cn_copy_async(dst_p, src_p, hi - lo, cs(sp)), "cn_copy_async")
                    _lib.check(L.cn_flag_signal(ready, None, self.sent[d][ln], cs(sp)), "cn_flag_signal")
        # receive: pieces as they land, interleaved over the sources (r-1, r-2, ...)
        plan = {}
        for k in range(1, n):
            src = (r - k) % n
            if recv_counts[src]:
                plan[src] = (k, self._pieces(recv_counts[src]))
        # receive batches this call runs; after the last one the receive state
        # is reset for the next call, beside the pieces still in flight
        left = sum(1 if self.early else len(v[1]) for v in plan.values())
        for p in range(max([len(v[1]) for v in plan.values()] or [0])):
            for k in range(1, n):
                src = (r - k) % n
                if src not in plan or p >= len(plan[src][1]):
                    continue
                ks = (r - src) % n  # the sender's stagger index for me -> its lane choice
                ln = (ks + p) % self.nl
                lo, hi = plan[src][1][p]
                self.recvd[src][ln] += 1
                freed = self.peer[src]["flags"] + 16 * n + 16 * r + 8 * ln  # src's freed[r][ln]
                if self.early and p > 0:  # nothing to run on this piece: wait for it and release it, one kernel
                    _lib.check(L.cn_flag_wait_signal(self.f_ready + 16 * src + 8 * ln, self.recvd[src][ln], None,
                                                     0, freed, self.recvd[src][ln], self.max_spins, self.f_err,
                                                     cs(s)), "cn_flag_wait_signal")
                    continue
                _lib.check(L.cn_flag_wait(self.f_ready + 16 * src + 8 * ln, None, self.recvd[src][ln],
                                          self.max_spins, self.f_err, cs(s)), "cn_flag_wait")
                a = lo // self.cb * ppc
                b = (L.cn_packet_count(recv_counts[src], self.cb, MAX_PAYLOAD) if hi == recv_counts[src]
                     else hi // self.cb * ppc)
                if self.early:  # every header of the message, once (they landed with piece 0)
                    a, b = 0, L.cn_packet_count(recv_counts[src], self.cb, MAX_PAYLOAD)
                hd = _PeerView(self._hdrs.data_ptr() + src * self.max_pkts * 64 + a * 64, (b - a) * 64)
                if self.direct:  # headers only: the bytes already sit in the receive slot
                    self.rx.rx_batch_async(hd, None, 0, s, n=b - a)
                else:
                    pl = _PeerView(self._stage.data_ptr() + src * self.cap, recv_counts[src])
                    self.rx.rx_batch_async(hd, pl, 0, s, n=b - a)
                left -= 1
                if left == 0:
                    self.rx.reset(s)
                    self._rx_clean = True
                _lib.check(L.cn_flag_post(freed, self.recvd[src][ln], cs(s)), "cn_flag_post")  # consumed
        for ln, ev in zip(self.lanes, self.ev_lanes):
            ev.record(ln)
        for ln in self.lanes + [self.hdr_stream]:
            s.wait_stream(ln)
        return self.recv_buffer()

    def check(self):
        if int(self.flags[4 * self.n].item()) != 0:
            raise _lib.ChunknetError(-5, "all-to-all flag wait timed out")
        res = _lib.RxResult.from_buffer_copy(bytes(self.rx._result.cpu().numpy()))
        if res.status:
            raise _lib.ChunknetError(-6, f"all-to-all receive status 0x{res.status:x}")
