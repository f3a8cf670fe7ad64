"""bench.py -- reassembly + ACK bookkeeping throughput of the B200 receive path.

Workload (BASELINE.json configs[1], "cfg2"): one 64 MiB message sprayed over
256 paths with 1% random drop and heavy reordering, as recorded from the
reference discrete-event simulator (tests/golden/cfg2_32k.npz: k=32 fat
tree 0 -> 8191, 32 KiB chunks, seed 1; 19,997 delivered data packets incl.
retransmissions, 2,885 acks).  One step = the device receive path over the
whole trace: reset receive state, classify, mark, scan, decide, scatter-copy
payloads into the message buffer, emit the ordered ack stream, finalize.

N > 1 GPUs: every rank runs its own replica (the transport shards by
connection; no data-path collective) -> weak scaling; the
ring all-reduce of configs[2] is reported beside it.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
MAX_PL = 4032
HDR = 64
ACK = 64


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="cfg2_32k")
    ap.add_argument("--conns", type=int, default=4,
                    help="concurrent connections per batch (each a copy of the workload trace)")
    ap.add_argument("--replicas", type=int, default=4,
                    help="rotating staging replicas so that inputs exceed L2")
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sched", action="store_true")
    ap.add_argument("--no-ring", action="store_true")
    ap.add_argument("--piece-mb", type=int, default=64, help="ring pipeline piece size (MiB)")
    ap.add_argument("--no-moe", action="store_true", help="skip the MoE all-to-all (configs[3]) at N > 1")
    ap.add_argument("--no-sweep", action="store_true", help="skip the configs[4] receive sweep")
    return ap.parse_args()


def load_trace(name):
    z = np.load(os.path.join(ROOT, "tests", "golden", f"{name}.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    return z["data"], meta, len(z["acks"])


def interleave(data, k):
    """k concurrent copies of a recorded single-connection trace as one
    receiver would see them: copy j comes from source host j (its own
    connection and message, tag j), packets merged round-robin."""
    if k == 1:
        return data.copy()
    out = np.empty(len(data) * k, dtype=data.dtype)
    for j in range(k):
        c = data.copy()
        c["src"] = j
        c["msg_tag"] = j
        out[j::k] = c
    return out


def copy_traffic(workload, conns):
    """DRAM bytes (read + write) per k_copy launch from the committed ncu
    --set full capture of this workload (profiles/), or None."""
    p = os.path.join(ROOT, "profiles", "r01_ncu_copy_traffic.json")
    if not os.path.exists(p):
        return None
    j = json.load(open(p))
    if j.get("workload") != workload or int(j.get("conns", 0)) != conns:
        return None
    return int(j["dram__bytes_read.sum"]) + int(j["dram__bytes_write.sum"])


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return float(j["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md)."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [int(s[0]) for s in self.samples if s[0].isdigit()]
        mx = [int(s[1]) for s in self.samples if s[1].isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if s[2 + k].lower() == "active"})
        return {"sm_mhz": int(statistics.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def message_bytes(data):
    """Total bytes of the distinct messages a trace delivers."""
    seen = {}
    for s, t, ln in zip(data["src"], data["msg_tag"], data["msg_len"]):
        seen[(int(s), int(t))] = int(ln)
    return sum(seen.values())


def cpu_reference(data, n_hosts, chunk_bytes, seconds, threads=None):
    """The reference's own receive path (oracle/_ref: the unmodified chunknet
    library, Transport::handle_packet replay) on this host's cores."""
    from oracle import ref
    threads = threads or os.cpu_count() or 1
    msg = message_bytes(data)
    if ref.available():
        t1 = ref.rx_replay_bench(data, n_hosts, chunk_bytes, threads, 1)
        reps = max(1, min(200, int(seconds / max(t1, 1e-3))))
        t = ref.rx_replay_bench(data, n_hosts, chunk_bytes, threads, reps)
        gbs = threads * reps * msg / t / 1e9
        return {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": "reference",
                "sample": f"{threads} threads x {reps} replays of the {len(data)}-packet "
                          f"trace (each thread its own Transport + source buffer), "
                          f"{t:.2f} s", "mpkts_per_s": round(threads * reps * len(data) / t / 1e6, 3)}
    from oracle import oracle as O
    staging = O.fill_staging(data)
    rx = O.OracleRx()
    t0 = time.perf_counter()
    reps = 0
    while time.perf_counter() - t0 < seconds / 4 or reps == 0:
        rx = O.OracleRx()
        rx.batch(data, staging)
        reps += 1
    t = time.perf_counter() - t0
    return {"value": round(reps * msg / t / 1e9, 3), "unit": "GB/s", "cores": 1, "kind": "port",
            "sample": f"{reps} single-thread oracle replays, {t:.2f} s",
            "mpkts_per_s": round(reps * len(data) / t / 1e6, 3)}


def sched_bench(dev, steps=20, conns=1024, paths=256, per_call=4096):
    """S1-S4 rows: batched select_path (p2_rtt) for `conns` connections x
    `paths` paths, `per_call` decisions per connection per call."""
    import torch

    import paper_2504_17307_b200 as cn
    s = cn.PathScheduler(conns, paths, 1, base_rtt_ns=10000.0, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(77)
    s.rtt_scores()[:] = 10000.0 + torch.randint(0, 5000, (conns, paths), device=dev,
                                                generator=g).double()
    out = torch.empty((conns, per_call), dtype=torch.int32, device=dev)
    for _ in range(3):
        s.select("p2_rtt", per_call, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        s.select("p2_rtt", per_call, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    r = {"decisions_per_s": round(conns * per_call * steps / (ms * 1e-3), 1),
         "config": f"{conns} connections x {paths} paths, p2_rtt, {per_call} decisions/conn/call",
         "ms_per_call": round(ms / steps, 4)}
    try:
        from oracle import ref
        if ref.available():
            threads = os.cpu_count() or 1
            t, _ = ref.select_paths_bench("p2_rtt", paths, conns, 2000, threads)
            r["cpu_reference_decisions_per_s"] = round(conns * 2000 / t, 1)
            r["cpu_threads"] = threads
    except Exception as e:  # noqa: BLE001
        r["cpu_reference_error"] = str(e)
    return r


def sender_bench(dev, conns=1024, scenario="cfg1", reps=3):
    """B1-B6 rows: the device sender engine (csrc/tx.cu) replaying, on each
    of `conns` connections, the recorded sender scenario (submissions + the
    acks the reference DES delivered, tests/golden/sender_<scenario>.npz):
    ack processing, fast retransmit, RTO, commit/egress with path draws."""
    import torch

    from paper_2504_17307_b200.sender import TxEngine
    z = np.load(os.path.join(ROOT, "tests", "golden", f"sender_{scenario}.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    acks, subs = z["acks"], z["submits"]
    ev = [(int(x["t"]), 0, k) for k, x in enumerate(subs)] + [(int(a["aux"]), 1, k) for k, a in enumerate(acks)]
    ev.sort()
    one = [(typ, k) for _, typ, k in ev]
    ms = []
    for r in range(reps + 1):
        eng = TxEngine(conns, chunk_bytes=meta["chunk_bytes"], rto_min=meta["rto_min"],
                       rto_max=meta["rto_max"], commit_ahead=meta["commit_ahead"],
                       base_rtt_ns=meta["base_rtt"], seed=meta["seed"], lb=meta["lb"],
                       max_paths=meta["n_paths"], src=[meta["src"]] * conns, dst=[meta["dst"]] * conns,
                       chunk_pool=conns * 2048, log_cap=max(1024, len(z["tx"]) + 16), device=dev)
        prep = eng.prepare([one] * conns, subs, acks)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.launch(prep, 60_000_000_000)
        e1.record()
        torch.cuda.synchronize()
        st = eng.stats_np()
        if r:
            ms.append(e0.elapsed_time(e1))
        ok = int(st[0]["chunk_rtx"]) == meta["stats"]["chunk_rtx"]
        eng.close()
    t = min(ms) * 1e-3
    n_tx = len(z["tx"]) * conns
    out = {"config": f"{conns} connections x sender_{scenario} ({len(acks)} acks, {len(z['tx'])} "
                     f"transmissions each; CC none)", "acks_per_s": round(conns * len(acks) / t, 1),
           "tx_decisions_per_s": round(n_tx / t, 1), "ms": round(t * 1e3, 3), "parity_chunk_rtx": ok,
           "note": "device-resident event streams; one cn_tx_run launch timed with CUDA events"}
    try:
        from oracle import ref
        if ref.available():
            threads = os.cpu_count() or 1
            kw = {k: meta[k] for k in ("chunk_bytes", "lb", "seed")}
            topo_arg = 32 if meta["n_paths"] > 16 else 8
            tc = ref.sender_replay_bench(acks, [(int(x["t"]), int(x["len"]), int(x["tag"])) for x in subs],
                                         meta["src"], meta["dst"], threads, 20, topo_arg=topo_arg,
                                         paths=meta["n_paths"], **kw)
            out["cpu_reference_acks_per_s"] = round(threads * 20 * len(acks) / tc, 1)
            out["cpu_threads"] = threads
    except Exception as e:  # noqa: BLE001
        out["cpu_reference_error"] = str(e)
    return out


def eqds_bench(dev, receivers=4096, senders=32, events=1000, reps=3, cpu_receivers=64):
    """§8(f) rank 1: the EQDS pull pacer (csrc/eqds.cu), one per receiving
    host, over synthetic incast input streams (RTS / chunk / trim events,
    `senders` per receiver); grants/s, with the reference EqdsReceiver on a
    sample of the same streams on all host threads beside it."""
    import concurrent.futures

    import torch

    from paper_2504_17307_b200.eqds import EV_DTYPE, EqdsPacers, transport_params
    P = transport_params()
    rs = np.random.RandomState(5)
    n = receivers * events
    ev = np.zeros(n, dtype=EV_DTYPE)
    dt = np.where(rs.rand(n) < 0.1, 0, rs.randint(1, 4000, size=n)).reshape(receivers, events)
    ev["t"] = np.cumsum(dt, axis=1).reshape(-1)
    u = rs.rand(n)
    ev["type"] = np.where(u < 0.15, 0, np.where(u < 0.25, 2, 1))
    ev["type"].reshape(receivers, events)[:, :senders] = 0  # every sender registers first
    ev["sender"] = (rs.randint(0, senders, size=n) + 1).reshape(-1)
    ev["sender"].reshape(receivers, events)[:, :senders] = np.arange(1, senders + 1)
    ev["arg"] = np.where(ev["type"] == 0, rs.randint(1, 64, size=n) * 32768, 32768)
    ev["flag"] = rs.rand(n) < 0.1
    off = np.arange(receivers + 1, dtype=np.uint32) * events
    ms, grants = [], 0
    for r in range(reps + 1):
        pc = EqdsPacers(receivers, quantum=P["quantum"], tick_ns=P["tick_ns"], bank_cap=P["bank_cap"],
                        max_senders=2 * senders, queue_cap=8192, log_cap=4 * events, device=dev)
        prep = pc.prepare(ev, off)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pc.launch(prep, 1 << 62)
        e1.record()
        torch.cuda.synchronize()
        if r:
            ms.append(e0.elapsed_time(e1))
        logs = pc.log_n.cpu().numpy()
        pc.close()
    t = min(ms) * 1e-3
    out = {"config": f"{receivers} receivers x {events} input events ({senders} senders each), "
                     f"quantum {P['quantum']} B, tick {P['tick_ns']} ns",
           "events_per_s": round(n / t, 1), "log_records_per_s": round(int(logs.sum()) / t, 1),
           "ms": round(t * 1e3, 3)}
    try:
        from oracle import ref
        if ref.available():
            threads = os.cpu_count() or 1
            sample = [ev[i * events:(i + 1) * events] for i in range(cpu_receivers)]
            t0 = time.perf_counter()
            with concurrent.futures.ThreadPoolExecutor(threads) as ex:  # ctypes releases the GIL
                list(ex.map(lambda e: ref.eqds_replay(e, quantum=P["quantum"], tick_ns=P["tick_ns"],
                                                      bank_cap=P["bank_cap"], max_out=4 * events), sample))
            tc = time.perf_counter() - t0
            out["cpu_reference_events_per_s"] = round(cpu_receivers * events / tc, 1)
            out["cpu_threads"] = threads
            out["cpu_sample"] = f"{cpu_receivers} of the receivers' streams"
    except Exception as e:  # noqa: BLE001
        out["cpu_reference_error"] = str(e)
    return out


def synth_trace(conns, size, chunk_bytes=32768, paths=256, seed=0, window=64, dev="cuda", conn_base=0):
    """configs[4] traffic into one receiver: `conns` connections (sources
    conn_base+1.., conn id = index & 0xFF), one `size`-byte message each,
    chunked and packetized as Transport::send_chunk does (DefaultPolicy),
    per-chunk paths from the S3 scheduler (P2-RTT over `paths` paths, one
    RngStream per connection), packets of all connections interleaved
    round-robin and reordered within a `window`-packet sliding window (the
    multipath spray).  Returns cn_pkt_hdr records (numpy PKT_DTYPE)."""
    import torch

    import paper_2504_17307_b200 as cn
    from paper_2504_17307_b200.records import PKT_DTYPE
    nch = -(-size // chunk_bytes)
    ppc = -(-chunk_bytes // MAX_PL)
    last = size - (nch - 1) * chunk_bytes
    lp = -(-last // MAX_PL)
    per = (nch - 1) * ppc + lp
    sch = cn.PathScheduler(conns, paths, seed + 1, base_rtt_ns=10000.0, device=dev)
    pth = sch.select("p2_rtt", nch).cpu().numpy()                      # [conns, nch]
    k = np.arange(per)
    c = np.minimum(k // ppc, nch - 1)
    sq = k - c * ppc
    clen = np.where(c == nch - 1, last, chunk_bytes)
    pl = np.minimum(MAX_PL, clen - sq * MAX_PL)
    rec = np.zeros((conns, per), dtype=PKT_DTYPE)
    j = np.arange(conns)[:, None]
    rec["src"] = conn_base + 1 + j
    rec["dst"] = 0
    rec["path_id"] = pth[:, c]
    hdr = ((j & 0xFF) << 24) | (0 << 17) | ((c & 0xFF) << 9) | ((c == nch - 1) << 8)
    rec["hdr"] = hdr.astype(np.uint32)
    rec["chunk_offset"] = (c * chunk_bytes)[None, :]
    rec["chunk_len"] = clen[None, :]
    rec["payload_len"] = pl[None, :]
    rec["seq_in_chunk"] = sq[None, :]
    rec["tx_time"] = k[None, :] * 10
    rec["msg_seq"] = 1
    rec["msg_tag"] = conn_base + j
    rec["msg_len"] = size
    out = rec.T.reshape(-1)                                            # round-robin over connections
    if window > 1 and len(out) > window:
        rs = np.random.RandomState(seed)
        key = np.arange(len(out)) + rs.randint(0, window, len(out))
        out = out[np.argsort(key, kind="stable")]
    return out


def sweep_bench(dev, world, rank, sizes=(4 << 10, 64 << 10, 1 << 20, 16 << 20, 256 << 20, 1 << 30),
                total_conns=1024, cap_bytes=2 << 30, steps=10, warmup=3):
    """BASELINE configs[4]: flow-collision sweep -- 1k connections x 256
    paths into the receive path, message sizes 4 KiB..1 GiB (connections per
    size capped so that <= 2 GiB of messages are in flight per GPU); the
    connections shard over the ranks.  Per size: one batch
    = every packet of every connection (reset + receive path, CUDA graph),
    time = max over ranks."""
    import torch
    import torch.distributed as dist

    import paper_2504_17307_b200 as cn
    out = []
    for size in sizes:
        conns = max(1, min(total_conns // world, cap_bytes // size))
        data = synth_trace(conns, size, seed=size % 9973 + rank, conn_base=rank * conns, dev=dev)
        n = len(data)
        hdrs = cn.to_device_records(data, dev)
        st = torch.randint(0, 256, (n * MAX_PL,), dtype=torch.uint8, device=dev)
        nchk = conns * (-(-size // 32768))
        tr = cn.Transport(cn.TransportConfig(chunk_bytes=32768, carry_payload=True), device=dev,
                          arena_bytes=conns * (size + 64) + (1 << 20), chunk_pool=2 * nchk + 64,
                          max_batch=n, max_conns=2 * conns + 16, max_msgs=2 * conns + 16)

        def step():
            s_ = torch.cuda.current_stream(dev)
            tr.reset(s_)
            tr.rx_batch_async(hdrs, st, MAX_PL, s_)

        step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        for _ in range(warmup):
            g.replay()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / steps], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        res = torch.empty(24, dtype=torch.uint8).copy_(tr._result)
        r = cn.lib  # noqa: F841
        from paper_2504_17307_b200 import _lib as L_
        rr = L_.RxResult.from_buffer_copy(bytes(res.numpy()))
        assert rr.status == 0 and rr.n_completions == conns, (size, rr.status, rr.n_completions)
        out.append({"msg_bytes": size, "connections": conns * world, "packets": n * world,
                    "ms_per_batch": round(ms, 4),
                    "GBps": round(world * conns * size / (ms * 1e-3) / 1e9, 1),
                    "Mpkts_per_s": round(world * n / (ms * 1e-3) / 1e6, 1)})
        del tr, g, hdrs, st
        torch.cuda.empty_cache()
    return out


def moe_routing(world, tokens, topk=8, experts_per_rank=32, hot=0, skew=10.0):
    """DeepSeek-V3-shaped routing for every rank (deterministic): each token
    picks `topk` distinct experts (Gumbel top-k), experts on rank `hot`
    weighted so that rank receives ~skew x the average per-rank load.
    Returns per source rank: (token index order grouped by destination rank,
    rows sent to each destination)."""
    E = world * experts_per_rank
    w = np.ones(E)
    others = world - 1
    # share(hot) / share(other) = skew  ->  per-expert weight ratio = skew
    w[hot * experts_per_rank:(hot + 1) * experts_per_rank] = skew
    out = []
    for s in range(world):
        rs = np.random.RandomState(1000 + s)
        g = np.log(w)[None, :] - np.log(-np.log(rs.rand(tokens, E)))
        top = np.argpartition(-g, topk - 1, axis=1)[:, :topk]       # [tokens, topk] experts
        dest = top // experts_per_rank
        order = np.argsort(dest.reshape(-1), kind="stable")          # copies grouped by destination
        tok = np.repeat(np.arange(tokens), topk)[order]
        rows = np.bincount(dest.reshape(-1), minlength=world)
        out.append((tok, rows))
    del others
    return out


def moe_bench(dev, world, rank, tokens=4096, hidden=7168, iters=5, warmup=2):
    """BASELINE configs[3]: 8-rank MoE all-to-all (DeepSeek-V3 shape: hidden
    7168 bf16 = 14,336 B per token copy, top-8 of 32 experts per rank) with
    incast -- rank 0's experts draw 10x the average load.  One step =
    dispatch (token copies to their experts' ranks) + combine (expert outputs
    back), through the transport all-to-all; NCCL all_to_all_single with the
    same splits beside it.  Time = max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2504_17307_b200.alltoall import AllToAll
    row = hidden * 2
    routing = moe_routing(world, tokens)
    rows = np.stack([r_[1] for r_ in routing])                     # [src, dst] rows
    rows_self = rows.copy()
    np.fill_diagonal(rows, 0)                                      # local experts need no transfer
    tok, _ = routing[rank]
    g = torch.Generator(device=dev)
    g.manual_seed(rank)
    x = torch.randn(tokens, hidden, device=dev, generator=g).to(torch.bfloat16)
    idx = torch.from_numpy(tok).to(dev)
    send = x.index_select(0, idx).view(torch.uint8).reshape(-1)    # dispatch payload, grouped by dest
    offs = np.concatenate([[0], np.cumsum(rows_self[rank])[:-1]]) * row
    sc, rc = rows[rank] * row, rows[:, rank] * row
    cap = int(max(rows.max() * row, 16))
    # pieces: about 8 per hot receiver's inbound volume (the receive path runs
    # once per piece, so fewer, larger pieces when the incast is heavy)
    inbound = int(rows.sum(0).max()) * row
    pb = max(64 << 20, (inbound // 8) >> 20 << 20)
    if os.environ.get("CN_A2A_PIECE_MB"):
        pb = int(os.environ["CN_A2A_PIECE_MB"]) << 20
    a2a = AllToAll(cap, piece_bytes=pb)   # dispatch
    a2c = AllToAll(cap, piece_bytes=pb)   # combine (its own slots: the dispatch slots are its send buffer)
    coffs = [s_ * a2a.cap for s_ in range(world)]

    def step():
        recv = a2a.run(send, sc, rc, send_offsets=offs)
        # combine: expert outputs (here: the received rows) return to their owners
        a2c.run(recv, rc, sc, send_offsets=coffs)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h0 = time.perf_counter()
    for _ in range(iters):
        step()
    host_ms = (time.perf_counter() - h0) * 1e3 / iters
    e1.record()
    torch.cuda.synchronize()
    a2a.check()
    a2c.check()
    t = torch.tensor([e0.elapsed_time(e1) / iters], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    # NCCL all_to_all_single with the same splits (local rows excluded on both sides)
    inp = torch.empty(int(sc.sum()), dtype=torch.uint8, device=dev)
    out = torch.empty(int(rc.sum()), dtype=torch.uint8, device=dev)
    sl, rl = [int(v) for v in sc], [int(v) for v in rc]

    def nstep():
        dist.all_to_all_single(out, inp, rl, sl)
        dist.all_to_all_single(inp, out, sl, rl)

    for _ in range(warmup):
        nstep()
    torch.cuda.synchronize()
    dist.barrier()
    e0.record()
    for _ in range(iters):
        nstep()
    e1.record()
    torch.cuda.synchronize()
    tn = torch.tensor([e0.elapsed_time(e1) / iters], device=dev, dtype=torch.float64)
    dist.all_reduce(tn, op=dist.ReduceOp.MAX)
    msn = float(tn.item())
    a2a.close()
    a2c.close()
    moved = int(rows.sum()) * row * 2  # dispatch + combine, all ranks
    hot_in = int(rows[:, 0].sum()) * row
    return {"piece_bytes": pb,
            "config": f"{world} ranks x {tokens} tokens, hidden {hidden} bf16 ({row} B/copy), top-8 of "
                      f"{32 * world} experts, rank 0 experts 10x weight (incast)",
            "ms_per_step": round(ms, 4), "nccl_ms_per_step": round(msn, 4),
            "host_enqueue_ms_per_step": round(host_ms, 4),
            "bytes_per_step_all_ranks": moved, "hot_rank_ingress_bytes": hot_in,
            "hot_rank_ingress_GBps": round(hot_in / (ms / 2 * 1e-3) / 1e9, 1),
            "algbw_GBps_all_ranks": round(moved / (ms * 1e-3) / 1e9, 1),
            "nccl_algbw_GBps_all_ranks": round(moved / (msn * 1e-3) / 1e9, 1)}


def ring_bench(dev, world, rank, iters=8, warmup=3, nbytes=1 << 30, piece_bytes=32 << 20):
    """BASELINE configs[2]: ring all-reduce of 1 GiB per rank (fp32 and bf16)
    through the transport (packetize -> NVLink zero-copy fused-reduce receive
    path), busbw = (S/t)*2(N-1)/N, max over ranks; NCCL's all_reduce on the
    same buffers beside it."""
    import torch
    import torch.distributed as dist

    from paper_2504_17307_b200.collective import RingAllreduce, busbw
    out = {}
    for dt, name in ((torch.float32, "fp32"), (torch.bfloat16, "bf16")):
        count = nbytes // (4 if dt == torch.float32 else 2)
        x = torch.randn(count, device=dev).to(dt)
        ring = RingAllreduce(count, dt, chunk_bytes=32768, paths=8, piece_bytes=piece_bytes)
        ring.buffer().copy_(x)
        ring.run()  # eager once, then one captured iteration replayed in place
        ring.capture()
        for _ in range(warmup):  # in place, like dist.all_reduce(y) below
            ring.run()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            ring.run()
        e1.record()
        torch.cuda.synchronize()
        ring.check()
        t = torch.tensor([e0.elapsed_time(e1) / iters], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        # NCCL on the same buffer size for context
        y = x.clone()
        for _ in range(warmup):
            dist.all_reduce(y)
        torch.cuda.synchronize()
        dist.barrier()
        e0.record()
        for _ in range(iters):
            dist.all_reduce(y)
        e1.record()
        torch.cuda.synchronize()
        tn = torch.tensor([e0.elapsed_time(e1) / iters], device=dev, dtype=torch.float64)
        dist.all_reduce(tn, op=dist.ReduceOp.MAX)
        msn = float(tn.item())
        out[name] = {"bytes": nbytes, "ms": round(ms, 4), "busbw_GBps": round(busbw(nbytes, ms * 1e-3, world), 1),
                     "pieces_per_step": ring.pieces,
                     "nccl_ms": round(msn, 4),
                     "nccl_busbw_GBps": round(busbw(nbytes, msn * 1e-3, world), 1)}
        ring.close()
        del x, y
        torch.cuda.empty_cache()
    out["roofline"] = {"bound": "nvlink", "peak_GBps_per_direction": 770.0,
                       "note": "measured peer copy per direction (B200_PROFILING.md); busbw ~ link rate"}
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    data1, meta, n_acks = load_trace(args.workload)
    data = interleave(data1, max(1, args.conns))
    from oracle import ref
    threads = os.cpu_count() or 1
    msg = message_bytes(data)
    if not ref.available():
        emit({"impl": "reference", "unavailable": "oracle/_ref not built"})
        return
    for _ in range(args.warmup):
        ref.rx_replay_bench(data, meta["n_hosts"], meta["chunk_bytes"], threads, 1)
    times = [ref.rx_replay_bench(data, meta["n_hosts"], meta["chunk_bytes"], threads, 1)
             for _ in range(args.steps)]
    t = sum(times)
    v = threads * args.steps * msg / t / 1e9
    line = {
        "metric": "reassembly_GBps", "value": round(v, 3), "unit": "GB/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * t / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "reference DES trace",
        "config": {"workload": f"{args.workload}: BASELINE configs[1] (64 MiB message, 256 paths, "
                               f"1% drop) x {args.conns} concurrent connections per batch; "
                               f"{threads} threads each replay it into its own Transport"},
        "mpkts_per_s": round(threads * args.steps * len(data) / t / 1e6, 3),
        "cpu_baseline": {"value": round(v, 3), "unit": "GB/s", "cores": threads,
                         "kind": "reference",
                         "sample": f"{threads} threads x 1 replay per step"},
        "e2e": {"value": round(v, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    emit(line)


_JSON_FD = None


def emit(line):
    """The one JSON line on the real stdout: library chatter (NCCL's version
    banner, CUDA/C printf) is sent to stderr while the bench runs."""
    os.write(_JSON_FD if _JSON_FD is not None else 1, (json.dumps(line) + "\n").encode())


def main():
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_2504_17307_b200 as cn

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    data1, meta, _ = load_trace(args.workload)
    K = max(1, args.conns)
    data = interleave(data1, K)
    n = len(data)
    msg_len = int(data["msg_len"][0])
    cb = meta["chunk_bytes"]

    hdrs = cn.to_device_records(data, dev)
    # synthetic payload: random message bytes on device (one message per
    # connection), gathered into the arrival-order staging slots (packet i
    # at i*4032) -- setup, untimed
    off = torch.from_numpy((data["chunk_offset"] + data["seq_in_chunk"].astype(np.uint64) * MAX_PL)
                           .astype(np.int64)).to(dev)
    pl = torch.from_numpy(data["payload_len"].astype(np.int64)).to(dev)
    conn_of = torch.from_numpy(data["msg_tag"].astype(np.int64)).to(dev)
    R = max(1, args.replicas if K == 1 else 2)
    srcs, stagings = [], []
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    col = torch.arange(MAX_PL, device=dev)
    for r in range(R):
        src = torch.randint(0, 256, (K, msg_len), dtype=torch.uint8, device=dev, generator=g)
        flat = src.view(-1)
        st = torch.zeros(n * MAX_PL, dtype=torch.uint8, device=dev)
        for a in range(0, n, 2048):
            b = min(n, a + 2048)
            pos = off[a:b, None] + col[None, :]
            mask = col[None, :] < pl[a:b, None]
            vals = flat[conn_of[a:b, None] * msg_len + pos.clamp(max=msg_len - 1)]
            st.view(n, MAX_PL)[a:b] = torch.where(mask, vals, torch.zeros_like(vals))
        srcs.append(src)
        stagings.append(st)

    tr = cn.Transport(cn.TransportConfig(chunk_bytes=cb, carry_payload=True), device=dev,
                      arena_bytes=K * (msg_len + (1 << 20)), chunk_pool=4 * K * ((msg_len + cb - 1) // cb),
                      max_batch=n, max_conns=64, max_msgs=64)
    stream = torch.cuda.current_stream(dev)

    def step(k, s=None):
        s = s or torch.cuda.current_stream(dev)
        tr.reset(s)
        tr.rx_batch_async(hdrs, stagings[k % R], MAX_PL, s)

    def check_buffers(r):
        arena = tr.arena()
        cp = tr.completions_np(K)
        assert len(cp) == K
        for c in cp:
            o = int(c["buf_offset"])
            assert torch.equal(arena[o: o + msg_len], srcs[r][int(c["tag"])]), \
                "reassembled message != source"

    # correctness gate before timing: ack count + reassembled bytes
    tr.reset(stream)
    out = tr.handle_packets(hdrs, stagings[0], MAX_PL, stream)
    check_buffers(0)
    n_acks = int(out.result.n_acks)
    bytes_copied = int(out.result.bytes_copied)
    assert bytes_copied == K * msg_len
    launches = tr.last_launches() + 1  # + the reset kernel

    # one CUDA graph per staging replica: reset + the 4 receive kernels
    graphs = []
    for r in range(R):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step(r)
        graphs.append(g)
    torch.cuda.synchronize()

    for k in range(args.warmup):
        graphs[k % R].replay()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for k in range(args.steps):
            graphs[k % R].replay()
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = e0.elapsed_time(e1)
        # per-kernel CUDA-event pass (eager launches, same inputs) for the roofline
        tr.set_profiling(True)
        tr.kernel_profile(reset=True)
        for k in range(args.steps):
            step(k, stream)
        torch.cuda.synchronize()
        tr.set_profiling(False)
        prof, nb = tr.kernel_profile(reset=True)
    # last step's buffers must equal their sources (the work was really done)
    check_buffers((args.steps - 1) % R)

    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_step = ms_max / args.steps
    value = world * K * msg_len * args.steps / (ms_max * 1e-3) / 1e9
    mpkts = world * n * args.steps / (ms_max * 1e-3) / 1e6

    # roofline of the dominant kernel (k_copy: the payload scatter)
    peak, peak_kind = peaks()
    work_ms = prof["copy"] / max(nb, 1)
    algo_work = 2 * bytes_copied + HDR * n
    achieved = algo_work / (work_ms * 1e-3) / 1e9
    algo_step = 2 * bytes_copied + HDR * n + ACK * n_acks
    step_gbs = algo_step / (ms_step * 1e-3) / 1e9

    # end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        h_hdr = hdrs.cpu().pin_memory()
        h_st = [s.cpu().pin_memory() for s in stagings[:2]]
        d_hdr = torch.empty_like(hdrs)
        d_st = torch.empty_like(stagings[0])
        h_acks = torch.empty((n_acks + 16) * ACK, dtype=torch.uint8).pin_memory()
        h_res = torch.empty(24, dtype=torch.uint8).pin_memory()

        def e2e_step(k):
            d_hdr.copy_(h_hdr, non_blocking=True)
            d_st.copy_(h_st[k % 2], non_blocking=True)
            tr.reset(stream)
            tr.rx_batch_async(d_hdr, d_st, MAX_PL, stream)
            h_acks[: n_acks * ACK].copy_(tr._acks[: n_acks * ACK], non_blocking=True)
            h_res.copy_(tr._result, non_blocking=True)

        for k in range(args.warmup):
            e2e_step(k)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for k in range(args.steps):
            e2e_step(k)
        f1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([f0.elapsed_time(f1)], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": round(world * K * msg_len * args.steps / (float(te.item()) * 1e-3) / 1e9, 3),
               "unit": "GB/s", "h2d_bytes_per_step": int(hdrs.numel() + stagings[0].numel()),
               "d2h_bytes_per_step": int(n_acks * ACK + 24),
               "path": "pinned host records+staging -> cn_rx_batch (C ABI) -> acks to host"}

    sched = sched_bench(dev) if not args.no_sched else None
    sender = sender_bench(dev) if not args.no_sched and rank == 0 else None
    eqds = eqds_bench(dev) if not args.no_sched and rank == 0 else None
    ring = ring_bench(dev, world, rank, piece_bytes=args.piece_mb << 20) if world > 1 and not args.no_ring else None
    moe = moe_bench(dev, world, rank) if world > 1 and not args.no_moe else None
    sweep = sweep_bench(dev, world, rank) if not args.no_sweep else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_reference(data, meta["n_hosts"], cb, args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": "reassembly_GBps", "value": round(value, 3), "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "reference DES trace + random payload",
            "config": {"workload": f"{args.workload}: BASELINE configs[1] (64 MiB message, "
                                   f"256 paths, 1% drop) x {K} concurrent connections per batch "
                                   f"(round-robin interleaved); {n} pkts, {n_acks} acks, chunk {cb} B",
                       "l2": f"inputs larger than L2: {R} rotating staging replicas "
                             f"({R * n * MAX_PL / 1e6:.0f} MB) + 64 MiB output per step",
                       "parallelism": f"replicas x{world} (shard by connection)"},
            "mpkts_per_s": round(mpkts, 3),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": copy_traffic(args.workload, K),
                         "kernel": "k_copy (payload scatter of first arrivals)",
                         "algorithmic_bytes_per_launch": algo_work,
                         "kernel_ms": round(work_ms, 5), "peak_kind": peak_kind,
                         "step_frac": round(step_gbs / peak, 4),
                         "step_algorithmic_bytes": algo_step},
            "kernel_ms_per_step": {k: round(v / max(nb, 1), 5) for k, v in prof.items()},
            "gpu_launches": launches * args.steps,
            "clocks": clk.summary(),
        }
        if e2e:
            line["e2e"] = e2e
        if sched:
            line["scheduler"] = sched
        if sender:
            line["sender"] = sender
        if eqds:
            line["eqds"] = eqds
        if ring:
            line["allreduce"] = ring
        if moe:
            line["moe_alltoall"] = moe
        if sweep:
            line["sweep_cfg5"] = sweep
        if cpu:
            line["cpu_baseline"] = cpu
        emit(line)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
