"""Profiling helper (not a test): GPU timeline of the receive-path graph
(bench.py's cfg2_32k x K workload) from CUPTI kernel records (torch.profiler),
to see launch gaps and stream overlap.  Usage:
    python tests/rx_timeline_tool.py [K] [steps]
STEADY=1: no reset between steps, msg_seq += 1 per step (bench.steady_bench)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    import bench
    import paper_2504_17307_b200 as cn
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    if os.environ.get("SYNTH"):  # SYNTH=<conns>x<bytes>: bench.synth_trace (configs[4] sweep)
        c_, b_ = (int(v) for v in os.environ["SYNTH"].split("x"))
        mpc = int(os.environ.get("SYNTH_MPC", "1"))  # messages per connection
        data = bench.synth_trace(c_, b_, seed=1, msgs=mpc)
        cb = 32768
        msg_len = b_
        K = c_ * mpc
    else:
        data, meta, _ = bench.load_trace("cfg2_32k")
        data = bench.interleave(data, K)
        cb = meta["chunk_bytes"]
        msg_len = int(data["msg_len"][0])
    n = len(data)
    hdrs = cn.to_device_records(data, dev)
    # two staging replicas, rotated per step as in bench.py (inputs larger than L2)
    sts = [torch.randint(0, 256, (n * bench.MAX_PL,), dtype=torch.uint8, device=dev) for _ in range(2)]
    st = sts[0]
    tr = cn.Transport(cn.TransportConfig(chunk_bytes=cb, carry_payload=True), device=dev,
                      arena_bytes=3 * K * (msg_len + 512) + (64 << 20), chunk_pool=4 * K * ((msg_len + cb - 1) // cb),
                      max_batch=n, max_conns=max(64, 2 * K + 8), max_msgs=max(64, 4 * K + 16))
    steady = os.environ.get("STEADY") == "1"
    if steady:
        from paper_2504_17307_b200.records import PKT_DTYPE
        seq_col = hdrs.view(n, 64).view(torch.int64)[:, PKT_DTYPE.fields["msg_seq"][1] // 8]
        tr = cn.Transport(cn.TransportConfig(chunk_bytes=cb, carry_payload=True), device=dev,
                          arena_bytes=3 * K * (msg_len + (1 << 20)), chunk_pool=3 * K * ((msg_len + cb - 1) // cb),
                          max_batch=n, max_conns=max(64, 2 * K + 8), max_msgs=max(64, 2 * K + 8))

    def step(r=0):
        s = torch.cuda.current_stream(dev)
        if steady:
            seq_col.add_(1)
        else:
            tr.reset(s)
        tr.rx_batch_async(hdrs, sts[r], bench.MAX_PL, s)

    pipe = os.environ.get("PIPE") == "1"
    if pipe:  # bench.py's headline: pipelined receiver, steady state, one graph of `steps` steps
        from paper_2504_17307_b200.records import PKT_DTYPE
        tr = cn.Transport(cn.TransportConfig(chunk_bytes=cb, carry_payload=True), device=dev,
                          arena_bytes=3 * K * (msg_len + 512) + (64 << 20),
                          chunk_pool=3 * K * ((msg_len + cb - 1) // cb) + 64,
                          max_batch=n, max_conns=max(64, 2 * K + 8), max_msgs=max(64, 4 * K + 16), pipeline=True)
        si = PKT_DTYPE.fields["msg_seq"][1] // 8
        hs = []
        for j in range(2 * steps + 1):
            h_ = hdrs.clone()
            h_.view(n, 64).view(torch.int64)[:, si] += j
            hs.append(h_)
        tr.handle_packets(hs[0], st, bench.MAX_PL)
        gs_ = []
        for r in range(2):
            g_ = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_):
                for j in range(1 + r * steps, 1 + (r + 1) * steps):
                    tr.rx_batch_async(hs[j], sts[j % 2], bench.MAX_PL, torch.cuda.current_stream(dev))
                tr.flush(torch.cuda.current_stream(dev))
            gs_.append(g_)
        gs_[0].replay()
        torch.cuda.synchronize()
        g = gs_[1]
        steps = 1

        def step():
            pass
    step()
    torch.cuda.synchronize()
    if not pipe:  # one graph per staging replica, replayed alternately
        gr = []
        for r in range(2):
            g_ = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_):
                step(r)
            gr.append(g_)

        class _Alt:
            k = 0

            def replay(self):
                gr[_Alt.k % 2].replay()
                _Alt.k += 1
        g = _Alt()
        for _ in range(5):
            g.replay()
    torch.cuda.synchronize()
    if os.environ.get("NOPROF") == "1":  # for ncu: plain replays, no CUPTI of our own
        for _ in range(steps):
            g.replay()
        torch.cuda.synchronize()
        print(f"ok: {steps} replays")
        return
    from torch.profiler import ProfilerActivity, profile
    eager = os.environ.get("EAGER") == "1"
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            if eager:
                step()
            else:
                g.replay()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    rows = sorted((e.time_range.start, e.time_range.end, e.name) for e in evs)
    t0 = rows[0][0]
    prev_reset = None
    for a, b, nm in rows:
        short = nm.split("(")[0].replace("void ", "").replace("cnb::", "")[:28]
        if ("k_reset" in short) or (steady and "elementwise" in short) or (pipe and "k_ingest" in short):
            if prev_reset is not None:
                print(f"--- step {(a - prev_reset):.1f} us")
            prev_reset = a
        print(f"{a - t0:9.1f} {b - t0:9.1f} {b - a:7.1f}  {short}")


if __name__ == "__main__":
    main()
