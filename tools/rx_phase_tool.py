"""Profiling helper (not a test): phase marks inside the receive kernels of a
CN_RX_TIMING build (make EXTRA=-DCN_RX_TIMING; CHUNKNET_B200_LIB=<that .so>),
steady-state headline batches (msg_seq + 1 per step, no reset), eager.
    python tools/rx_phase_tool.py [K] [steps]"""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
NAMES = {0: "fin start", 1: "fin dirty-clear", 2: "fin adv pool", 3: "fin adv arena", 4: "fin tiles",
         5: "fin arena release", 6: "fin retire", 7: "fin end", 10: "ing start", 11: "ing conn", 12: "ing gen",
         13: "ing end", 20: "scan start", 21: "scan end", 22: "acks start", 23: "acks end", 24: "copy start",
         25: "copy end", 30: "scan plan start", 31: "scan plan lens", 32: "scan plan placed", 34: "fin plan start",
         35: "fin plan lens", 36: "fin plan placed"}


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    import bench
    import paper_2504_17307_b200 as cn
    from paper_2504_17307_b200 import _lib
    from paper_2504_17307_b200.records import PKT_DTYPE
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    if os.environ.get("SYNTH"):
        c_, b_ = (int(v) for v in os.environ["SYNTH"].split("x"))
        mpc = int(os.environ.get("SYNTH_MPC", "1"))  # messages per connection
        data, cb, msg_len, K = bench.synth_trace(c_, b_, seed=1, msgs=mpc), 32768, b_, c_ * mpc
    else:
        data, meta, _ = bench.load_trace(os.environ.get("TRACE", "cfg2_32k"))
        data = bench.interleave(data, K)
        cb, msg_len = meta["chunk_bytes"], int(data["msg_len"][0])
    n = len(data)
    hdrs = cn.to_device_records(data, dev)
    seq_col = hdrs.view(n, 64).view(torch.int64)[:, PKT_DTYPE.fields["msg_seq"][1] // 8]
    st = torch.randint(0, 256, (n * bench.MAX_PL,), dtype=torch.uint8, device=dev)
    tr = cn.Transport(cn.TransportConfig(chunk_bytes=cb, carry_payload=True), device=dev,
                      arena_bytes=3 * K * (msg_len + (1 << 20)), chunk_pool=3 * K * ((msg_len + cb - 1) // cb),
                      max_batch=n, max_conns=max(64, 2 * K + 8), max_msgs=max(64, 2 * K + 8))
    lib = _lib.lib()
    fn = lib.cn_rx_debug_timing
    fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
    buf = (ctypes.c_ulonglong * 64)()
    s = torch.cuda.current_stream(dev)
    fn(buf, 64)
    for k in range(steps):
        seq_col.add_(1)
        torch.cuda.synchronize()
        fn(buf, 64)
        tr.rx_batch_async(hdrs, st, bench.MAX_PL, s)
        torch.cuda.synchronize()
        fn(buf, 64)
        t0 = buf[10]
        marks = sorted((buf[j] - t0, NAMES[j]) for j in NAMES if 0 < buf[j] < (1 << 63))
        print(f"--- step {k}: " + "  ".join(f"{nm} {v / 1e3:.1f}" for v, nm in marks))
        if os.environ.get("INGEST") == "1" and k == steps - 1:  # k_ingest per-packet-block marks
            import numpy as np
            ib = (ctypes.c_ulonglong * (5 * 64))()
            lib.cn_rx_debug_ingest_timing.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
            lib.cn_rx_debug_ingest_timing(ib)
            a = np.frombuffer(ib, dtype=np.uint64).reshape(5, 64).astype(np.int64)
            nb = int((a[3] > 0).sum())
            a = a[:, :nb]
            print(f"ingest packet blocks {nb}: start after the first block (us) " +
                  " ".join(f"{(v - buf[10]) / 1e3:.1f}" for v in a[0][:16]))
            for nm, x, y in (("hdr load", 0, 4), ("conn", 4, 1), ("gen", 1, 2), ("chunks", 2, 3), ("block", 0, 3)):
                dd = (a[y] - a[x]) / 1e3
                print(f"  {nm:9s} p50 {np.median(dd):.2f} max {dd.max():.2f} us")
        if os.environ.get("TILES") == "1" and k == steps - 1:  # k_acks per-tile marks
            import numpy as np
            tb = (ctypes.c_ulonglong * (4 * 8192))()
            lib.cn_rx_debug_tile_timing.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
            lib.cn_rx_debug_tile_timing(tb)
            a = np.frombuffer(tb, dtype=np.uint64).reshape(4, 8192).astype(np.int64)
            nt = int((a[3] > 0).sum())
            a = a[:, :nt]
            a0 = buf[22]
            st = (a[0] - a0) / 1e3
            print(f"tiles {nt}: start  p10 {np.percentile(st, 10):.1f} p50 {np.median(st):.1f} "
                  f"p90 {np.percentile(st, 90):.1f} max {st.max():.1f} us after the first block")
            for nm, x, y in (("decide", 0, 1), ("build", 1, 2), ("write", 2, 3), ("tile", 0, 3)):
                dd = (a[y] - a[x]) / 1e3
                print(f"  {nm:7s} p50 {np.median(dd):.2f} p90 {np.percentile(dd, 90):.2f} max {dd.max():.2f} us")
            order = np.argsort(a[0])
            print("  tiles started per 5 us:", np.histogram(st, bins=np.arange(0, st.max() + 5, 5))[0].tolist())


if __name__ == "__main__":
    main()
