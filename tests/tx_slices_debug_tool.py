"""Debug helper (not a test): replay a sender golden through TxEngine with
the input events handed over in NSLICE time slices (state persisting across
cn_tx_run calls) and compare the transmit log.  Usage:
    python tests/tx_slices_debug_tool.py NAME NSLICE"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(name, nslice):
    import ctypes
    import torch
    from paper_2504_17307_b200.sender import TxEngine
    torch.zeros(1, device="cuda")
    if os.environ.get("CN_STACK"):
        rt = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so.12")
        print("set stack", rt.cudaDeviceSetLimit(0, ctypes.c_size_t(int(os.environ["CN_STACK"]))))
    z = np.load(os.path.join(ROOT, "tests", "golden", f"sender_{name}.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    eng = TxEngine(1, chunk_bytes=meta["chunk_bytes"], rto_min=meta["rto_min"], rto_max=meta["rto_max"],
                   commit_ahead=meta["commit_ahead"], base_rtt_ns=meta["base_rtt"], seed=meta["seed"],
                   lb=meta["lb"], max_paths=meta["n_paths"], src=[meta["src"]], dst=[meta["dst"]],
                   chunk_pool=1 << 18, log_cap=1 << 17, cc=meta.get("cc", "none"),
                   swift_target_ns=meta.get("swift_target_ns", 0))
    subs, acks = z["submits"], z["acks"]
    ev = sorted([(int(s["t"]), 0, k) for k, s in enumerate(subs)] + [(int(a["aux"]), 1, k) for k, a in enumerate(acks)])
    ts = sorted({e[0] for e in ev})
    cuts = [ts[int(len(ts) * (i + 1) / nslice) - 1] for i in range(nslice)]
    if os.environ.get("CN_CUTS"):
        cuts = [int(c) for c in os.environ["CN_CUTS"].split(",")] + [0]
    cuts[-1] = 60_000_000_000
    k = 0
    for c in cuts:
        part = []
        while k < len(ev) and ev[k][0] <= c:
            part.append(ev[k])
            k += 1
        sub_idx = [e[2] for e in part if e[1] == 0]
        ack_idx = [e[2] for e in part if e[1] == 1]
        s2 = subs[sub_idx] if sub_idx else subs[:0]
        a2 = acks[ack_idx] if ack_idx else acks[:0]
        # events re-indexed into this slice's arrays
        m_s = {j: i for i, j in enumerate(sub_idx)}
        m_a = {j: i for i, j in enumerate(ack_idx)}
        evs = [(0, m_s[e[2]]) if e[1] == 0 else (1, m_a[e[2]]) for e in part]
        if len(s2) == 0:
            s2 = subs[:1]
        if len(a2) == 0:
            a2 = acks[:1]
        eng.run([evs], s2, a2, c)
        print("slice to", c, "events", len(evs), flush=True)
        if os.environ.get("CN_DUMP"):
            L = eng._L
            L.cn_tx_debug_state.restype = ctypes.c_int64
            L.cn_tx_debug_state.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_uint64]
            n = L.cn_tx_debug_state(eng._h, 0, None, 0)
            buf = np.zeros(n, np.uint8)
            L.cn_tx_debug_state(eng._h, 0, buf.ctypes.data, n)
            buf.tofile(os.environ["CN_DUMP"] + f"_{c}.bin")
            return
    got, want = eng.log_np(0), z["tx"]
    print("tx", len(got), len(want))
    if len(sys.argv) > 3:
        for i in range(min(12, len(got))):
            print(i, got[i], want[i])
        print("events", ev[:40])
    for f in ("t", "msg_id", "chunk", "path", "is_rtx"):
        bad = np.nonzero(got[f][: len(want)] != want[f][: len(got)])[0]
        print(f, "mismatches", len(bad), bad[:3])


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
