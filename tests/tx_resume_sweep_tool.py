"""Diagnostic (GPU, not collected by pytest): the sender engine resumed across
cn_tx_run calls -- every selective-mode single-connection scenario (CC none
and Swift) and every host-level scenario (fan-out, engines, conn_split,
CUBIC, per-path scope, receiver-driven) handed over in 2 to 64 time slices,
each checked against the reference transmit log.  Run it on the uniformity
debug build to check that every decision value is equal in all 32 lanes
(a divergent one sets CN_TX_STATUS_INTERNAL and the replay raises):
    make -C paper_2504_17307_b200/csrc EXTRA=-DCN_TX_CHECK_UNIFORM -B
    python tests/tx_resume_sweep_tool.py"""
import glob
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from conftest import GOLDEN  # noqa: E402
import test_host_gpu as H  # noqa: E402
import test_tx_gpu as T  # noqa: E402

names = sorted(os.path.basename(p)[7:-4] for p in glob.glob(os.path.join(GOLDEN, "sender_*.npz")))
# selective mode, DefaultPolicy (incl. the trim-storm incasts); the policy,
# receiver-driven and ordered replays need their own engine configuration
names = [n for n in names if not n.startswith(("rr_", "single_", "user_", "eqds", "ordered", "swift_eqds",
                                              "swift_ordered"))]
hosts = sorted(os.path.basename(p)[5:-4] for p in glob.glob(os.path.join(GOLDEN, "host_*.npz")))
bad = runs = 0
for n in names:
    for ns in (2, 3, 5, 9, 17, 31, 42, 64):
        runs += 1
        try:
            T.test_tx_engine_resumes_across_runs(n, ns)
        except Exception as e:  # noqa: BLE001
            bad += 1
            print("FAIL", n, ns, type(e).__name__, str(e)[:200], flush=True)
for n in hosts:
    for ns in (2, 5, 17, 64):
        runs += 1
        try:
            H.test_host_engine_resumes_across_runs(n, ns)
        except Exception as e:  # noqa: BLE001
            bad += 1
            print("FAIL host", n, ns, type(e).__name__, str(e)[:200], flush=True)
print(f"resume sweep: {len(names)} connection scenarios x 8 slicings + {len(hosts)} host scenarios x 4 "
      f"slicings = {runs} resumed replays, {bad} failures", flush=True)
