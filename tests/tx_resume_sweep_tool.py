"""Diagnostic (GPU, not collected by pytest): the sender engine resumed across
cn_tx_run calls, every selective-mode scenario (CC none and Swift) handed over
in 2 to 64 time slices, each checked against the reference transmit log.
Run it against an alternative build of k_tx_run (csrc/tx.cu's
CN_TX_PUMP_NOINLINE / CN_TX_DEFERRED_INLINE layouts) to probe the known
layout-sensitive fault:
    python tests/tx_resume_sweep_tool.py"""
import glob, os, sys, traceback
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from conftest import GOLDEN
import test_tx_gpu as T
names = sorted(os.path.basename(p)[7:-4] for p in glob.glob(os.path.join(GOLDEN, "sender_*.npz")))
# selective mode, DefaultPolicy (incl. the trim-storm incasts); the policy,
# receiver-driven and ordered replays need their own engine configuration
names = [n for n in names if not n.startswith(("rr_", "single_", "user_", "eqds", "ordered", "swift_eqds",
                                              "swift_ordered"))]
bad = 0
for n in names:
    for ns in (2, 3, 5, 9, 17, 31, 42, 64):
        try:
            T.test_tx_engine_resumes_across_runs(n, ns)
        except Exception as e:
            bad += 1
            print("FAIL", n, ns, type(e).__name__, str(e)[:200], flush=True)
print("resume sweep:", len(names), "scenarios x 8 slicings,", bad, "failures", flush=True)
