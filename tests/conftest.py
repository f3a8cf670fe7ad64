import glob
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def golden_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                  if os.path.basename(p) not in ("rng.npz", "trace.npz", "eqds.npz")
                  and not os.path.basename(p).startswith(("sender_", "probe_", "host_")))


def load_psn(name):
    """conn_psn per data packet of an ordered-reliability golden (None otherwise)."""
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    return z["psn"] if "psn" in z.files else None


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    return z["data"], z["acks"], z["completions"], meta


@pytest.fixture(scope="session")
def rng_golden():
    return np.load(os.path.join(GOLDEN, "rng.npz"))
