"""EQDS pull pacer on the device (csrc/eqds.cu) vs the reference's own
EqdsReceiver (src/eqds.cpp) driven by the same scripted input streams
(golden tests/golden/eqds.npz, oracle/gen_fixtures.py): identical grant and
RTS-ack sequences -- time, sender, bytes, in callback order -- and grant
counts, for one receiver and for 16 independent receivers in one launch."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

SCEN = ["basic", "incast40", "noidle", "multi16"]


def _load(name):
    z = np.load(os.path.join(GOLDEN, "eqds.npz"))
    prm = json.loads(bytes(z[f"{name}_params"]).decode())
    return (prm, z[f"{name}_events"], z[f"{name}_offsets"], z[f"{name}_log"], z[f"{name}_log_offsets"],
            z[f"{name}_grants_sent"])


def test_eqds_golden_shapes():
    for name in SCEN:
        prm, ev, off, log, loff, gs = _load(name)
        assert off[-1] == len(ev) and loff[-1] == len(log) and len(gs) == len(off) - 1
        assert (log["kind"] == 0).sum() == gs.sum()  # every grant logged


@pytest.mark.gpu
@pytest.mark.parametrize("name", SCEN)
def test_eqds_pacer_matches_reference(name):
    from paper_2504_17307_b200.eqds import EqdsPacers
    prm, ev, off, log, loff, gs = _load(name)
    n = len(off) - 1
    pc = EqdsPacers(n, quantum=prm["quantum"], tick_ns=prm["tick_ns"], bank_cap=prm["bank_cap"],
                    grant_to_idle=prm["grant_to_idle"])
    pc.run(ev, off, 1 << 62)
    for r in range(n):
        got, want = pc.log_np(r), log[loff[r]:loff[r + 1]]
        st, g = pc.status(r)
        assert st == 0
        assert g == gs[r]
        assert len(got) == len(want), (r, len(got), len(want))
        for f in ("t", "sender", "bytes", "kind"):
            bad = np.nonzero(got[f] != want[f])[0]
            assert len(bad) == 0, (r, f, int(bad[0]), got[bad[0]], want[bad[0]])
    pc.close()
