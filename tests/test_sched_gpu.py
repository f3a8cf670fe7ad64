"""Parity of the device scheduler (csrc/sched.cu) with the reference's
RngStream / select_path (golden sequences from the compiled reference,
tests/golden/rng.npz) and the C oracle."""
import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _u64(t):
    return t.cpu().numpy().view(np.uint64)


def test_raw_streams_match_reference(rng_golden):
    import paper_2504_17307_b200 as cn
    g = rng_golden
    for idx in (0, 1, 2, 255, 1023):
        s = cn.PathScheduler(1, 1, 1, index0=idx)
        assert (_u64(s.draws(0, 1000)) == g[f"u64_conn{idx}"]).all(), idx
    s = cn.PathScheduler(1, 1, 42, stream_name="loss", index0=7)
    assert (_u64(s.draws(0, 1000)) == g["u64_named_loss7"]).all()
    s = cn.PathScheduler(1, 1, 9, stream_name="workload", index0=-1)
    assert (_u64(s.draws(0, 1000)) == g["u64_unindexed"]).all()


def test_next_below_matches_reference(rng_golden):
    import paper_2504_17307_b200 as cn
    g = rng_golden
    s = cn.PathScheduler(1, 1, 3, index0=17)
    ns = torch.from_numpy(g["below_ns"].view(np.int64).copy())
    assert (_u64(s.draws(0, ns=ns)) == g["below_vals"]).all()


@pytest.mark.parametrize("n", [1, 2, 7, 8, 256])
@pytest.mark.parametrize("pol", ["oblivious", "p2_rtt", "p2_ecn"])
def test_select_path_sequences_match_reference(rng_golden, n, pol):
    import paper_2504_17307_b200 as cn
    g = rng_golden
    # connections 0..5 share the board; reference sequences exist for 0 and 5
    s = cn.PathScheduler(6, n, 1)
    s.rtt_scores()[:] = torch.from_numpy(g[f"board{n}_rtt"]).cuda()
    s.ecn_scores()[:] = torch.from_numpy(g[f"board{n}_ecn"]).cuda()
    # several calls of uneven sizes: the stream state persists across calls
    outs = [s.select(pol, c) for c in (7, 300, 1, 1000, 692)]
    seq = torch.cat(outs, dim=1).cpu().numpy()
    for idx in (0, 5):
        assert (seq[idx] == g[f"sel_{pol}_{n}_{idx}"]).all(), idx
    for idx in (1, 2, 3, 4):
        want = O.select_paths(pol, g[f"board{n}_rtt"], g[f"board{n}_ecn"], 1, "transport.conn",
                              idx, 2000)
        assert (seq[idx] == want).all(), idx


def test_rtx_avoid_prev_path_and_grouping():
    """DefaultPolicy::on_tx_rtx_chunk: same draws, previous path avoided."""
    import paper_2504_17307_b200 as cn
    rs = np.random.RandomState(3)
    n = 16
    rtt = 10000.0 + rs.randint(0, 3000, size=n)
    s = cn.PathScheduler(4, n, 1)
    s.rtt_scores()[:] = torch.from_numpy(np.tile(rtt, (4, 1))).cuda()
    cnt = [50, 0, 33, 100]
    offs = torch.tensor(np.concatenate([[0], np.cumsum(cnt)]), dtype=torch.int32).cuda()
    conns = torch.tensor([0, 1, 2, 3], dtype=torch.int32).cuda()
    prev = rs.randint(-1, n, size=sum(cnt)).astype(np.int32)
    out = s.select("p2_rtt", conns=conns, offsets=offs, prev_paths=torch.from_numpy(prev).cuda())
    out = out.cpu().numpy()
    o = 0
    for c, k in enumerate(cnt):
        base = O.select_paths("p2_rtt", rtt, np.zeros(n), 1, "transport.conn", c, k)
        want = np.where((prev[o:o + k] >= 0) & (base == prev[o:o + k]), (base + 1) % n, base)
        assert (out[o:o + k] == want).all()
        o += k


def test_scoreboard_ewma_matches_reference_arithmetic():
    """PathScoreboard::record_rtt/record_ecn (lb.hpp:23-28), test_lb.cpp:10-32."""
    import paper_2504_17307_b200 as cn
    s = cn.PathScheduler(1, 2, 0, base_rtt_ns=10000.0)
    conn = torch.zeros(2, dtype=torch.int32).cuda()
    path = torch.zeros(2, dtype=torch.int32).cuda()
    rtt = torch.full((2,), 18000, dtype=torch.int64).cuda()
    ecn = torch.zeros(2, dtype=torch.uint8).cuda()
    offs = torch.tensor([0, 2], dtype=torch.int32).cuda()
    s.record(conn, path, rtt, ecn, offs)
    b = s.rtt_scores().cpu().numpy()
    assert b[0, 0] == 11875.0 and b[0, 1] == 10000.0
