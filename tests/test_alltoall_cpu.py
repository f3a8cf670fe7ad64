"""Host-side piece schedule of the transport all-to-all (alltoall.py): pieces
are chunk-aligned, contiguous, cover the message exactly once, respect the
piece size, and the tail schedule puts one large head before `tail` pieces of
piece_bytes.  No GPU needed (the schedule is pure host logic)."""
import pytest

from paper_2504_17307_b200.alltoall import AllToAll


def _sched(piece, tail=0, cb=32768):
    a = AllToAll.__new__(AllToAll)  # the schedule only reads these fields
    a.piece_bytes, a.tail, a.cb = piece, tail, cb
    return a


@pytest.mark.parametrize("cnt", [1, 16, 32768, 32769, 5 << 20, (64 << 20) + 12345, 421621760])
@pytest.mark.parametrize("piece,tail", [(1 << 20, 0), (64 << 20, 0), (32 << 20, 2), (48 << 20, 3)])
def test_pieces_cover_message_chunk_aligned(cnt, piece, tail):
    a = _sched(piece, tail)
    ps = a._pieces(cnt)
    assert ps[0][0] == 0 and ps[-1][1] == cnt
    for (lo, hi), (lo2, _) in zip(ps, ps[1:]):
        assert hi == lo2 and hi > lo
    for lo, hi in ps[:-1]:
        assert lo % a.cb == 0 and hi % a.cb == 0  # chunk-aligned boundaries
    if tail and cnt > (tail + 1) * piece:
        assert len(ps) == tail + 1
        assert all(hi - lo == piece for lo, hi in ps[1:-1])
    elif not tail:
        assert all(hi - lo <= piece + a.cb for lo, hi in ps)


def test_pieces_empty_message():
    assert _sched(64 << 20)._pieces(0) == []
