"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/chunknet_b200.h declares, and the host-callable wire codec
matches the reference's own test vectors (proj/tests/test_wire.cpp)."""
import numpy as np
import pytest

import paper_2504_17307_b200 as cn
from paper_2504_17307_b200 import _lib
from paper_2504_17307_b200.records import PKT_DTYPE as P1, ACK_DTYPE as A1, CPL_DTYPE as C1
from oracle.records import PKT_DTYPE as P2, ACK_DTYPE as A2, CPL_DTYPE as C2


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    names = _lib.exported_symbols()
    assert len(names) >= 12
    for n in names:
        assert hasattr(L, n), n


def test_record_layouts_agree_with_oracle():
    assert P1 == P2 and A1 == A2 and C1 == C2
    assert P1.itemsize == A1.itemsize == C1.itemsize == 64


def test_header_bit_positions():  # test_wire.cpp:32-42
    assert cn.encode_header(5, 3, 200, True, 0) == 0x05079100
    assert cn.encode_header(0, 0, 0, False, 0) == 0
    assert cn.encode_header(255, 127, 255, True, 255) == 0xFFFFFFFF
    assert cn.encode_header(1, 0, 0) == 1 << 24
    assert cn.encode_header(0, 1, 0) == 1 << 17
    assert cn.encode_header(0, 0, 1) == 1 << 9
    assert cn.encode_header(0, 0, 0, True) == 1 << 8
    assert cn.encode_header(0, 0, 0, False, 1) == 1


def test_header_round_trips():  # test_wire.cpp:44-84
    for conn in range(256):
        assert cn.decode_header(cn.encode_header(conn, 9, 77, False, 3)) == (conn, 9, 77, False, 3)
    for msg in range(128):
        assert cn.decode_header(cn.encode_header(11, msg, 0, True, 255)) == (11, msg, 0, True, 255)
    for csn in range(256):
        assert cn.decode_header(cn.encode_header(0, 127, csn, False, 0)) == (0, 127, csn, False, 0)
    rs = np.random.RandomState(777)
    for w in rs.randint(0, 2**32, size=2000, dtype=np.uint64):
        assert cn.encode_header(*cn.decode_header(int(w))) == int(w)


def test_msg_id_range_error():  # test_wire.cpp:86-90
    for bad in (128, 255):
        with pytest.raises(cn.ChunknetError) as e:
            cn.encode_header(0, bad, 0)
        assert e.value.status == -3
    cn.encode_header(0, 127, 0)


def test_csn_ordering_brute_force():  # test_wire.cpp:99-127
    for w in (1, 2, 63, 100, 127, 128):
        for base in range(0, 256, 17):
            for i in range(0, w, max(1, w // 9)):
                for j in range(0, w, max(1, w // 7)):
                    a, b = (base + i) & 0xFF, (base + j) & 0xFF
                    assert cn.csn_before(a, b, base, w) == (i < j)


def test_csn_wrap_and_errors():  # test_wire.cpp:129-150
    assert cn.csn_before(254, 2, 250, 12)
    assert cn.csn_before(255, 0, 250, 12)
    assert not cn.csn_before(3, 252, 250, 12)
    assert not cn.csn_before(0, 0, 250, 12)
    for args in ((15, 12, 10, 5), (12, 9, 10, 5), (100, 200, 10, 5), (6, 250, 250, 12)):
        with pytest.raises(cn.ChunknetError) as e:
            cn.csn_before(*args)
        assert e.value.status == -4
    for w in (0, 129):
        with pytest.raises(cn.ChunknetError) as e:
            cn.csn_before(0, 0, 0, w)
        assert e.value.status == -3
