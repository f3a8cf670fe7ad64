"""The collectives' progress primitives on one GPU (the multi-rank workers
skip on 1-GPU boxes): cn_copy_sm_signal copies and raises its flag from the
last block and leaves its counter zero; cn_flag_post stores; and
cn_flag_wait_signal passes on flags that are already met, then posts, and
times out (error word set) on one that is not.  No kernel here waits for
another kernel (the flags are set before the waits launch)."""
import ctypes

import pytest
import torch

from paper_2504_17307_b200 import _lib

pytestmark = pytest.mark.gpu


def _p(t):
    return ctypes.c_void_p(t.data_ptr())


def test_copy_sm_signal_raises_flag_and_resets_counter():
    L = _lib.lib()
    s = torch.cuda.current_stream()
    cs = ctypes.c_void_p(s.cuda_stream)
    src = torch.randint(0, 256, (3 << 20,), dtype=torch.uint8, device="cuda")
    dst = torch.zeros_like(src)
    flag = torch.zeros(2, dtype=torch.int64, device="cuda")
    ctr = torch.zeros(4, dtype=torch.int32, device="cuda")
    for k, (nbytes, blocks) in enumerate([(3 << 20, 64), (1 << 20, 7), (16, 32)]):
        dst.zero_()
        _lib.check(L.cn_copy_sm_signal(_p(dst), _p(src), nbytes, blocks, _p(flag), 5 + k, _p(ctr), cs),
                   "cn_copy_sm_signal")
        torch.cuda.synchronize()
        assert torch.equal(dst[:nbytes], src[:nbytes]) and not dst[nbytes:].any()
        assert int(flag[0]) == 5 + k and int(flag[1]) == 0
        assert int(ctr[0]) == 0  # left zero for the next copy on the stream
    # misaligned or empty copies are refused (they go by copy engine)
    assert L.cn_copy_sm_signal(ctypes.c_void_p(dst.data_ptr() + 1), _p(src), 32, 8, _p(flag), 1, _p(ctr), cs) != 0
    assert L.cn_copy_sm_signal(_p(dst), _p(src), 0, 8, _p(flag), 1, _p(ctr), cs) != 0


def test_flag_post_and_wait_signal():
    L = _lib.lib()
    cs = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    f = torch.zeros(4, dtype=torch.int64, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    fp = f.data_ptr()
    _lib.check(L.cn_flag_post(ctypes.c_void_p(fp), 7, cs), "cn_flag_post")
    _lib.check(L.cn_flag_post(ctypes.c_void_p(fp + 8), 3, cs), "cn_flag_post")
    # both met (7 >= 6, 3 >= 3): posts 9 into f[2]
    _lib.check(L.cn_flag_wait_signal(ctypes.c_void_p(fp), 6, ctypes.c_void_p(fp + 8), 3,
                                     ctypes.c_void_p(fp + 16), 9, 1 << 20, _p(err), cs), "cn_flag_wait_signal")
    # a wait alone (no notice), one flag
    _lib.check(L.cn_flag_wait_signal(ctypes.c_void_p(fp), 7, None, 0, None, 0, 1 << 20, _p(err), cs),
               "cn_flag_wait_signal")
    torch.cuda.synchronize()
    assert f.tolist() == [7, 3, 9, 0] and int(err[0]) == 0
    # an unmet flag: bounded spin, error word set
    _lib.check(L.cn_flag_wait_signal(ctypes.c_void_p(fp + 8), 4, None, 0, None, 0, 100, _p(err), cs),
               "cn_flag_wait_signal")
    torch.cuda.synchronize()
    assert int(err[0]) != 0
    assert L.cn_flag_wait_signal(ctypes.c_void_p(fp), 1, None, 0, None, 0, 10, None, cs) != 0
