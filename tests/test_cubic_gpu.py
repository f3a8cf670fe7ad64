"""CUBIC on the device (B6 / SURVEY 8(f)2): the glibc cbrt and pow(x, 3)
restatement in csrc/libm_exact.cuh against the host libm the reference
links (10^7 inputs over CUBIC's ranges and every exponent).  The CUBIC
sender itself is pinned by the host-level goldens (test_host_gpu.py:
host_*_cubic*, closed-loop where the DES sender ran CUBIC -- BASELINE
configs[0]/[1] included)."""
import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", [0, 1])
def test_libm_restatement_matches_host(mode):
    from oracle import oracle as O
    from paper_2504_17307_b200 import _lib
    L = _lib.lib()
    x = O.libm_test_inputs(10_000_000, seed=11 + mode)
    if mode == 0:
        x = np.concatenate([np.abs(x), -np.abs(x[:1000])])
    want = O.libm(mode, x)
    dx = torch.from_numpy(x).cuda()
    dy = torch.empty_like(dx)
    _lib.check(L.cn_libm_eval(mode, dx.data_ptr(), dy.data_ptr(), len(x), None), "cn_libm_eval")
    torch.cuda.synchronize()
    got = dy.cpu().numpy()
    bad = np.nonzero(want.view(np.int64) != got.view(np.int64))[0]
    assert len(bad) == 0, (len(bad), x[bad[:3]], want[bad[:3]], got[bad[:3]])
