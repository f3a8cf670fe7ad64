"""Profiling helper (not a test): NVLink push bandwidth from GPU 0 to GPU 1
by copy engine (1 and 2 concurrent streams), by SM kernel, and both."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2504_17307_b200 import _lib
    L = _lib.lib()
    torch.cuda.set_device(0)
    n = 256 << 20
    src = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    dst = torch.empty(n, dtype=torch.uint8, device="cuda:1")
    torch.cuda.set_device(0)
    ok = torch.cuda.can_device_access_peer(0, 1)
    print("peer access", ok)
    try:
        torch.cuda.set_device(0)
        ctypes.CDLL("libcudart.so.12").cudaDeviceEnablePeerAccess(1, 0)
    except OSError:
        pass
    ss = [torch.cuda.Stream() for _ in range(4)]

    def ce(st, d, s_, b):
        _lib.check(L.cn_copy_async(d, s_, b, ctypes.c_void_p(st.cuda_stream)), "ce")

    def sm(st, d, s_, b, blocks):
        _lib.check(L.cn_copy_sm(d, s_, b, blocks, ctypes.c_void_p(st.cuda_stream)), "sm")

    def timeit(fn, reps=10):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fn()
        torch.cuda.synchronize()
        e0.record(ss[0])
        for st in ss[1:]:
            st.wait_event(e0)
        for _ in range(reps):
            fn()
        for st in ss[1:]:
            ev = torch.cuda.Event()
            ev.record(st)
            ss[0].wait_event(ev)
        e1.record(ss[0])
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    S, D = src.data_ptr(), dst.data_ptr()
    t = timeit(lambda: ce(ss[0], D, S, n))
    print(f"CE x1: {n / t / 1e6:.1f} GB/s")
    t = timeit(lambda: (ce(ss[0], D, S, n // 2), ce(ss[1], D + n // 2, S + n // 2, n // 2)))
    print(f"CE x2 streams: {n / t / 1e6:.1f} GB/s")
    for blocks in (16, 32, 64, 148, 296):
        t = timeit(lambda: sm(ss[0], D, S, n, blocks))
        print(f"SM {blocks} blocks: {n / t / 1e6:.1f} GB/s")
    for frac in (0.25, 0.4):
        a = int(n * frac) // 16 * 16
        t = timeit(lambda: (ce(ss[0], D, S, n - a), sm(ss[1], D + n - a, S + n - a, a, 64)))
        print(f"CE + SM(64 blocks, {frac:.2f}): {n / t / 1e6:.1f} GB/s")
    # read direction (pull) by SM for reference
    t = timeit(lambda: sm(ss[0], S, D, n, 148))
    print(f"SM pull 148 blocks: {n / t / 1e6:.1f} GB/s")


if __name__ == "__main__":
    main()
