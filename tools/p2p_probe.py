"""Profiling helper (not a test): copy-engine push bandwidth between two
ranks over CUDA-IPC-mapped NVLink memory (the transport's wire), by piece
size, lanes (streams) and direction.
    torchrun --nproc-per-node 2 tools/p2p_probe.py"""
import ctypes
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2504_17307_b200 import _lib
    from paper_2504_17307_b200.collective import DeviceBuffer, _ipc_handle, _ipc_open
    L = _lib.lib()
    r = dist.get_rank()
    N = 512 << 20
    src = DeviceBuffer(N, torch.device("cuda", local))
    dst = DeviceBuffer(N, torch.device("cuda", local))
    tsrc = torch.empty(N, dtype=torch.uint8, device="cuda")  # a caching-allocator source
    hs = [None, None]
    dist.all_gather_object(hs, _ipc_handle(dst))
    peer = _ipc_open(hs[1 - r])
    lanes = [torch.cuda.Stream() for _ in range(4)]

    pusher = int(os.environ.get("PUSHER", "1"))

    def run(piece, nl, both, torch_src=False, total=N):
        sp = (tsrc.data_ptr() if torch_src else src.data_ptr())
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        e0.record(cur)
        if r == pusher or both:
            for ln in lanes[:nl]:
                ln.wait_stream(cur)
            for k, o in enumerate(range(0, total, piece)):
                ln = lanes[k % nl]
                _lib.check(L.cn_copy_async(peer + o, sp + o, min(piece, total - o), ctypes.c_void_p(ln.cuda_stream)),
                           "copy")
            for ln in lanes[:nl]:
                cur.wait_stream(ln)
        e1.record(cur)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        t = torch.tensor([ms if (r == pusher or both) else 0.0], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return total / (float(t.item()) * 1e-3) / 1e9

    for both in (False,):
        for piece in (64 << 20, 512 << 20):
            for nl in (1, 2):
                g = [run(piece, nl, both) for _ in range(3)][-1]
                if r == 0:
                    print(f"{'bidir' if both else 'uni  '} piece {piece >> 20:4d} MiB lanes {nl}: {g:7.1f} GB/s per direction")
    g = run(64 << 20, 2, False, torch_src=True)
    if r == 0:
        print(f"uni   torch-allocator source, 64 MiB x2: {g:.1f} GB/s")
    # the all-to-all's protocol without the receive path: rank 1 pushes
    # pieces on alternating lanes, each followed by a flag release into rank
    # 0's flag word; rank 0 waits for every piece's flag on its stream
    fl = DeviceBuffer(4096, torch.device("cuda", local))
    fl.tensor(torch.int64, 512).zero_()
    fh = [None, None]
    dist.all_gather_object(fh, _ipc_handle(fl))
    pfl = _ipc_open(fh[1 - r])
    err = fl.data_ptr() + 2048
    base = [0]

    def proto(piece, total=450 << 20, spin=True):
        torch.cuda.synchronize()
        dist.barrier()
        cur = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        k = 0
        for o in range(0, total, piece):
            k += 1
            if r == 1:
                ln = lanes[k % 2]
                ln.wait_stream(cur) if k <= 2 else None
                _lib.check(L.cn_copy_async(peer + o, src.data_ptr() + o, min(piece, total - o),
                                           ctypes.c_void_p(ln.cuda_stream)), "copy")
                _lib.check(L.cn_flag_signal(pfl + 8 * (k % 2), None, base[0] + (k + 1) // 2,
                                            ctypes.c_void_p(ln.cuda_stream)), "sig")
            elif spin:
                _lib.check(L.cn_flag_wait(fl.data_ptr() + 8 * (k % 2), None, base[0] + (k + 1) // 2, 1 << 40, err,
                                          ctypes.c_void_p(cur.cuda_stream)), "wait")
        if r == 1:
            for ln in lanes[:2]:
                cur.wait_stream(ln)
        e1.record(cur)
        torch.cuda.synchronize()
        base[0] += (k + 1) // 2
        t = torch.tensor([e0.elapsed_time(e1)], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return total / (float(t.item()) * 1e-3) / 1e9
    for piece in ():
        for spin in (False, True):
            g = [proto(piece, spin=spin) for _ in range(3)][-1]
            if r == 0:
                print(f"protocol: 450 MiB in {piece >> 20} MiB pieces, 2 lanes + flag per piece, receiver "
                      f"{'spins per piece' if spin else 'idle'}: {g:.1f} GB/s")
    _lib.lib().cn_ipc_close(ctypes.c_void_p(pfl))
    dist.barrier()
    _lib.lib().cn_ipc_close(ctypes.c_void_p(peer))
    src.free()
    dst.free()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
