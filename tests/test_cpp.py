"""The C++ host facade (include/chunknet_b200.hpp) compiles against the C ABI
and runs: wire codec + exception mapping on CPU, a golden trace replay on
the GPU."""
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, load_golden

CUDA_INC = "/usr/local/cuda/include"
LIBDIR = os.path.join(ROOT, "paper_2504_17307_b200")


def _cudart_dir():
    import nvidia.cuda_runtime as m  # the image's CUDA runtime wheel
    return os.path.join(os.path.dirname(m.__file__), "lib")


def _build(src, out):
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), "-I", CUDA_INC,
           os.path.join(ROOT, "tests", "cpp", src), "-o", out, "-L", LIBDIR, "-lchunknet_b200",
           "-L", _cudart_dir(), "-l:libcudart.so.12",
           f"-Wl,-rpath,{LIBDIR}", f"-Wl,-rpath,{_cudart_dir()}"]
    subprocess.run(cmd, check=True)


def test_cpp_wire_facade(tmp_path):
    exe = str(tmp_path / "wire_test")
    _build("wire_test.cpp", exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stderr
    assert "CPP_WIRE_OK" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cfg1", "concurrent_k4"])
def test_cpp_rx_facade_replays_golden(tmp_path, name):
    from oracle import oracle as O
    exe = str(tmp_path / "rx_golden")
    _build("rx_golden.cpp", exe)
    data, acks, _, meta = load_golden(name)
    data.tofile(tmp_path / "data.bin")
    O.fill_staging(data).tofile(tmp_path / "staging.bin")
    acks.tofile(tmp_path / "acks.bin")
    r = subprocess.run([exe, str(tmp_path / "data.bin"), str(tmp_path / "staging.bin"),
                        str(tmp_path / "acks.bin"), str(meta["chunk_bytes"])],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "CPP_RX_OK" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cfg1", "lossy_2m"])
def test_cpp_endpoint_replays_sender(tmp_path, name):
    import json
    from paper_2504_17307_b200.sender import LB
    exe = str(tmp_path / "endpoint_replay")
    _build("endpoint_replay.cpp", exe)
    z = np.load(os.path.join(ROOT, "tests", "golden", f"sender_{name}.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    z["submits"].tofile(tmp_path / "subs.bin")
    z["acks"].tofile(tmp_path / "acks.bin")
    z["tx"].tofile(tmp_path / "tx.bin")
    args = [exe, str(tmp_path / "subs.bin"), str(tmp_path / "acks.bin"), str(tmp_path / "tx.bin"),
            str(meta["chunk_bytes"]), str(meta["n_paths"]), str(LB[meta["lb"]]), str(meta["rto_min"]),
            str(meta["rto_max"]), str(meta["commit_ahead"]), str(meta["base_rtt"]), str(meta["seed"]),
            str(meta["src"]), str(meta["dst"])]
    r = subprocess.run(args, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "CPP_ENDPOINT_OK" in r.stdout
