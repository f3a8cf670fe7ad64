# receive-path check: GPU tests of the receive path, phase marks, timeline
timeout 900 python -m pytest tests/test_rx_gpu.py tests/test_rx_edges_gpu.py tests/test_sweep_gpu.py tests/test_props_gpu.py tests/test_reduce_gpu.py -x -q > gpurun_out/rc_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/rc_tests.txt
CHUNKNET_B200_LIB=$PWD/tools/gpu/libexp_tm.so python tools/rx_phase_tool.py 4 8 > gpurun_out/rc_ph1.txt 2>&1
CHUNKNET_B200_LIB=$PWD/tools/gpu/libexp_tm.so SYNTH=1024x4096 python tools/rx_phase_tool.py 4 6 > gpurun_out/rc_ph2.txt 2>&1
STEADY=1 python tests/rx_timeline_tool.py 4 4 > gpurun_out/rc_tl.txt 2>&1
