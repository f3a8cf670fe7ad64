timeout 900 python -m pytest tests/test_rx_gpu.py tests/test_rx_edges_gpu.py tests/test_sweep_gpu.py tests/test_props_gpu.py tests/test_endpoint_gpu.py -x -q > gpurun_out/r2_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/r2_tests.txt
CHUNKNET_B200_LIB=$PWD/tools/gpu/libexp_tm.so TILES=1 python tools/rx_phase_tool.py 4 6 > gpurun_out/r2_ph.txt 2>&1
PIPE=1 python tests/rx_timeline_tool.py 4 6 > gpurun_out/r2_tl.txt 2>&1
