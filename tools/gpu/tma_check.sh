timeout 900 python -m pytest tests/test_rx_gpu.py tests/test_rx_edges_gpu.py tests/test_sweep_gpu.py tests/test_props_gpu.py -x -q > gpurun_out/t1_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/t1_tests.txt
for v in 1 0; do
  CN_COPY_TMA=$v PIPE=1 python tests/rx_timeline_tool.py 4 6 > gpurun_out/t1_pipe_$v.txt 2>&1
  CN_COPY_TMA=$v python tests/rx_timeline_tool.py 4 4 > gpurun_out/t1_strict_$v.txt 2>&1
done
