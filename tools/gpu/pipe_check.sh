timeout 900 python -m pytest tests/test_rx_gpu.py tests/test_rx_edges_gpu.py tests/test_sweep_gpu.py tests/test_reduce_gpu.py tests/test_endpoint_gpu.py -x -q > gpurun_out/pc_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/pc_tests.txt
timeout 600 python bench.py --no-sweep --no-sched --no-extra --no-cpu > gpurun_out/pc_bench.json 2> gpurun_out/pc_bench.err
echo "rc=$?" >> gpurun_out/pc_bench.err
