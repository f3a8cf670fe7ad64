timeout 900 python -m pytest tests/test_rx_gpu.py tests/test_rx_edges_gpu.py tests/test_sweep_gpu.py tests/test_props_gpu.py tests/test_reduce_gpu.py -x -q > gpurun_out/pdl_tests.txt 2>&1; echo rc=$? >> gpurun_out/pdl_tests.txt
for v in 1 0 1 0; do
CN_PDL=$v python bench.py --steps 30 --warmup 5 --no-sched --no-extra --no-cpu --no-e2e > gpurun_out/pdl.json 2>/dev/null
python -c "
import json,sys; d=json.load(open('gpurun_out/pdl.json')); s=d['sweep_cfg5']; print('pdl', sys.argv[1], 'pipe', d['ms_per_step'], 'strict', d['strict_reset']['ms_per_step'], 'sweep 4K', s[0]['ms_per_batch'], '64K', s[1]['ms_per_batch'], '4Kx16', s[-1]['ms_per_batch'])" $v >> gpurun_out/pdl.txt
done
