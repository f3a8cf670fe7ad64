timeout 600 python -m pytest tests/test_rx_gpu.py -x -q -k "pipelined or matches_reference or split" > gpurun_out/ab2_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/ab2_tests.txt
for cfg in "CN_COPY_TMA=0" "CN_COPY_TMA=1" "CN_COPY_TMA=0" "CN_COPY_TMA=1"; do
  env $cfg python bench.py --steps 30 --warmup 5 --no-sweep --no-sched --no-extra --no-cpu --no-e2e > gpurun_out/ab2.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/ab2.json')); print(sys.argv[1], 'pipe', d['ms_per_step'], 'strict', d['strict_reset']['ms_per_step'], 'copy alone', d['kernel_ms_per_step']['copy'], 'frac', d['roofline']['frac'])" "$cfg" >> gpurun_out/ab2.txt
done
