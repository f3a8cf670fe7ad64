for cfg in "CN_COPY_TMA=0" "CN_TMA_BPS=1" "CN_TMA_BPS=2" "CN_TMA_BPS=3"; do
  env $cfg python bench.py --steps 10 --warmup 3 --no-sweep --no-sched --no-extra --no-cpu --no-e2e > gpurun_out/ab.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/ab.json')); print(sys.argv[1], 'pipe', d['ms_per_step'], 'strict', d['strict_reset']['ms_per_step'], 'copy alone', d['kernel_ms_per_step']['copy'], 'frac', d['roofline']['frac'])" "$cfg" >> gpurun_out/ab.txt
done
