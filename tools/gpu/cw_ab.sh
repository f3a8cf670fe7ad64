for cfg in "CN_COPY_WARPS=8" "CN_COPY_WARPS=4" "CN_COPY_WARPS=2" "CN_COPY_WARPS=4 CN_COPY_BLOCKS_PER_SM=128" "CN_COPY_WARPS=8" "CN_COPY_WARPS=4"; do
  env $cfg python bench.py --steps 30 --warmup 5 --no-sweep --no-sched --no-extra --no-cpu --no-e2e > gpurun_out/cw.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/cw.json')); print(sys.argv[1], 'pipe', d['ms_per_step'], 'strict', d['strict_reset']['ms_per_step'], 'copy', d['kernel_ms_per_step']['copy'])" "$cfg" >> gpurun_out/cw.txt
done
