for k in 1 2; do
CN_COPY_TMA=0 python bench.py --steps 30 --warmup 5 --no-sweep --no-sched --no-extra --no-cpu --no-e2e > gpurun_out/pv.json 2>/dev/null
python -c "
import json,sys; d=json.load(open('gpurun_out/pv.json')); print('bench30', 'pipe', d['ms_per_step'], 'strict', d['strict_reset']['ms_per_step'], 'copy alone', d['kernel_ms_per_step']['copy'], d['clocks'])" >> gpurun_out/pv2.txt
done
