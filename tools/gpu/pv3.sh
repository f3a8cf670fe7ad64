for k in 1 2; do
python bench.py --steps 30 --warmup 5 --no-sweep --no-sched --no-extra --no-cpu --no-e2e > gpurun_out/pv3.json 2>gpurun_out/pv3.err
python -c "
import json,sys; d=json.load(open('gpurun_out/pv3.json')); print('pipe', d['ms_per_step'], 'strict', d['strict_reset']['ms_per_step'], 'copy alone', d['kernel_ms_per_step']['copy'], d['roofline']['step_frac'], d['clocks'])" >> gpurun_out/pv3.txt
done
