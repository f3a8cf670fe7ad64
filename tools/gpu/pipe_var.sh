for k in 1 2; do
CN_COPY_TMA=0 python bench.py --steps 30 --warmup 5 --no-sweep --no-sched --no-extra --no-cpu --no-e2e > gpurun_out/pv.json 2>/dev/null
python -c "
import json,sys; d=json.load(open('gpurun_out/pv.json')); print('bench30', 'pipe', d['ms_per_step'], 'strict', d['strict_reset']['ms_per_step'], 'copy alone', d['kernel_ms_per_step']['copy'], d['clocks'])" >> gpurun_out/pv.txt
CN_COPY_TMA=0 PIPE=1 python tests/rx_timeline_tool.py 4 10 > gpurun_out/pv_tl.txt 2>&1
grep step gpurun_out/pv_tl.txt | tr '\n' ' ' >> gpurun_out/pv.txt; echo >> gpurun_out/pv.txt
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv >> gpurun_out/pv.txt
