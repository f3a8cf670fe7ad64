for b in 4 2 1 3; do
CN_ACK_BPS=$b python bench.py --steps 30 --warmup 5 --no-sweep --no-sched --no-extra --no-cpu --no-e2e > gpurun_out/ab3.json 2>/dev/null
python -c "
import json,sys; d=json.load(open('gpurun_out/ab3.json')); print('ack_bps', sys.argv[1], 'pipe', d['ms_per_step'], 'strict', d['strict_reset']['ms_per_step'], 'acks alone', d['kernel_ms_per_step']['acks'])" $b >> gpurun_out/ab3.txt
done
