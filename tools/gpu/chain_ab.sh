for cfg in "CN_CHAIN_BPS=2" "CN_CHAIN_BPS=1" "CN_CHAIN_BPS=1 CN_ACK_BPS=2" "CN_CHAIN_BPS=2" "CN_CHAIN_BPS=1" "CN_CHAIN_BPS=1 CN_ACK_BPS=2"; do
  env $cfg python bench.py --steps 30 --warmup 5 --no-sweep --no-sched --no-extra --no-cpu --no-e2e > gpurun_out/ca.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/ca.json')); print(sys.argv[1], 'pipe', d['ms_per_step'], 'strict', d['strict_reset']['ms_per_step'], d['kernel_ms_per_step'])" "$cfg" >> gpurun_out/ca.txt
done
