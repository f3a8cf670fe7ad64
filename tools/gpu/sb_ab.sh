for k in 1 2; do for cfg in "CN_SCAN_BLOCKS=296" "CN_SCAN_BLOCKS=16" "CN_SCAN_BLOCKS=4" "CN_SCAN_BLOCKS=16 CN_ACK_BPS=2"; do
  env $cfg python bench.py --steps 30 --warmup 5 --no-sched --no-extra --no-cpu --no-e2e --no-sweep > gpurun_out/sb.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/sb.json')); print(sys.argv[1], 'pipe', d['ms_per_step'], 'strict', d['strict_reset']['ms_per_step'], d['kernel_ms_per_step']['ingest'])" "$cfg" >> gpurun_out/sb.txt
done; done
