for k in 1 2; do for p in 0 1; do
  CN_PDL=$p python bench.py --no-cpu --no-e2e --no-sched --no-ring --no-moe --no-extra > gpurun_out/pdls.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/pdls.json')); s=d['sweep_cfg5']; print('pdl', sys.argv[1], 'pipe', d['ms_per_step'], [(x['msg_bytes']>>10, x['msgs_per_conn'], x['ms_per_batch']) for x in s])" $p >> gpurun_out/pdls.txt
done; done
