for k in 1 2; do for sb in default 100000; do
  if [ "$sb" = default ]; then unset CN_ACK_SMALL; else export CN_ACK_SMALL=$sb; fi
  python bench.py --no-cpu --no-e2e --no-sched --no-ring --no-moe --no-extra > gpurun_out/as.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/as.json')); s=d['sweep_cfg5']; print('small', sys.argv[1], 'pipe', d['ms_per_step'], 'strict', d['strict_reset']['ms_per_step'], [(x['msg_bytes']>>10, x['msgs_per_conn'], x['ms_per_batch']) for x in s])" $sb >> gpurun_out/as.txt
done; done
