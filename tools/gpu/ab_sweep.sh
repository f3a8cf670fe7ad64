for k in 1 2; do for lib in "" lib_881.so; do
  if [ -n "$lib" ]; then export CHUNKNET_B200_LIB=$PWD/tools/gpu/$lib; else unset CHUNKNET_B200_LIB; fi
  python bench.py --steps 10 --warmup 3 --no-sched --no-extra --no-cpu --no-e2e > gpurun_out/abs.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/abs.json')); s=d['sweep_cfg5']; print(sys.argv[1] or 'new', 'pipe', d['ms_per_step'], [ (r['msg_bytes']>>10, r['msgs_per_conn'], r['ms_per_batch']) for r in s])" "$lib" >> gpurun_out/abs.txt
done; done
