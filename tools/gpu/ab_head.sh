for k in 1 2; do for lib in "" lib_head.so; do
  if [ -n "$lib" ]; then export CHUNKNET_B200_LIB=$PWD/tools/gpu/$lib; else unset CHUNKNET_B200_LIB; fi
  python bench.py --steps 30 --warmup 5 --no-sched --no-extra --no-cpu --no-e2e > gpurun_out/abh.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/abh.json')); s=d['sweep_cfg5']; print(sys.argv[1] or 'new', 'pipe', d['ms_per_step'], 'strict', d['strict_reset']['ms_per_step'], 'fin', d['kernel_ms_per_step']['finalize'], '4K', s[0]['ms_per_batch'], '64K', s[1]['ms_per_batch'], '1M', s[2]['ms_per_batch'])" "$lib" >> gpurun_out/abh.txt
done; done
