for k in 1 2; do
for lib in "" lib_u4m4.so lib_u8m4.so; do
  if [ -n "$lib" ]; then export CHUNKNET_B200_LIB=$PWD/tools/gpu/$lib; else unset CHUNKNET_B200_LIB; fi
  python bench.py --steps 30 --warmup 5 --no-sweep --no-sched --no-extra --no-cpu --no-e2e > gpurun_out/ua.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/ua.json')); print(sys.argv[1] or 'base', 'pipe', d['ms_per_step'], 'strict', d['strict_reset']['ms_per_step'], 'copy alone', d['kernel_ms_per_step']['copy'])" "$lib" >> gpurun_out/ua.txt
done; done
