for k in 1 2; do for lib in "" lib_m5.so lib_m6.so; do
  if [ -n "$lib" ]; then export CHUNKNET_B200_LIB=$PWD/tools/gpu/$lib; else unset CHUNKNET_B200_LIB; fi
  python bench.py --steps 30 --warmup 5 --no-sweep --no-sched --no-extra --no-cpu --no-e2e > gpurun_out/mb.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/mb.json')); print(sys.argv[1] or 'base', 'pipe', d['ms_per_step'], 'strict', d['strict_reset']['ms_per_step'], 'copy alone', d['kernel_ms_per_step']['copy'])" "$lib" >> gpurun_out/mb.txt
done; done
