for k in 1 2; do for cfg in "base" "aw4" "aw4_bps8"; do
  unset CHUNKNET_B200_LIB CN_ACK_BPS
  case $cfg in aw4) export CHUNKNET_B200_LIB=$PWD/tools/gpu/lib_aw4.so;; aw4_bps8) export CHUNKNET_B200_LIB=$PWD/tools/gpu/lib_aw4.so CN_ACK_BPS=8;; esac
  python bench.py --steps 30 --warmup 5 --no-sched --no-extra --no-cpu --no-e2e > gpurun_out/aw.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/aw.json')); s=d['sweep_cfg5']; print(sys.argv[1], 'pipe', d['ms_per_step'], 'strict', d['strict_reset']['ms_per_step'], 'acks', d['kernel_ms_per_step']['acks'], '4K', s[0]['ms_per_batch'], '64K', s[1]['ms_per_batch'])" "$cfg" >> gpurun_out/aw.txt
done; done
