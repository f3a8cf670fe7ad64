for pm in 0 89 60; do
if [ "$pm" = 0 ]; then unset CN_A2A_PIECE_MB; else export CN_A2A_PIECE_MB=$pm; fi
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29672 bench.py --gpus 4 --no-sweep --no-extra --no-sched --no-cpu --no-e2e --no-ring > gpurun_out/m4.json 2>gpurun_out/m4.err
python -c "
import json,sys; d=json.load(open('gpurun_out/m4.json'))['moe_alltoall']; print('n4', d['piece_bytes']>>20, d['ms_per_step'], d['nccl_ms_per_step'])" >> gpurun_out/m4b.txt
done
