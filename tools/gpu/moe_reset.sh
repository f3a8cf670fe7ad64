timeout 300 python -m pytest tests/ -q -m gpu -k "alltoall" > gpurun_out/mr_t.txt 2>&1
for k in 1 2 3; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29672 bench.py --gpus 2 --no-sweep --no-extra --no-sched --no-cpu --no-e2e --no-ring > gpurun_out/mr.json 2>gpurun_out/mr.err
python -c "
import json,sys; d=json.load(open('gpurun_out/mr.json'))['moe_alltoall']; print('sigcopy', d['piece_bytes']>>20, d['ms_per_step'], d['nccl_ms_per_step'])" >> gpurun_out/mr.txt
done
