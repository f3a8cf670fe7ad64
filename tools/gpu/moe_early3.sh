timeout 300 python -m pytest tests/ -q -m gpu -k "alltoall" > gpurun_out/me_t.txt 2>&1
for k in 1 2; do for pm in 64 96 128; do
CN_A2A_PIECE_MB=$pm timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29672 bench.py --gpus 2 --no-sweep --no-extra --no-sched --no-cpu --no-e2e --no-ring > gpurun_out/me.json 2>gpurun_out/me.err
python -c "
import json,sys; d=json.load(open('gpurun_out/me.json'))['moe_alltoall']; print('hc pieces', sys.argv[1], d['ms_per_step'], d['nccl_ms_per_step'])" $pm >> gpurun_out/me3.txt
done; done
