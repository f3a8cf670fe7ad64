for pm in 16 32 64 128; do
CN_A2A_PIECE_MB=$pm CN_A2A_PUSH=sm:32 CN_A2A_DIRECT=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29672 bench.py --gpus 2 --no-sweep --no-extra --no-sched --no-cpu --no-e2e --no-ring > gpurun_out/mp.json 2>gpurun_out/mp.err
python -c "
import json,sys; d=json.load(open('gpurun_out/mp.json'))['moe_alltoall']; print('pieces', sys.argv[1], 'direct sm:32', d['ms_per_step'], d['nccl_ms_per_step'])" $pm >> gpurun_out/mp2.txt
done
