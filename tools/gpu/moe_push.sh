for push in ce sm:64 sm:148 sm:32; do
CN_A2A_PUSH=$push CN_A2A_DIRECT=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29671 bench.py --gpus 2 --no-sweep --no-extra --no-sched --no-cpu --no-e2e --no-ring > gpurun_out/mp.json 2>gpurun_out/mp.err
python -c "
import json,sys; d=json.load(open('gpurun_out/mp.json'))['moe_alltoall']; print(sys.argv[1], 'staged', d['ms_per_step'], d['nccl_ms_per_step'])" $push >> gpurun_out/mp.txt
CN_A2A_PUSH=$push CN_A2A_DIRECT=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29672 bench.py --gpus 2 --no-sweep --no-extra --no-sched --no-cpu --no-e2e --no-ring > gpurun_out/mp.json 2>gpurun_out/mp.err
python -c "
import json,sys; d=json.load(open('gpurun_out/mp.json'))['moe_alltoall']; print(sys.argv[1], 'direct', d['ms_per_step'], d['nccl_ms_per_step'])" $push >> gpurun_out/mp.txt
done
