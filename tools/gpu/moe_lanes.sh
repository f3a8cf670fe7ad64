for cfg in "CN_A2A_LANES=1" "CN_A2A_LANES=2" "CN_A2A_LANES=1 CN_A2A_PUSH=sm:64" "CN_A2A_LANES=1 CN_A2A_PIECE_MB=32" "CN_A2A_LANES=1 CN_A2A_PIECE_MB=48"; do
env $cfg timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29672 bench.py --gpus 2 --no-sweep --no-extra --no-sched --no-cpu --no-e2e --no-ring > gpurun_out/ml.json 2>gpurun_out/ml.err
python -c "
import json,sys; d=json.load(open('gpurun_out/ml.json'))['moe_alltoall']; print(sys.argv[1], d['ms_per_step'], d['nccl_ms_per_step'], d['parity'])" "$cfg" >> gpurun_out/ml.txt
done
