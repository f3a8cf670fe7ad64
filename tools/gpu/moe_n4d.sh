for cfg in "sm:64 2" "ce 2" "sm:64 1"; do
set -- $cfg
CN_A2A_PUSH=$1 CN_A2A_LANES=$2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29672 bench.py --gpus 4 --no-sweep --no-extra --no-sched --no-cpu --no-e2e --no-ring > gpurun_out/m4.json 2>gpurun_out/m4.err
python -c "
import json,sys; d=json.load(open('gpurun_out/m4.json'))['moe_alltoall']; print('n4', sys.argv[1], sys.argv[2], d['ms_per_step'], d['nccl_ms_per_step'])" $1 $2 >> gpurun_out/m4d.txt
done
