for k in 1 2; do for N in 2 4; do for pu in sm:32 sm:64; do
CN_A2A_PUSH=$pu timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29672 bench.py --gpus $N --no-sweep --no-extra --no-sched --no-cpu --no-e2e --no-ring > gpurun_out/m4.json 2>gpurun_out/m4.err
python -c "
import json,sys; d=json.load(open('gpurun_out/m4.json'))['moe_alltoall']; print('N', sys.argv[2], sys.argv[1], d['ms_per_step'], d['nccl_ms_per_step'], round(d['ms_per_step']/d['nccl_ms_per_step'],3))" $pu $N >> gpurun_out/mp3.txt
done; done; done
