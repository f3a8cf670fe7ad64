for N in 4 2 4 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29672 bench.py --gpus $N --no-sweep --no-extra --no-sched --no-cpu --no-e2e --no-ring > gpurun_out/m4.json 2>gpurun_out/m4.err
python -c "
import json,sys; d=json.load(open('gpurun_out/m4.json'))['moe_alltoall']; print('N', sys.argv[1], d['piece_bytes']>>20, d['ms_per_step'], d['nccl_ms_per_step'])" $N >> gpurun_out/m24.txt
done
