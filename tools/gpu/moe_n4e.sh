for e in 1 0; do
CN_A2A_EARLY=$e timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29672 bench.py --gpus 4 --no-sweep --no-extra --no-sched --no-cpu --no-e2e --no-ring > gpurun_out/m4.json 2>gpurun_out/m4.err
python -c "
import json,sys; d=json.load(open('gpurun_out/m4.json'))['moe_alltoall']; print('n4 early', sys.argv[1], d['ms_per_step'], d['nccl_ms_per_step'])" $e >> gpurun_out/m4e.txt
done
