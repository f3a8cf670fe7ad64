for k in 1 2; do for push in sm:32 sm:64 sm:20; do for pm in 128 256; do
CN_A2A_PUSH=$push CN_A2A_PIECE_MB=$pm timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29672 bench.py --gpus 2 --no-sweep --no-extra --no-sched --no-cpu --no-e2e --no-ring > gpurun_out/me.json 2>gpurun_out/me.err
python -c "
import json,sys; d=json.load(open('gpurun_out/me.json'))['moe_alltoall']; print('push', sys.argv[1], 'pieces', sys.argv[2], d['ms_per_step'], d['nccl_ms_per_step'])" $push $pm >> gpurun_out/me2.txt
done; done; done
