timeout 300 python -m pytest tests/ -q -m gpu -k "alltoall" > gpurun_out/me_t.txt 2>&1
for k in 1 2; do for e in 1 0; do for pm in 64 128; do
CN_A2A_EARLY=$e CN_A2A_PIECE_MB=$pm timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29672 bench.py --gpus 2 --no-sweep --no-extra --no-sched --no-cpu --no-e2e --no-ring > gpurun_out/me.json 2>gpurun_out/me.err
python -c "
import json,sys; d=json.load(open('gpurun_out/me.json'))['moe_alltoall']; print('early', sys.argv[1], 'pieces', sys.argv[2], d['ms_per_step'], d['nccl_ms_per_step'], d.get('parity'))" $e $pm >> gpurun_out/me.txt
done; done; done
