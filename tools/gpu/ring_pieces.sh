for pm in 32 64 128 256; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 2 --no-sweep --no-extra --no-sched --no-cpu --no-e2e --no-moe --piece-mb $pm > gpurun_out/rp.json 2>/dev/null
python -c "
import json,sys; d=json.load(open('gpurun_out/rp.json'))['allreduce']; print(sys.argv[1], 'fp32', d['fp32']['busbw_GBps'], d['fp32']['pieces_per_step'], 'bf16', d['bf16']['busbw_GBps'], 'nccl', d['fp32']['nccl_busbw_GBps'], d['fp32']['parity']['sample_bit_exact_vs_fold'])" $pm >> gpurun_out/rp.txt
done
