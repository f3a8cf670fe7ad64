timeout 600 python -m pytest tests/test_alltoall_gpu.py -x -q > gpurun_out/m2_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/m2_tests.txt
for pm in 64 128; do for dm in 1 0; do for rep in 1 2; do
CN_A2A_PIECE_MB=$pm CN_A2A_DIRECT=$dm timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29641 bench.py --gpus 2 --no-sweep --no-extra --no-sched --no-cpu --no-e2e --no-ring > gpurun_out/ms.json 2>/dev/null
python -c "
import json,sys; d=json.load(open('gpurun_out/ms.json'))['moe_alltoall']; print(sys.argv[1], sys.argv[2], d['ms_per_step'], d['nccl_ms_per_step'], d['host_enqueue_ms_per_step'])" $pm $dm >> gpurun_out/ms2.txt
done; done; done
