cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_rx_gpu.py tests/test_props_gpu.py tests/test_sweep_gpu.py tests/test_reduce_gpu.py tests/test_rx_edges_gpu.py -q -x 2>&1 | tail -3
python bench.py --steps 10 --warmup 3 --no-extra --no-sched --no-e2e --no-cpu 2>>gpurun_out/ab_err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['kernel_ms'], [(x['msg_bytes'],x['msgs_per_conn'],x['GBps']) for x in d['sweep_cfg5']])"
SYNTH=1024x4096 python tests/rx_timeline_tool.py 1 2 2>&1 | tail -8
