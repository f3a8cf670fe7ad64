timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/F_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/F_tests.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/F_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/F_bench.json 2> gpurun_out/F_bench.err; echo "rc=$?" >> gpurun_out/F_bench.err
timeout 300 python bench.py --impl reference > gpurun_out/F_ref.json 2> gpurun_out/F_ref.err
python bench.py --steps 3 --warmup 3 --no-sweep --no-extra --no-sched --no-cpu --no-e2e > gpurun_out/F_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/F_launches.csv python bench.py --steps 3 --warmup 3 --no-sweep --no-extra --no-sched --no-cpu --no-e2e > gpurun_out/F_ncu.log 2>&1
