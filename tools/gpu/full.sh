timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/f_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/f_tests.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "rc=$?" >> gpurun_out/f_bench.err
