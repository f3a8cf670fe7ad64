export STEADY=1
python tests/rx_timeline_tool.py 4 6 > gpurun_out/e1_base.txt 2>&1
CHUNKNET_B200_LIB=$PWD/tools/gpu/libexp_adv32.so python tests/rx_timeline_tool.py 4 6 > gpurun_out/e1_adv32.txt 2>&1
