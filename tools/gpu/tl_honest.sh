CN_COPY_TMA=0 PIPE=1 python tests/rx_timeline_tool.py 4 8 > gpurun_out/h_pipe.txt 2>&1
CN_COPY_TMA=0 python tests/rx_timeline_tool.py 4 6 > gpurun_out/h_strict.txt 2>&1
CN_COPY_TMA=1 PIPE=1 python tests/rx_timeline_tool.py 4 8 > gpurun_out/h_pipe_tma.txt 2>&1
