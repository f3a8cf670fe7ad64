export STEADY=1 NOPROF=1
python tests/rx_timeline_tool.py 4 6 > gpurun_out/n1_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_(ingest|finalize)" -s 8 -c 4 -o gpurun_out/n1_steady python tests/rx_timeline_tool.py 4 6 > gpurun_out/n1_ncu.log 2>&1
