export PIPE=1 NOPROF=1 SYNTH=1024x4096 SYNTH_MPC=16
python tests/rx_timeline_tool.py 4 6 > gpurun_out/nm_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_(ingest|copy|scan|acks|finalize)" -s 40 -c 5 -o gpurun_out/r02_rx_full_many python tests/rx_timeline_tool.py 4 6 > gpurun_out/nm_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/nm_ncu.log
