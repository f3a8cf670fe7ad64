export PIPE=1 NOPROF=1
python tests/rx_timeline_tool.py 4 6 > gpurun_out/np_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread --clock-control none -k regex:"k_(ingest|copy|scan|trim|acks|finalize)" -s 30 -c 12 --csv --log-file gpurun_out/np_metrics.csv python tests/rx_timeline_tool.py 4 6 > gpurun_out/np_ncu.log 2>&1
