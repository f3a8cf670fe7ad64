for b in 2 4 8 16 64; do
  echo "== CN_COPY_BLOCKS_PER_SM=$b" >> gpurun_out/bps.txt
  CN_COPY_BLOCKS_PER_SM=$b PIPE=1 python tests/rx_timeline_tool.py 4 6 > gpurun_out/bps_$b.txt 2>&1
  python - "$b" >> gpurun_out/bps.txt <<'PY'
import sys, re
rows=[l.split() for l in open(f"gpurun_out/bps_{sys.argv[1]}.txt") if l.strip() and l.split()[0].replace('.','').isdigit()]
cp=[r for r in rows if 'k_copy' in r[3]]
print("copy us:", [r[2] for r in cp], "span per step:", round((float(cp[-1][1])-float(cp[0][0]))/len(cp),1))
PY
done
