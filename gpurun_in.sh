T=r02fin5; O=gpurun_out/$T; mkdir -p $O
for c in 3 1; do
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:vh_insert_frames_kernel|register_edges_kernel|mt_tc_kernel" -c 6 \
  -o $O/prof_c$c python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-extras --no-floor > $O/ncu_c$c.log 2>&1; echo full_rc=$?
python tools/ncu_traffic.py $O/prof_c$c.ncu-rep > $O/kernel_traffic_c$c.json 2> $O/traffic_c$c.err
tools/ncu_metrics.sh $O/prof_c$c.ncu-rep > $O/full_metrics_c$c.txt 2>&1
ncu -i $O/prof_c$c.ncu-rep --page source --csv --print-source sass > $O/source.csv 2>/dev/null
python tools/ncu_stalls.py $O/source.csv 25 > $O/stalls_c$c.txt 2>&1
rm -f $O/source.csv
done
rm -f $O/*.ncu-rep
python -c "
import json
for c in (3,1):
  d=json.load(open('$O/kernel_traffic_c%d.json'%c))['kernels']; print(c, {k:(round(v['dram_bytes_per_launch']/1e9,3), round(v['ncu_ms_per_launch'],3)) for k,v in d.items()})"
