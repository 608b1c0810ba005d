OUT=gpurun_out/r02z2; mkdir -p $OUT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k "regex:ec3r::|CUB_200802" -c 600 --csv \
    --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-extras --no-floor > "$OUT/ncu_bench.log" 2>&1
echo ncu_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on \
        -k "regex:vh_insert_frames_kernel|register_edges_kernel|mt_tc_kernel" -c 6 \
        -o "$OUT/prof" python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-extras --no-floor > "$OUT/ncu_full.log" 2>&1
echo full_rc=$?
python tools/ncu_traffic.py "$OUT/prof.ncu-rep" > "$OUT/kernel_traffic.json" 2> "$OUT/traffic.err"
tools/ncu_metrics.sh "$OUT/prof.ncu-rep" > "$OUT/full_metrics.txt" 2>&1
ncu -i "$OUT/prof.ncu-rep" --page source --csv --print-source sass > "$OUT/source.csv" 2>/dev/null
python tools/ncu_stalls.py "$OUT/source.csv" 25 > "$OUT/stalls.txt" 2>&1
rm -f "$OUT/source.csv"
python tools/launch_summary.py "$OUT/launches.csv" > "$OUT/launch_summary.txt" 2>&1
