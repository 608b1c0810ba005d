#!/usr/bin/env bash
# One GPU verification pass (run under gpurun from the repo root):
#   tools/gpu_check.sh TAG [full]
# gpu tests, a bench line, the ncu launch list of a short bench and, with
# "full", one `ncu --set full` capture of the fusion / registration / matcher
# kernels.  Everything lands in gpurun_out/TAG/.
set -u
TAG=${1:?tag}
MODE=${2:-}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > "$OUT/smi.txt" 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q --timeout 600 > "$OUT/gpu_tests.log" 2>&1
echo "tests_rc=$?"
timeout 600 python bench.py ${BENCH_ARGS:-} > "$OUT/bench.log" 2>&1
echo "bench_rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k "regex:ec3r::|CUB_200802" -c 600 --csv \
    --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-extras --no-floor \
    > "$OUT/ncu_bench.log" 2>&1
echo "ncu_rc=$?"
if [ "$MODE" = "full" ]; then
    timeout 900 ncu --set full --clock-control none --import-source on \
        -k "regex:vh_insert_frames_kernel|register_edges_kernel|mt_tc_kernel" -c 6 \
        -o "$OUT/prof" python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-extras --no-floor \
        > "$OUT/ncu_full.log" 2>&1
    echo "full_rc=$?"
fi
if [ "$MODE" = "full" ] && [ -f "$OUT/prof.ncu-rep" ]; then
    python tools/ncu_traffic.py "$OUT/prof.ncu-rep" > "$OUT/kernel_traffic.json" 2> "$OUT/traffic.err"
    tools/ncu_metrics.sh "$OUT/prof.ncu-rep" > "$OUT/full_metrics.txt" 2>&1
    ncu -i "$OUT/prof.ncu-rep" --page source --csv --print-source sass > "$OUT/source.csv" 2>/dev/null
    python tools/ncu_stalls.py "$OUT/source.csv" 25 > "$OUT/stalls.txt" 2>&1
    rm -f "$OUT/source.csv"
    python tools/launch_summary.py "$OUT/launches.csv" > "$OUT/launch_summary.txt" 2>&1
fi
