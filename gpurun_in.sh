#!/usr/bin/env bash
# r02g22: certification kernels with staged pair offsets: matcher tests, bench, launch list
O=gpurun_out/r02g22; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 -k "match or track or loop or verify or dropin or empty or bench_parity" > $O/tests.log 2>&1; echo tests_rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 --no-extras > $O/bench.log 2>&1; echo bench_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k "regex:mt_need_cols|mx_finalize|mt_tc" -c 12 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-extras --no-floor > $O/ncu.log 2>&1; echo ncu_rc=$?
