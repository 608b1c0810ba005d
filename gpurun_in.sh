T=r02fin3; O=gpurun_out/$T; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k "regex:ec3r::|CUB_200802" -c 600 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-extras --no-floor > $O/ncu_bench.log 2>&1; echo ncu_rc=$?
python tools/launch_summary.py $O/launches.csv > $O/launch_summary.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k "regex:ec3r::|CUB_200802" -c 600 --csv --log-file $O/launches_c1.csv python bench.py --config 1 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-extras --no-floor > $O/ncu_bench_c1.log 2>&1; echo ncu1_rc=$?
python tools/launch_summary.py $O/launches_c1.csv > $O/launch_summary_c1.txt 2>&1
head -14 $O/launch_summary.txt; head -8 $O/launch_summary_c1.txt
