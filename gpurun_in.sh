T=r02d; O=gpurun_out/$T; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_fusion_engines.py -q -x > $O/engine_tests.log 2>&1; echo tests_rc=$?; tail -3 $O/engine_tests.log
EC3R_DEBUG_BINS=1 timeout 600 python tools/fuse_ab.py --reps 5 > $O/fuse_ab.json 2> $O/fuse_ab.err; echo ab_rc=$?; cat $O/fuse_ab.json; grep vbin $O/fuse_ab.err | tail -2
timeout 900 ncu -k regex:"bn_|bf_|vh_|vb_|Radix|Scan" --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ab_launches.csv python tools/fuse_ab.py --reps 1 > /dev/null 2>&1; echo ncu_rc=$?
python tools/launch_summary.py $O/ab_launches.csv 2>/dev/null | head -30
timeout 900 ncu -k regex:"bn_bin_frames|bn_aggregate" -c 2 --set full --import-source on --clock-control none -o $O/bin_full python tools/fuse_ab.py --reps 1 > $O/ncu_full.log 2>&1; echo ncu_full_rc=$?; tail -3 $O/ncu_full.log
