T=r02e; O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "voxel or fuse" > $O/tests.log 2>&1; echo t_rc=$?; tail -3 $O/tests.log
for v in default m3 m3r64; do
  if [ $v = default ]; then unset EC3R_B200_LIB; else export EC3R_B200_LIB=variants/libec3r_$v.so; fi
  timeout 600 python tools/fuse_ab.py --reps 5 > $O/fuse_ab_$v.json 2> $O/fuse_ab_$v.err; echo $v rc=$?; cat $O/fuse_ab_$v.json; tail -2 $O/fuse_ab_$v.err
done
unset EC3R_B200_LIB
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k "regex:ec3r::" -c 200 --csv --log-file $O/launches.csv python tools/fuse_ab.py --reps 1 > /dev/null 2>&1; echo l_rc=$?
python tools/launch_summary.py $O/launches.csv > $O/launch_summary.txt 2>&1; head -40 $O/launch_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:bf_bin_kernel|bf_aggregate_kernel" -c 2 -o $O/prof python tools/fuse_ab.py --reps 1 > $O/ncu_full.log 2>&1; echo f_rc=$?
tools/ncu_metrics.sh $O/prof.ncu-rep > $O/full_metrics.txt 2>&1; cat $O/full_metrics.txt
