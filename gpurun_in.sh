#!/usr/bin/env bash
# r02g25: insert CTA size chosen by wave count: timing (auto / forced), fusion tests in both forms, c3 parity, bench
O=gpurun_out/r02g25; mkdir -p $O
for kf in 300 1500; do
  for v in auto 0 1 auto; do
    if [ $v = auto ]; then L=""; else L="EC3R_FI_NT128=$v"; fi
    env $L timeout 600 python tools/fuse_timing.py --keyframes $kf --reps 10 | sed "s/^{/{\"mode\": \"$v\", /" >> $O/fuse_timing.jsonl 2>> $O/fuse_timing.err
  done
done
EC3R_FI_NT128=1 timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -k "fus or voxel or edges" > $O/tests_nt128.log 2>&1; echo t128_rc=$?
timeout 1500 python -m pytest tests/test_gpu_bench_parity_c3.py tests/test_gpu_bench_parity.py -x -q --timeout 900 > $O/tests_parity.log 2>&1; echo parity_rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_c3.log 2>&1; echo c3_rc=$?
timeout 600 python bench.py --config 1 --steps 20 --warmup 5 --no-extras > $O/bench_c1.log 2>&1; echo c1_rc=$?
