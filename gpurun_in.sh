#!/usr/bin/env bash
# r02g28: auto CTA form at 6 waves: configs[4] / [1] / [3] bench, fusion tests
O=gpurun_out/r02g28; mkdir -p $O
for c in 4 1 3; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-extras > $O/bench_c$c.log 2>&1; echo c${c}_rc=$?
done
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -k "fus or voxel or edges or smoke" > $O/tests.log 2>&1; echo tests_rc=$?
