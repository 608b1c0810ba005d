#!/usr/bin/env bash
# r02g30: final check of the shipped binary: full GPU suite, smoke, driver-style bench
O=gpurun_out/r02g30; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -x -q --timeout 600 > $O/gpu_tests.log 2>&1; echo tests_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.log 2>&1; echo bench_rc=$?
