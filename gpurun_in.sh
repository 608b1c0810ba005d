#!/usr/bin/env bash
# r02g26: final set at HEAD: full GPU suite, bench, launch list, ncu full captures (configs[3]), smoke, configs[1], reference arm
O=gpurun_out/r02g26; mkdir -p $O
BENCH_ARGS="--steps 20 --warmup 5" bash tools/gpu_check.sh r02g26 full
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?
timeout 600 python bench.py --config 1 --steps 20 --warmup 5 --no-extras > $O/bench_c1.log 2>&1; echo c1_rc=$?
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.log 2>&1; echo ref_rc=$?
