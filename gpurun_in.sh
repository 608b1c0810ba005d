T=r02v; O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py tests/test_gpu_chain.py tests/test_gpu_dist.py tests/test_gpu_reference_suite.py -q -x -k "regist or chain or bench or single_pass or window or loop or mapping" > $O/tests.log 2>&1; echo tests_rc=$?; tail -3 $O/tests.log
timeout 900 python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline --no-e2e > $O/bench.json 2> $O/bench.err; echo b_rc=$?
python -c "
import json;d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['stages_ms']); print(d['rooflines']['register'])"
