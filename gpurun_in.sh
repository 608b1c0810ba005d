T=r02y; O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py tests/test_gpu_chain.py tests/test_gpu_dist.py -q -x -k "regist or chain or bench or single_pass or window or loop" > $O/tests.log 2>&1; echo tests_rc=$?; tail -3 $O/tests.log
timeout 600 python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline --no-e2e > $O/bench.json 2> $O/bench.err
python -c "
import json;d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]);print('c1', d['ms_per_step'], d['rooflines']['register'])"
for c in 3 4; do
timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-extras --no-cpu-baseline --no-e2e > $O/bench_c$c.json 2> $O/bench_c$c.err
python -c "
import json;d=json.loads(open('$O/bench_c$c.json').read().strip().splitlines()[-1]);print('c$c', d['ms_per_step'], d['rooflines']['register'])"
done
