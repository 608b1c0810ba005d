T=r02ar; O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py tests/test_gpu_chain.py -q -x -k "regist or chain or single_pass or bench_registration" > $O/tests.log 2>&1; echo tests_rc=$?; tail -2 $O/tests.log
for c in 1 3; do
timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-extras --no-floor > $O/bench_c$c.json 2> $O/bench_c$c.err
python -c "
import json;d=json.loads(open('$O/bench_c$c.json').read().strip().splitlines()[-1]);print('c$c', round(d['ms_per_step'],4), {k:round(v,3) for k,v in d['stages_ms'].items()}, round(d['rooflines']['register']['ms'],4), round(d['rooflines']['register']['frac'],4), d['stage_rooflines']['align_fuse'])"
done
