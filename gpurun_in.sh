T=r02ae; O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py -q -x -k "match or bench or verify" > $O/tests.log 2>&1; echo tests_rc=$?; tail -2 $O/tests.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-floor > $O/bench.json 2> $O/bench.err
python -c "
import json;d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],4), {k:round(v,3) for k,v in d['stages_ms'].items()}); print(d['rooflines']['match']); print(json.dumps(d['extras'].get('matcher_sweep'))[:1500])"
