T=r02ab; O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_bench_parity.py -q -x > $O/tests.log 2>&1; echo tests_rc=$?; tail -2 $O/tests.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-extras --no-cpu-baseline --no-e2e > $O/bench.json 2> $O/bench.err
python -c "
import json;d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],4), {k:round(v,3) for k,v in d['stages_ms'].items()}, d['config']['voxels_per_gpu'], d['roofline']['reduction_floor']['frac'])"
