T=r02ax; O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "match" > $O/tests.log 2>&1; echo tests_rc=$?; tail -1 $O/tests.log
for v in default row1 default row1; do
if [ $v = default ]; then unset EC3R_B200_LIB; else export EC3R_B200_LIB=variants/libec3r_$v.so; fi
timeout 600 python bench.py --config 1 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-extras --no-floor > $O/bench_$v.json 2> $O/bench_$v.err
python -c "
import json;d=json.loads(open('$O/bench_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step'],4), round(d['rooflines']['match']['ms'],4), round(d['rooflines']['match']['frac'],4))"
done
