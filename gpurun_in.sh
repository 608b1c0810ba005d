T=r02bc; O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "regist or single_pass or odd_frame" > $O/tests.log 2>&1; echo tests_rc=$?; tail -1 $O/tests.log
for v in default oldreg default oldreg; do
if [ $v = default ]; then unset EC3R_B200_LIB; else export EC3R_B200_LIB=variants/libec3r_$v.so; fi
for c in 1 3; do
timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-extras --no-floor > $O/bench_${v}_$c.json 2> $O/bench_${v}_$c.err
python -c "
import json;d=json.loads(open('$O/bench_${v}_$c.json').read().strip().splitlines()[-1]);print('$v c$c', round(d['ms_per_step'],4), round(d['rooflines']['register']['ms'],4), round(d['rooflines']['register']['frac'],4))"
done; done
