T=r02af; O=gpurun_out/$T; mkdir -p $O
for v in default colfirst nosplit default; do
if [ $v = default ]; then unset EC3R_B200_LIB; else export EC3R_B200_LIB=variants/libec3r_$v.so; fi
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-floor --no-extras > $O/bench_$v.json 2> $O/bench_$v.err
python -c "
import json;d=json.loads(open('$O/bench_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step'],4), round(d['rooflines']['match']['ms'],4), round(d['rooflines']['match']['frac'],4))"
done
