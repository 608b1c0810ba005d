T=r02o; O=gpurun_out/$T; mkdir -p $O
for ov in serial early late; do EC3R_BENCH_OVERLAP=$ov timeout 900 python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline > $O/bench_$ov.json 2> $O/bench_$ov.err; echo b_rc=$?; tail -2 $O/bench_$ov.err
python -c "
import json;d=json.loads(open('$O/bench_$ov.json').read().strip().splitlines()[-1]);print('$ov', d['ms_per_step'],d['value'],d['stages_ms'],d['e2e']['ms_per_step'], d['roofline']['frac'], d['rooflines']['match']['frac'], d['rooflines']['register']['frac'])"; done
