T=r02fin4; O=gpurun_out/$T; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo tests_rc=$?; tail -1 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo c3_rc=$?
timeout 900 python bench.py --config 1 > $O/bench_c1.json 2> $O/bench_c1.err; echo c1_rc=$?
for c in c3 c1; do python -c "
import json;d=json.loads(open('$O/bench_$c.json').read().strip().splitlines()[-1]);print('$c', round(d['ms_per_step'],4), d['value'], {k:(round(v['ms'],4), round(v['frac'],4)) for k,v in d['rooflines'].items()}, round(d['roofline'].get('reduction_floor',{}).get('frac',0),3), round(d['e2e']['ms_per_step'],2), d['cpu_baseline']['value'], d['stage_rooflines']['align_fuse']['frac'])"; done
for cl in 4 8; do EC3R_RE_CL=$cl timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-extras --no-floor > $O/re_$cl.json 2>/dev/null; python -c "
import json;d=json.loads(open('$O/re_$cl.json').read().strip().splitlines()[-1]);print('c3 cl$cl', round(d['rooflines']['register']['ms'],4))"; done
