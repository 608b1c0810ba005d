T=r02am; O=gpurun_out/$T; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo b_rc=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref_rc=$?
python -c "
import json;d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],4), d['value'], {k:round(v,3) for k,v in d['stages_ms'].items()}); print(d['e2e']); print(d['roofline']); print(d['clocks'], d['gpu_launches'])
r=json.loads(open('$O/bench_ref.json').read().strip().splitlines()[-1]); print({k:r[k] for k in ('impl','value','unit','ms_per_step')}, r.get('cpu_baseline',{}).get('sample','')[:200])"
