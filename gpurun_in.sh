T=r02bm; O=gpurun_out/$T; mkdir -p $O
for g in 148 144 140 136 128; do for c in 1 3; do
EC3R_MT_GRID=$g timeout 600 python bench.py --config $c --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-extras --no-floor > $O/b_${g}_$c.json 2>/dev/null; python -c "
import json;d=json.loads(open('$O/b_${g}_$c.json').read().strip().splitlines()[-1]);print('grid $g c$c', round(d['ms_per_step'],4), {k:round(v,3) for k,v in d['stages_ms'].items()})"
done; done
