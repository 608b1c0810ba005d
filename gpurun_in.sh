T=r02bb; O=gpurun_out/$T; mkdir -p $O
for c in 1 3; do for cfg in late:148 early:100 mid:148 mid:110 mid:100 mid:90 mid:80; do
ov=${cfg%%:*}; g=${cfg##*:}
export EC3R_BENCH_OVERLAP=$ov EC3R_MT_GRID=$g
timeout 600 python bench.py --config $c --steps 20 --warmup 4 --no-cpu-baseline --no-e2e --no-extras --no-floor > $O/b_${c}_${ov}_$g.json 2> $O/b_${c}_${ov}_$g.err
python -c "
import json;d=json.loads(open('$O/b_${c}_${ov}_$g.json').read().strip().splitlines()[-1]);print('c$c $ov $g', round(d['ms_per_step'],4), round(d['rooflines']['fuse_insert']['ms'],3), round(d['rooflines']['match']['ms'],3), round(d['rooflines']['register']['ms'],3))"
done; done
