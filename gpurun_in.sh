T=r02g; O=gpurun_out/$T; mkdir -p $O
timeout 900 ncu -k regex:"vc_|vb_|Radix|Scan|bbox" --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/emit_launches.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > /dev/null 2>&1; echo ncu_rc=$?
python tools/launch_summary.py $O/emit_launches.csv | head -20
EC3R_EMIT_VOXEL_SORT=1 timeout 900 python bench.py --steps 20 --warmup 5 --no-extras --no-cpu-baseline > $O/bench_old.json 2> $O/bench_old.err; python -c "
import json;d=json.loads(open('$O/bench_old.json').read().strip().splitlines()[-1]);print('old',d['ms_per_step'],d['stages_ms'])"
timeout 900 python bench.py --steps 20 --warmup 5 --no-extras --no-cpu-baseline > $O/bench_new.json 2> $O/bench_new.err; python -c "
import json;d=json.loads(open('$O/bench_new.json').read().strip().splitlines()[-1]);print('new',d['ms_per_step'],d['stages_ms'])"
