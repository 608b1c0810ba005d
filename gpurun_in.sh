T=r02bk; O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py -q -x -k "match or bench_tracking" > $O/tests.log 2>&1; echo tests_rc=$?; tail -1 $O/tests.log
for v in default oldscan; do
if [ $v = default ]; then unset EC3R_B200_LIB; else export EC3R_B200_LIB=variants/libec3r_$v.so; fi
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:mt_unit" -c 4 --csv --log-file $O/l_$v.csv python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-extras --no-floor > /dev/null 2>&1
python - <<PY
import csv
rows=[r for r in csv.reader(open('$O/l_$v.csv')) if len(r)>10]
h=rows[0]; i=h.index('Kernel Name'); j=h.index('Metric Value')
for r in rows[1:]: print('$v', r[i][:20], r[j])
PY
for c in 3 1; do timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-extras --no-floor > $O/b_${v}_$c.json 2>/dev/null; python -c "
import json;d=json.loads(open('$O/b_${v}_$c.json').read().strip().splitlines()[-1]);print('$v c$c', round(d['ms_per_step'],4), round(d['stages_ms']['match'],3))"; done
done
