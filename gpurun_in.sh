T=r02al; O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fusion_engines.py -q -x -k "tma" > $O/tests.log 2>&1; echo tests_rc=$?; tail -2 $O/tests.log
/usr/local/cuda/bin/compute-sanitizer --tool racecheck --target-processes all --print-limit 20 --error-exitcode 17 python -m pytest tests/test_gpu_fusion_engines.py -m gpu -x -q -p no:cacheprovider -k tma_strip > $O/sanitizer_racecheck_tma.log 2>&1; echo rc=$?; tail -3 $O/sanitizer_racecheck_tma.log
for v in tma notma; do
if [ $v = tma ]; then export EC3R_FI_TMA=1; else unset EC3R_FI_TMA; fi
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-extras --no-floor > $O/bench_$v.json 2> $O/bench_$v.err
python -c "
import json;d=json.loads(open('$O/bench_$v.json').read().strip().splitlines()[-1]);r=d['rooflines']['fuse_insert'];print('$v', round(d['ms_per_step'],4), round(r['ms'],4))"
done
