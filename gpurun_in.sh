T=r02ah; O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py tests/test_gpu_fusion_engines.py tests/test_gpu_dist.py -q -x -k "tma or fused or fusion" > $O/tests.log 2>&1; echo tests_rc=$?; tail -2 $O/tests.log
for v in default; do
if [ $v = notma ]; then export EC3R_FI_NOTMA=1; else unset EC3R_FI_NOTMA; fi
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-extras > $O/bench_$v.json 2> $O/bench_$v.err
python -c "
import json;d=json.loads(open('$O/bench_$v.json').read().strip().splitlines()[-1]);r=d['rooflines']['fuse_insert'];print('$v', round(d['ms_per_step'],4), round(r['ms'],4), r['reduction_floor']['replay_ms'], round(r['reduction_floor']['frac'],3))"
done
