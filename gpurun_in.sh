T=r02bi; O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py tests/test_gpu_dist.py -q -x -k "voxel or fused or bench or map or window" > $O/tests.log 2>&1; echo tests_rc=$?; tail -2 $O/tests.log
for v in default emit64 default emit64; do
if [ $v = default ]; then unset EC3R_B200_LIB; else export EC3R_B200_LIB=variants/libec3r_$v.so; fi
for c in 3 1; do
timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-extras > $O/b_${v}_$c.json 2> $O/b_${v}_$c.err
python -c "
import json;d=json.loads(open('$O/b_${v}_$c.json').read().strip().splitlines()[-1]);print('$v c$c', round(d['ms_per_step'],4), {k:round(v,3) for k,v in d['stages_ms'].items()})"
done; done
