T=r02r; O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py tests/test_gpu_dist.py -q -x -k "voxel or fused or bench or loop or window" > $O/tests.log 2>&1; echo tests_rc=$?; tail -3 $O/tests.log
timeout 900 python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo b_rc=$?
python -c "
import json;d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['value'],d['stages_ms'])"
EC3R_BENCH_OVERLAP=serial timeout 900 python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline > $O/bench_serial.json 2> $O/bench_serial.err
python -c "
import json;d=json.loads(open('$O/bench_serial.json').read().strip().splitlines()[-1]);print('serial', d['ms_per_step'],d['value'],d['stages_ms'])"
