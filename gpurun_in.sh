T=r02s; O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py tests/test_gpu_chain.py -q -x -k "regist or chain or bench or single_pass" > $O/tests.log 2>&1; echo tests_rc=$?; tail -3 $O/tests.log
timeout 900 python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline --no-e2e > $O/bench.json 2> $O/bench.err; echo b_rc=$?
python -c "
import json;d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['value'],d['stages_ms']); print(d.get('kernels_ms', d.get('kernel_ms')))"
EC3R_B200_LIB=variants/libec3r_e6.so timeout 300 python tools/fuse_timing.py --reps 10 > $O/e6.log 2>&1; tail -1 $O/e6.log
