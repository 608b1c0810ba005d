bash tools/gpu_check.sh r02ao full
O=gpurun_out/r02ao
python -c "
import json;d=json.loads(open('$O/bench.log').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['value'],d['config']['workload'][:40], {k:round(v,3) for k,v in d['stages_ms'].items()}); print(d['e2e']['ms_per_step'], d['cpu_baseline']['value'], d['cpu_baseline']['sample'][-120:])" 2>&1 | tail -3
tail -2 $O/gpu_tests.log; cat $O/kernel_traffic.json | head -40
