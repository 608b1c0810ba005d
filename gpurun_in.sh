T=r02be; O=gpurun_out/$T; mkdir -p $O
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 4 --steps 3 --warmup 3 --no-extras > $O/n4_c3.json 2> $O/n4_c3.err; echo n4_rc=$?
tail -1 $O/n4_c3.json | python -c "
import json,sys;d=json.loads(sys.stdin.read());print(d['n_gpus'], round(d['ms_per_step'],2), d['value'], d['config'].get('validation_only','')[:60], d['config']['workload'][:30])"
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 8 --config 1 --steps 3 --warmup 3 --no-extras --no-e2e > $O/n8_c1.json 2> $O/n8_c1.err; echo n8_rc=$?
tail -1 $O/n8_c1.json | python -c "
import json,sys;d=json.loads(sys.stdin.read());print(d['n_gpus'], round(d['ms_per_step'],2), d['value'], d['config'].get('validation_only','')[:60])"
tail -3 $O/n8_c1.err | cut -c1-200
