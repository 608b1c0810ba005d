T=r02q; O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x -k loop > $O/dist.log 2>&1; echo t_rc=$?; tail -2 $O/dist.log
NCCL_DEBUG=WARN timeout 600 python tools/nccl_one_gpu.py > $O/nccl.log 2>&1; echo rc=$?; tail -2 $O/nccl.log
for n in 2 4 8; do timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n bench.py --gpus $n --steps 3 --warmup 3 --no-extras --no-cpu-baseline > $O/n${n}_nccl.json 2> $O/n${n}_nccl.err; echo n${n}_rc=$?; tail -2 $O/n${n}_nccl.err
python -c "
import json;d=json.loads(open('$O/n${n}_nccl.json').read().strip().splitlines()[-1]);print($n, d['ms_per_step'], d['value'], d['config'].get('validation_only'), d['config']['voxels_per_gpu'], d['stages_ms'])"; done
