T=r02h; O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x -k loop > $O/dist_tests.log 2>&1; echo tests_rc=$?; tail -30 $O/dist_tests.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --no-extras --no-cpu-baseline > $O/n2_gloo.json 2> $O/n2_gloo.err; echo n2_rc=$?; tail -c 600 $O/n2_gloo.json; tail -5 $O/n2_gloo.err
