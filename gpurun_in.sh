T=r02i; O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_pnp.py tests/test_gpu_reference_suite.py tests/test_gpu_dist.py -q -x -k "loop" > $O/tests.log 2>&1; echo tests_rc=$?; tail -30 $O/tests.log
