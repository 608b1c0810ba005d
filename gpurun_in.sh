T=r02l; O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_decode.py -q -x > $O/tests.log 2>&1; echo tests_rc=$?; tail -30 $O/tests.log
