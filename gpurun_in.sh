T=r02aw; O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "odd_frame" > $O/tests.log 2>&1; echo tests_rc=$?; tail -15 $O/tests.log
