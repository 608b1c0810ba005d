T=r02bd; O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fusion_engines.py -q -x > $O/tests.log 2>&1; echo tests_rc=$?; tail -3 $O/tests.log
