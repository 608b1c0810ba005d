T=r02g; O=gpurun_out/$T; mkdir -p $O
timeout 2400 python -m pytest tests/test_gpu_reference_suite.py tests/test_gpu_fusion_engines.py tests/test_gpu_bench_parity.py tests/test_gpu_chain.py -m gpu -q --timeout 1200 -p no:cacheprovider -rA > $O/gpu_tests.log 2>&1; echo t_rc=$?
grep -E "passed|failed|PASSED|FAILED|ERROR" $O/gpu_tests.log | tail -40
