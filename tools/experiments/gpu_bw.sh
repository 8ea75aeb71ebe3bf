timeout 1200 python -m pytest tests/test_gpu_backward.py -q -x > gpurun_out/bw_tests.log 2>&1; tail -15 gpurun_out/bw_tests.log
