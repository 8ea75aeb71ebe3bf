timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t_tests.log 2>&1; tail -5 gpurun_out/t_tests.log
