timeout 1700 python -m pytest tests/test_gpu_sanitizer.py -v > gpurun_out/san.log 2>&1; tail -30 gpurun_out/san.log
