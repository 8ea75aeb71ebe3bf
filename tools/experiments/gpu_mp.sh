timeout 1500 python -m pytest tests/test_gpu_multiproc.py -v -x > gpurun_out/mp.log 2>&1; tail -15 gpurun_out/mp.log
