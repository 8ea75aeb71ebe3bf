# baseline check: GPU suite + driver-style default bench (20 steps) + batch sweep of the bf16 paths
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/base_tests.log 2>&1; tail -2 gpurun_out/base_tests.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/base_bench.json 2> gpurun_out/base_bench.err; tail -c 600 gpurun_out/base_bench.json
