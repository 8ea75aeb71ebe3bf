mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tcdec.py tests/test_gpu_bounds.py -x -q > gpurun_out/rows_tests.log 2>&1; tail -3 gpurun_out/rows_tests.log
echo "== config 3"; timeout 300 python tools/sweep_paths.py --shape 4096,14336,4 --bs 1,4,8,16,24,32,48,64 --paths tcdec 2>&1 | grep -v Warn
echo "== config 5 n_m=8"; timeout 300 python tools/sweep_paths.py --shape 8192,28672,8 --bs 1,8 --paths tcdec --steps 100 2>&1 | grep -v Warn
echo "== config 5 n_m=4"; timeout 300 python tools/sweep_paths.py --shape 8192,28672,4 --bs 1,16 --paths tcdec --steps 100 2>&1 | grep -v Warn
