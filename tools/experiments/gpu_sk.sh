# stream-K rework: tcdec tests, then B sweep of tcdec vs tile GEMM (in-process, same box)
timeout 900 python -m pytest tests/test_gpu_tcdec.py tests/test_gpu_parity.py -q -x -k "tcdec or fast_path" > gpurun_out/sk_tests.log 2>&1; tail -3 gpurun_out/sk_tests.log
for B in 1 5 8 12 16 24 32 48 64; do echo "== B=$B"; python tools/ab_time.py --shape 4096,14336,4,$B --libs prod --path 4 --reps 3 2>&1 | tail -1; python tools/ab_time.py --shape 4096,14336,4,$B --libs prod --path 3 --reps 3 2>&1 | tail -1; done > gpurun_out/sk_sweep.txt 2>&1
for B in 1 8 16 32; do echo "== n_m=8 B=$B"; python tools/ab_time.py --shape 8192,28672,8,$B --libs prod --path 4 --reps 3 --layers 2 2>&1 | tail -1; done >> gpurun_out/sk_sweep.txt 2>&1
cat gpurun_out/sk_sweep.txt
