mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_tcgen05.py tests/test_gpu_fullsize.py tests/test_gpu_shard.py tests/test_gpu_wide_nm.py tests/test_gpu_multiproc.py tests/test_gpu_variants.py tests/test_gpu_topk.py -x -q > gpurun_out/pf_tests.log 2>&1; tail -3 gpurun_out/pf_tests.log
( echo "== prefill tile GEMM, AUTO (prod = 80-token tiles) vs head (64-token tiles), interleaved"
  timeout 600 python tools/ab_time.py --shape 8192,28672,4,4096 --libs prod head --path 0 --reps 3 --steps 10 --layers 2 2>&1 | grep -v Warn
  for nm in 1 2 4 8; do echo "-- config 5 B=2048 n_m=$nm"; timeout 600 python tools/ab_time.py --shape 8192,28672,$nm,2048 --libs prod head --path 0 --reps 3 --steps 10 --layers 2 2>&1 | grep -v Warn; done
) > gpurun_out/prefill_tiles.txt 2>&1; cat gpurun_out/prefill_tiles.txt
