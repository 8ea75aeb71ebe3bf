timeout 1500 python -m pytest tests/test_gpu_tcgen05.py tests/test_gpu_tcdec.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_topk.py tests/test_gpu_wide_nm.py tests/test_gpu_hooks.py -q -x 2>&1 | tail -2
( echo "== prefill epilogue: prod (ex2/rcp swish) vs pre (expf + IEEE division), interleaved"
  python tools/ab_time.py --shape 8192,28672,4,4096 --libs prod pre --path 0 --reps 5 --steps 10 --layers 2 2>&1 | grep -v Warn | cut -c1-150
  python tools/ab_time.py --shape 8192,28672,8,2048 --libs prod pre --path 0 --reps 5 --steps 10 --layers 2 2>&1 | grep -v Warn | cut -c1-150
  python tools/ab_time.py --shape 8192,28672,2,2048 --libs prod pre --path 0 --reps 5 --steps 10 --layers 2 2>&1 | grep -v Warn | cut -c1-150
  python tools/ab_time.py --shape 8192,28672,1,2048 --libs prod pre --path 0 --reps 5 --steps 10 --layers 2 2>&1 | grep -v Warn | cut -c1-150
  for B in 16 32 48 64; do echo "-- config 3 B=$B (AUTO)"; python tools/ab_time.py --shape 4096,14336,4,$B --libs prod pre --path 0 --reps 5 --steps 200 2>&1 | grep -v Warn | cut -c1-100; done ) > gpurun_out/prefill_epilogue.txt 2>&1; cat gpurun_out/prefill_epilogue.txt
