timeout 900 python -m pytest tests/test_gpu_ffn_fused.py tests/test_gpu_ffn.py -x -q 2>&1 | tail -3
( echo "== FFN block (up-projection + W_o), config 3 shape"; timeout 300 python tools/time_ffn.py --shape 4096,14336,4 --bs 1,2,4 2>&1 | grep -v Warn
  echo "== config 2 shape (LLaMA-7B)"; timeout 300 python tools/time_ffn.py --shape 4096,11008,4 --bs 1 2>&1 | grep -v Warn ) > gpurun_out/ffn_fused.txt 2>&1; cat gpurun_out/ffn_fused.txt
