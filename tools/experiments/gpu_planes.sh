timeout 900 python -m pytest tests/test_gpu_planes.py tests/test_gpu_topk.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
( echo "== routed Top-K, config 3 shape n_m = 8 (d=4096 h=14336)"; timeout 300 python tools/time_routed.py --shape 4096,14336,8 --bs 1,2,4 --ks 1,2 2>&1 | grep -v Warn
  echo "== config 3 n_m = 4"; timeout 300 python tools/time_routed.py --shape 4096,14336,4 --bs 1 --ks 1,2 2>&1 | grep -v Warn ) > gpurun_out/routed_planes.txt 2>&1; cat gpurun_out/routed_planes.txt
echo "== BN=8 experiment (stream-K / row split at B <= 8)"
for s in "8192,28672,8,1" "4096,14336,4,8" "4096,14336,4,5"; do timeout 300 python tools/ab_time.py --shape $s --libs prod bn8 --path 4 --reps 3 --steps 100 2>&1 | grep -v Warn; done
