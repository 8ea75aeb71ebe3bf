timeout 900 python -m pytest tests/test_gpu_planes.py -x -q 2>&1 | tail -2
( echo "== routed Top-K, config 3 shape n_m = 8 (d=4096 h=14336), G precomputed"; timeout 300 python tools/time_routed.py --shape 4096,14336,8 --bs 1,2,4 --ks 1,2 2>&1 | grep -v Warn
  echo "== config 3 n_m = 4"; timeout 300 python tools/time_routed.py --shape 4096,14336,4 --bs 1,2 --ks 1,2 2>&1 | grep -v Warn ) > gpurun_out/routed_planes.txt 2>&1; cat gpurun_out/routed_planes.txt
