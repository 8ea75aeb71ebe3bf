# full GPU suite + AUTO / per-path sweep at config 3 (profiles/r02/tcrow_sweep.txt)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tcrow_tests.log 2>&1; tail -3 gpurun_out/tcrow_tests.log
( echo "== config 3 (d=4096 h=14336 n_m=4), us/call, 200 calls x 3 reps, 4 layer copies > L2"
  timeout 600 python tools/sweep_paths.py --shape 4096,14336,4 --bs 1,2,4,5,8,9,12,16,24,32,48,64 --paths auto,mma,tcdec,tcrow,tcgen05 2>&1 | grep -v "Warn\|refused"
  echo "== config 5 (d=8192 h=28672) B=1, AUTO"; for nm in 1 2 4 8; do timeout 300 python tools/sweep_paths.py --shape 8192,28672,$nm --bs 1 --paths auto --steps 100 2>&1 | grep -v Warn; done
) > gpurun_out/tcrow_sweep.txt 2>&1; cat gpurun_out/tcrow_sweep.txt
