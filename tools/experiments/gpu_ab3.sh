for B in 1 8 16 32 64; do
echo "== B=$B tcdec (prod: row split, head: stream-K)"; timeout 300 python tools/ab_time.py --shape 4096,14336,4,$B --libs prod head --path 4 --reps 5 2>&1 | grep -v Warn
done
echo "== B=16 ring cap 5"; MGLU_SK_WSTAGES=5 timeout 300 python tools/ab_time.py --shape 4096,14336,4,16 --libs prod --path 4 --reps 5 2>&1 | grep -v Warn
echo "== tile GEMM B=32,64"; for B in 32 64; do timeout 300 python tools/ab_time.py --shape 4096,14336,4,$B --libs prod --path 3 --reps 5 2>&1 | grep -v Warn; done
echo "== config 5 n_m=8 B=1 tcdec / mma"; timeout 300 python tools/ab_time.py --shape 8192,28672,8,1 --libs prod --path 4 --reps 3 --steps 100 2>&1 | grep -v Warn; timeout 300 python tools/ab_time.py --shape 8192,28672,8,1 --libs prod --path 2 --reps 3 --steps 100 2>&1 | grep -v Warn
timeout 900 python -m pytest tests/test_gpu_tcdec.py -x -q 2>&1 | tail -2
