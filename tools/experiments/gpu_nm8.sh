echo "== config 5 n_m=8 B=1"; timeout 300 python tools/ab_time.py --shape 8192,28672,8,1 --libs prod head --path 4 --reps 3 --steps 100 2>&1 | grep -v Warn
echo "== config 5 n_m=8 B=1 stream-K"; MGLU_SK_ROWS=0 timeout 300 python tools/ab_time.py --shape 8192,28672,8,1 --libs prod --path 4 --reps 3 --steps 100 2>&1 | grep -v Warn
for B in 1 8 16 32; do echo "== config 3 n_m=8 B=$B"; timeout 300 python tools/ab_time.py --shape 4096,14336,8,$B --libs prod head --path 4 --reps 3 2>&1 | grep -v Warn; done
echo "== config 3 n_m=8 B=1 mma"; timeout 300 python tools/ab_time.py --shape 4096,14336,8,1 --libs prod --path 2 --reps 3 2>&1 | grep -v Warn
timeout 900 python -m pytest tests/test_gpu_tcdec.py -x -q 2>&1 | tail -2
