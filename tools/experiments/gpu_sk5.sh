timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/sk5_tests.log 2>&1; tail -3 gpurun_out/sk5_tests.log
echo "== B=1 mma"; python tools/ab_time.py --shape 4096,14336,4,1 --libs prod A3 --path 2 --reps 3 2>&1 | tail -2
for B in 5 8 12 16 24 32 48 64; do echo "== B=$B tcdec / tcgen05"; python tools/ab_time.py --shape 4096,14336,4,$B --libs prod --path 4 --reps 3 2>&1 | tail -1; python tools/ab_time.py --shape 4096,14336,4,$B --libs prod --path 3 --reps 3 2>&1 | tail -1; done
