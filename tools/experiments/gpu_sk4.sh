for B in 64; do echo "== B=$B tcgen05"; python tools/ab_time.py --shape 4096,14336,4,$B --libs prod noz R1 --path 3 --reps 3 2>&1 | tail -3; done
for B in 1 8 16 32 64; do echo "== B=$B tcdec"; python tools/ab_time.py --shape 4096,14336,4,$B --libs prod R1 --path 4 --reps 3 2>&1 | tail -2; done
