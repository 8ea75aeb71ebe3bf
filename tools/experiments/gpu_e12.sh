echo "== tcgen05 GEMV: prod | e1 LG=1 (one A-stage in registers) | e2 KA=16 (n_m <= 4)"
for B in 1 8 16 32 48; do echo "-- row split B=$B"; timeout 300 python tools/ab_time.py --shape 4096,14336,4,$B --libs prod e1 e2 --path 5 --reps 5 --steps 200 2>&1 | grep -v Warn | cut -c1-80; done
echo "-- stream-K B=8"; timeout 300 python tools/ab_time.py --shape 4096,14336,4,8 --libs prod e1 e2 --path 4 --reps 5 --steps 200 2>&1 | grep -v Warn | cut -c1-80
