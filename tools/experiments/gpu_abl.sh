echo "== row split (tcrow) config 3: prod | abl2 no masked-copy STTM | abl3 t-MMA only"
for B in 1 16 32; do echo "-- B=$B"; timeout 300 python tools/ab_time.py --shape 4096,14336,4,$B --libs prod abl2 abl3 --path 5 --reps 5 --steps 200 2>&1 | grep -v Warn | cut -c1-80; done
echo "-- stream-K n_m=8 config 5 B=1"; timeout 300 python tools/ab_time.py --shape 8192,28672,8,1 --libs prod abl2 abl3 --path 4 --reps 3 --steps 100 2>&1 | grep -v Warn | cut -c1-80
