for B in 1 16 64; do
echo "== B=$B tcdec (prod: row split, head: stream-K)"; timeout 300 python tools/ab_time.py --shape 4096,14336,4,$B --libs prod head --path 4 --reps 5 2>&1 | grep -v Warn
done
echo "== B=1 stream-K in both"; MGLU_SK_ROWS=0 timeout 300 python tools/ab_time.py --shape 4096,14336,4,1 --libs prod head --path 4 --reps 5 2>&1 | grep -v Warn
