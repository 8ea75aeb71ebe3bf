python tools/ab_time.py --shape 4096,14336,4,1 --libs H0 H1 --reps 7 2>&1 | tail -2
python tools/ab_time.py --shape 4096,11008,4,1 --libs H0 H1 --reps 5 2>&1 | tail -2
python tools/ab_time.py --shape 8192,28672,4,1 --libs H0 H1 --reps 5 --layers 2 2>&1 | tail -2
python tools/ab_time.py --shape 4096,14336,4,1 --libs H0 H1 --reps 5 --steps 20 2>&1 | tail -2
