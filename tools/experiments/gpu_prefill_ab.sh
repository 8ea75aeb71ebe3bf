# prefill tile-GEMM variants, interleaved in one process (config 4: d=8192 h=28672 n_m=4 B=4096)
echo "== config 4 prefill, tcgen05 (prod: BN=64 KA=32 TS-t 2 slots | v1: BN=80 KA=16 SS-t 3 slots | v2: BN=64 KA=16 SS-t 4 slots | v3: BN=80 KA=16 TS-t 2 slots)"
timeout 600 python tools/ab_time.py --shape 8192,28672,4,4096 --libs prod v1 v2 v3 --path 3 --reps 3 --steps 10 --layers 2 2>&1 | grep -v Warn
echo "== config 3 B=64"
timeout 300 python tools/ab_time.py --shape 4096,14336,4,64 --libs prod v1 v2 v3 --path 3 --reps 5 --steps 100 2>&1 | grep -v Warn
