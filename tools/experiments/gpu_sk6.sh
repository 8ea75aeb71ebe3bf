timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/sk6_tests.log 2>&1; tail -3 gpurun_out/sk6_tests.log
echo "== B=1 mma"; python tools/ab_time.py --shape 4096,14336,4,1 --libs prod A3 --path 2 --reps 3 2>&1 | tail -2
for r in 1 2; do python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/sk6_d20_$r.json 2>/dev/null; done
python tools/summ.py gpurun_out/sk6_d20_*.json
