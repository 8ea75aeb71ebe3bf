for B in 32 64; do echo "== B=$B"; python tools/ab_time.py --shape 4096,14336,4,$B --libs prod --path 3 --reps 3 2>&1 | tail -1; done
python bench.py --shape 4096,14336,4,64 --path tcgen05 --steps 200 --no-cpu-baseline --no-comparator --e2e-streams 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['us_per_call'], d['clocks'])"
nvidia-smi -q -d PERFORMANCE,CLOCK | head -60
