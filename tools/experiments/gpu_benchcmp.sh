export MGLU_LIB=$PWD/tools/experiments/lib/libmglu_A3.so
python tools/ab_time.py --libs A3 --reps 3 > gpurun_out/bc_ab.txt 2>&1
for r in 1 2; do
MGLU_BENCH_AHEAD_US=25 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-comparator --e2e-streams 0 > gpurun_out/bc_old_$r.json 2>/dev/null
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-comparator --e2e-streams 0 > gpurun_out/bc_new_$r.json 2>/dev/null
MGLU_BENCH_NO_SAMPLER=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-comparator --e2e-streams 0 > gpurun_out/bc_nosamp_$r.json 2>/dev/null
python bench.py --steps 500 --warmup 5 --no-cpu-baseline --no-comparator --e2e-streams 0 > gpurun_out/bc_new500_$r.json 2>/dev/null
done
python tools/ab_time.py --libs A3 --reps 3 >> gpurun_out/bc_ab.txt 2>&1
