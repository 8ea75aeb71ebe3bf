set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
python bench.py --workload decode_b8 --no-cpu-baseline > gpurun_out/bench_b8.json 2>&1
python bench.py --workload decode7b_b1 --no-cpu-baseline > gpurun_out/bench_7b.json 2>&1
for nm in 1 2 4 8; do python bench.py --workload sweep_b1_nm$nm --no-cpu-baseline --no-comparator --layers 2 > gpurun_out/bench_sweep_nm$nm.json 2>&1; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_decode_b1.csv python bench.py --steps 20 --warmup 3 --no-comparator --no-cpu-baseline --clock-window 0 > gpurun_out/ncu_launch_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemv_mma -s 5 -c 1 -o gpurun_out/prof_gemv_mma_decode_b1 python bench.py --steps 10 --warmup 3 --no-comparator --no-cpu-baseline --clock-window 0 > gpurun_out/ncu_full_run.log 2>&1
echo done
