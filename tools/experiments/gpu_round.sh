# round artifacts: full GPU tests, smoke, default bench, reference arm, launch list, ncu full of decode + prefill kernels
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw,temperature.gpu --format=csv > gpurun_out/nvsmi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 300 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; cat gpurun_out/bench_default.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; cat gpurun_out/bench_reference.json
for w in prefill decode_b8 decode7b_b1; do timeout 300 python bench.py --workload $w --no-cpu-baseline --layers 2 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_decode_b1.csv python bench.py --steps 20 --warmup 3 --no-comparator --no-cpu-baseline --clock-window 0 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_prefill.csv python bench.py --workload prefill --layers 1 --steps 5 --warmup 3 --no-comparator --no-cpu-baseline --clock-window 0 > /dev/null 2>&1
bash tools/gpu_profx.sh decode_b1 gemv_mma --workload decode_b1
bash tools/gpu_profx.sh prefill gemm_tc --workload prefill --layers 1
bash tools/gpu_profx.sh decode_b8 gemv_tc --workload decode_b8
echo round done
