# the driver's 20-step command under variations of the enqueue-ahead spin and the NVML sampler
run() { python bench.py --steps 20 --warmup 5 --no-comparator --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['us_per_call'],2), round(d['roofline']['frac'],3), d['clocks']['samples'])"; }
for i in 1 2 3; do run default; MGLU_BENCH_NO_SAMPLER=1 run nosampler; MGLU_BENCH_AHEAD_US=200 run ahead200; done
python bench.py --steps 100 --warmup 5 --no-comparator --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('steps100', round(d['us_per_call'],2))"
