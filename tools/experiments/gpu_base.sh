# baseline: the driver's exact bench command x3, then a 500-step run
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
for r in 1 2 3; do python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --no-comparator > gpurun_out/base_d20_$r.json 2> gpurun_out/base_d20_$r.err; done
python bench.py --steps 500 --no-cpu-baseline --no-comparator > gpurun_out/base_500.json 2> gpurun_out/base_500.err
for f in gpurun_out/base_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['us_per_call'],2), 'us', round(d['roofline']['frac'],3), d['e2e']['us_per_call'], d['clocks'])"; done
