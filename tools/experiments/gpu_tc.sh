# prefill / large-batch tcgen05 numbers
for w in prefill sweep_b2048_nm1 sweep_b2048_nm2 sweep_b2048_nm8 decode_b64; do
  timeout 100 python bench.py --workload $w --no-cpu-baseline --steps 20 --warmup 3 --layers 2 --clock-window 0.1 > gpurun_out/tc_$w.json 2> gpurun_out/tc_$w.err
  python -c "import json; d=json.loads(open('gpurun_out/tc_$w.json').read().strip().splitlines()[-1]); c=d.get('cublas_swiglu',{}); print('$w', d['config']['kernel_path'], round(d['us_per_call'],1), 'us', round(d['value'],1), d['unit'], 'frac', round(d['roofline']['frac'],3), 'cublas_us', round(c.get('us_per_call',0),1), 'cublas_tflops', round(c.get('tflops',0),1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/tc_$w.err
done
