# small-batch regime: tcgen05 (TS) vs the HMMA decode kernel, config-3 shape
for B in 1 4 8 16 32 64; do
  for path in tcgen05 mma; do
    if [ $path = mma ] && [ $B -gt 8 ]; then continue; fi
    timeout 100 python bench.py --shape 4096,14336,4,$B --path $path --no-cpu-baseline --steps 200 --warmup 10 --clock-window 0.1 $( [ $B -ne 64 ] && echo --no-comparator ) > gpurun_out/sm.json 2> gpurun_out/sm.err
    python -c "import json; d=json.loads(open('gpurun_out/sm.json').read().strip().splitlines()[-1]); c=d.get('cublas_swiglu',{}); print('B=$B', '$path', round(d['us_per_call'],2), 'us', round(d['value'],1), d['unit'], 'cublas_us', round(c.get('us_per_call',0),1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/sm.err
  done
done
