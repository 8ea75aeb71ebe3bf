# stream-K tcgen05 decode kernel: parity tests, then the small-batch sweep vs the HMMA kernel
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tcdec.py -x -q > gpurun_out/tcdec_tests.log 2>&1; tail -15 gpurun_out/tcdec_tests.log
for B in 1 4 8 16 32 64; do
  for path in tcdec mma; do
    if [ $path = mma ] && [ $B -gt 8 ]; then continue; fi
    timeout 100 python bench.py --shape 4096,14336,4,$B --path $path --no-cpu-baseline --no-comparator --steps 300 --warmup 10 --clock-window 0.1 > gpurun_out/sm.json 2> gpurun_out/sm.err
    python -c "import json; d=json.loads(open('gpurun_out/sm.json').read().strip().splitlines()[-1]); print('B=$B', '$path', round(d['us_per_call'],2), 'us', round(d['value'],1), d['unit'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/sm.err
  done
done
for nm in 1 2 8; do
  timeout 100 python bench.py --shape 4096,14336,$nm,1 --path tcdec --no-cpu-baseline --no-comparator --steps 300 --warmup 10 --clock-window 0.1 > gpurun_out/sm.json 2> gpurun_out/sm.err
  python -c "import json; d=json.loads(open('gpurun_out/sm.json').read().strip().splitlines()[-1]); print('nm=$nm B=1 tcdec', round(d['us_per_call'],2), 'us', round(d['value'],1), d['unit'], round(d['roofline']['frac'],3))" || tail -3 gpurun_out/sm.err
done
