# tcgen05 kernels: parity of both tcgen05 test files, then prefill / mid-batch timings for the
# production build and experimental builds in $TCEXP (tools/probes/libmglu_<e>.so)
[ -z "$NOTEST" ] && timeout 900 python -m pytest tests/test_gpu_tcgen05.py tests/test_gpu_tcdec.py -x -q > gpurun_out/tc_tests.log 2>&1; tail -2 gpurun_out/tc_tests.log
cp paper_2506_23225_b200/libmglu.so /tmp/libmglu_prod.so
for e in prod $TCEXP; do
  if [ $e = prod ]; then cp /tmp/libmglu_prod.so paper_2506_23225_b200/libmglu.so; else cp tools/probes/libmglu_$e.so paper_2506_23225_b200/libmglu.so; fi
  for w in ${WLS:-prefill sweep_b2048_nm8 sweep_b2048_nm2 decode_b64}; do
    timeout 120 python bench.py --workload $w --no-cpu-baseline --no-comparator --steps 20 --warmup 3 --layers 2 --clock-window 0.1 > gpurun_out/tcx.json 2> gpurun_out/tcx.err
    python -c "import json; d=json.loads(open('gpurun_out/tcx.json').read().strip().splitlines()[-1]); print('$e $w', d['config']['kernel_path'], round(d['us_per_call'],1), 'us', round(d['value'],1), d['unit'], 'frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/tcx.err
  done
  for B in 8 16; do
    timeout 100 python bench.py --shape 4096,14336,4,$B --path tcdec --no-cpu-baseline --no-comparator --steps 300 --warmup 10 --clock-window 0.05 > gpurun_out/tcx.json 2> gpurun_out/tcx.err
    python -c "import json; d=json.loads(open('gpurun_out/tcx.json').read().strip().splitlines()[-1]); print('$e tcdec B=$B', round(d['us_per_call'],2), 'us')" || tail -3 gpurun_out/tcx.err
  done
done
cp /tmp/libmglu_prod.so paper_2506_23225_b200/libmglu.so
