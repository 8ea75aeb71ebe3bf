mkdir -p gpurun_out
[ -z "$NOTEST" ] && timeout 600 python -m pytest tests/test_gpu_tcdec.py -x -q > gpurun_out/tcdec_tests.log 2>&1; tail -3 gpurun_out/tcdec_tests.log
cp paper_2506_23225_b200/libmglu.so /tmp/libmglu_prod.so
for e in prod $SKEXP; do
  if [ $e = prod ]; then cp /tmp/libmglu_prod.so paper_2506_23225_b200/libmglu.so; else cp tools/probes/libmglu_$e.so paper_2506_23225_b200/libmglu.so; fi
  for sh in ${SHAPES:-4096,14336,4,1 4096,14336,1,1 4096,14336,8,1 4096,14336,4,16 4096,14336,4,64}; do
    timeout 100 python bench.py --shape $sh --path tcdec --no-cpu-baseline --no-comparator --steps 300 --warmup 10 --clock-window 0.05 > gpurun_out/sm.json 2> gpurun_out/sm.err
    python -c "import json; d=json.loads(open('gpurun_out/sm.json').read().strip().splitlines()[-1]); print('$e $sh', round(d['us_per_call'],2), 'us', round(d['value'],1), d['unit'], round(d['roofline']['frac'],3))" || tail -3 gpurun_out/sm.err
  done
done
cp tools/probes/libmglu_${TRACE:-t3}.so paper_2506_23225_b200/libmglu.so
timeout 100 python bench.py --shape 4096,14336,4,1 --path tcdec --no-cpu-baseline --no-comparator --steps 30 --warmup 5 --clock-window 0 --layers 4 > gpurun_out/trace_${TRACE:-t3}.log 2>&1
cp /tmp/libmglu_prod.so paper_2506_23225_b200/libmglu.so
