# stream-K decode kernel: experimental builds (tools/probes/libmglu_eN.so) swapped in, timed
cp paper_2506_23225_b200/libmglu.so /tmp/libmglu_prod.so
for e in 0 $SKEXP; do
  if [ $e = 0 ]; then cp /tmp/libmglu_prod.so paper_2506_23225_b200/libmglu.so; else cp tools/probes/libmglu_$e.so paper_2506_23225_b200/libmglu.so; fi
  for sh in 4096,14336,4,1 4096,14336,1,1 4096,14336,4,16 4096,14336,4,64; do
    timeout 100 python bench.py --shape $sh --path tcdec --no-cpu-baseline --no-comparator --steps 200 --warmup 10 --clock-window 0.05 > gpurun_out/skexp.json 2> gpurun_out/skexp.err
    python -c "import json; d=json.loads(open('gpurun_out/skexp.json').read().strip().splitlines()[-1]); print('exp $e $sh', round(d['us_per_call'],2), 'us', round(d['value'],1), d['unit'])" || tail -2 gpurun_out/skexp.err
  done
done
cp /tmp/libmglu_prod.so paper_2506_23225_b200/libmglu.so
