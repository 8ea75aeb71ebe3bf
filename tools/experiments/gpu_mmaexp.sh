# HMMA decode kernel experiments: row-balance bound (h = 148 * 96) and consumer-warp count variants
cp paper_2506_23225_b200/libmglu.so /tmp/libmglu_prod.so
for e in prod $MEXP; do
  if [ $e = prod ]; then cp /tmp/libmglu_prod.so paper_2506_23225_b200/libmglu.so; else cp tools/probes/libmglu_$e.so paper_2506_23225_b200/libmglu.so; fi
  for sh in ${SHAPES:-4096,14336,4,1 4096,14208,4,1 4096,14336,1,1 4096,14336,4,8}; do
    timeout 100 python bench.py --shape $sh --path mma --no-cpu-baseline --no-comparator --steps 500 --warmup 10 --clock-window 0.05 > gpurun_out/mx.json 2> gpurun_out/mx.err
    python -c "import json; d=json.loads(open('gpurun_out/mx.json').read().strip().splitlines()[-1]); print('$e $sh', round(d['us_per_call'],2), 'us', round(d['value'],1), d['unit'], round(d['roofline']['frac'],3))" || tail -3 gpurun_out/mx.err
  done
done
cp /tmp/libmglu_prod.so paper_2506_23225_b200/libmglu.so
