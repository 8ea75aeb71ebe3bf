# stream-K GEMV timing ablation: production vs no fix-up (MGLU_SK_NOFIXUP=1, wrong results)
cp paper_2506_23225_b200/libmglu.so /tmp/libmglu_prod.so
for e in prod ${SKEXP:-nofix}; do
  if [ $e = prod ]; then cp /tmp/libmglu_prod.so paper_2506_23225_b200/libmglu.so; else cp tools/probes/libmglu_$e.so paper_2506_23225_b200/libmglu.so; fi
  for shp in 4096,14336,4,1 4096,14336,4,8 4096,14336,4,16 4096,14336,4,24 8192,28672,8,8; do
    timeout 100 python bench.py --shape $shp --path tcdec --no-cpu-baseline --no-comparator --steps 300 --warmup 10 --clock-window 0.05 > gpurun_out/tcx.json 2> gpurun_out/tcx.err
    python -c "import json; d=json.loads(open('gpurun_out/tcx.json').read().strip().splitlines()[-1]); print('$e $shp', round(d['us_per_call'],2), 'us')" || tail -3 gpurun_out/tcx.err
  done
done
cp /tmp/libmglu_prod.so paper_2506_23225_b200/libmglu.so
