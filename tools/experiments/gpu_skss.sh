# stream-K tcgen05 GEMV: production (t's MMA TS) vs MGLU_SK_SS_T=1 (t's MMA SS from shared memory)
cp paper_2506_23225_b200/libmglu.so /tmp/libmglu_prod.so
for e in prod ${SKEXP:-skss}; do
  if [ $e = prod ]; then cp /tmp/libmglu_prod.so paper_2506_23225_b200/libmglu.so; else cp tools/probes/libmglu_$e.so paper_2506_23225_b200/libmglu.so; fi
  [ $e = prod ] && { timeout 600 python -m pytest tests/test_gpu_tcdec.py -x -q 2>&1 | tail -1; }
  for shp in 4096,14336,4,8 4096,14336,4,16 4096,14336,4,24 4096,14336,1,8 4096,14336,2,8 8192,28672,8,1 8192,28672,8,8 8192,28672,4,8; do
    timeout 100 python bench.py --shape $shp --path tcdec --no-cpu-baseline --no-comparator --steps 300 --warmup 10 --clock-window 0.05 > gpurun_out/tcx.json 2> gpurun_out/tcx.err
    python -c "import json; d=json.loads(open('gpurun_out/tcx.json').read().strip().splitlines()[-1]); print('$e $shp', round(d['us_per_call'],2), 'us frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/tcx.err
  done
done
cp /tmp/libmglu_prod.so paper_2506_23225_b200/libmglu.so
