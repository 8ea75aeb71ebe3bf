# run the prefill bench with experimental builds of the library swapped in
cp paper_2506_23225_b200/libmglu.so /tmp/libmglu_prod.so
for e in 0 1 2; do
  if [ $e = 0 ]; then cp /tmp/libmglu_prod.so paper_2506_23225_b200/libmglu.so; else cp tools/probes/libmglu_e$e.so paper_2506_23225_b200/libmglu.so; fi
  for w in prefill sweep_b2048_nm8; do
    timeout 100 python bench.py --workload $w --no-cpu-baseline --no-comparator --steps 10 --warmup 3 --layers 2 --clock-window 0.1 > gpurun_out/tcexp.json 2> gpurun_out/tcexp.err
    python -c "import json; d=json.loads(open('gpurun_out/tcexp.json').read().strip().splitlines()[-1]); print('exp $e $w', round(d['us_per_call'],1), 'us', round(d['value'],1), d['unit'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/tcexp.err
  done
done
cp /tmp/libmglu_prod.so paper_2506_23225_b200/libmglu.so
