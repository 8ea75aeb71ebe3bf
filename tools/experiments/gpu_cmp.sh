cp paper_2506_23225_b200/libmglu.so /tmp/prod.so
for e in prod split; do
  if [ $e = prod ]; then cp /tmp/prod.so paper_2506_23225_b200/libmglu.so; else cp tools/probes/libmglu_$e.so paper_2506_23225_b200/libmglu.so; fi
  for w in decode_b1 decode_b8; do timeout 200 python bench.py --workload $w --no-cpu-baseline --no-comparator --layers 2 > gpurun_out/v.json 2>&1; python -c "import json; d=json.loads(open('gpurun_out/v.json').read().strip().splitlines()[-1]); print('$e $w', round(d['us_per_call'],2), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"; done
done
cp /tmp/prod.so paper_2506_23225_b200/libmglu.so
