for sh in 4096,14336,4 4096,18944,4 4096,9472,4 4096,14208,4 8192,28672,4 4096,14336,1 4096,14336,8; do
  python bench.py --shape $sh,1 --no-cpu-baseline --no-comparator --steps 300 --clock-window 0.05 > /tmp/o.json 2>/tmp/o.err
  python -c "import json; d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); print('$sh', round(d['us_per_call'],2), 'us', round(d['value']), 'GB/s', round(d['roofline']['frac'],3))" || tail -2 /tmp/o.err
done
