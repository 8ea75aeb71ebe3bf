# per-B comparison of the three bf16 paths at the config-3 shape (d=4096, h=14336, n_m=4)
for B in ${BS:-1 2 3 4 6 8 12 16}; do
  for path in mma tcdec tcgen05; do
    if [ $path = mma ] && [ $B -gt 8 ]; then continue; fi
    timeout 100 python bench.py --shape ${DH:-4096,14336,4},$B --path $path --no-cpu-baseline --no-comparator --steps 300 --warmup 10 --clock-window 0.05 > gpurun_out/pp.json 2> gpurun_out/pp.err
    python -c "import json; d=json.loads(open('gpurun_out/pp.json').read().strip().splitlines()[-1]); print('B=$B', '$path', round(d['us_per_call'],2), 'us', round(d['value'],1), d['unit'])" || tail -2 gpurun_out/pp.err
  done
done
