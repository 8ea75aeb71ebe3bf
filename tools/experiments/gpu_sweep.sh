# round tables: config 3 per batch (AUTO path, vs same-box cuBLAS SwiGLU) and the config-5 n_m sweep
echo "== config 3 (d=4096, h=14336, n_m=4) by batch, AUTO dispatch"
for B in 1 2 4 8 16 32 64; do
  timeout 200 python bench.py --shape 4096,14336,4,$B --no-cpu-baseline --steps 300 --clock-window 0.05 > gpurun_out/sw.json 2> gpurun_out/sw.err
  python -c "import json; d=json.loads(open('gpurun_out/sw.json').read().strip().splitlines()[-1]); c=d['cublas_swiglu']; print('B=%d path=%s mglu_us=%.2f %s=%.1f frac=%.3f cublas_swiglu_us=%.2f speedup=%.2f e2e_us=%.2f' % ($B, d['config']['kernel_path'], d['us_per_call'], d['unit'], d['value'], d['roofline']['frac'], c['us_per_call'], c['mglu_speedup'], d['e2e']['us_per_call']))" || tail -2 gpurun_out/sw.err
done
echo "== config 5 (d=8192, h=28672) n_m sweep, AUTO dispatch"
for nm in 1 2 4 8; do for B in 1 2048; do
  timeout 300 python bench.py --shape 8192,28672,$nm,$B --no-cpu-baseline --steps $([ $B = 1 ] && echo 300 || echo 10) --layers 2 --clock-window 0.05 > gpurun_out/sw.json 2> gpurun_out/sw.err
  python -c "import json; d=json.loads(open('gpurun_out/sw.json').read().strip().splitlines()[-1]); c=d['cublas_swiglu']; print('n_m=%d B=%d path=%s mglu_us=%.2f %s=%.1f frac=%.3f cublas_swiglu_us=%.2f' % ($nm, $B, d['config']['kernel_path'], d['us_per_call'], d['unit'], d['value'], d['roofline']['frac'], c['us_per_call']))" || tail -2 gpurun_out/sw.err
done; done
