mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tcdec.py -x -q > gpurun_out/tcdec_tests.log 2>&1; tail -5 gpurun_out/tcdec_tests.log
for sh in 4096,14336,4,1 4096,14336,1,1 4096,14336,2,1 4096,14336,8,1 4096,14336,4,8 4096,14336,4,16 4096,14336,4,32 4096,14336,4,64 8192,28672,4,1; do
  timeout 100 python bench.py --shape $sh --path tcdec --no-cpu-baseline --no-comparator --steps 300 --warmup 10 --clock-window 0.05 > gpurun_out/sm.json 2> gpurun_out/sm.err
  python -c "import json; d=json.loads(open('gpurun_out/sm.json').read().strip().splitlines()[-1]); print('$sh tcdec', round(d['us_per_call'],2), 'us', round(d['value'],1), d['unit'], round(d['roofline']['frac'],3))" || tail -3 gpurun_out/sm.err
done
cp paper_2506_23225_b200/libmglu.so /tmp/libmglu_prod.so; cp tools/probes/libmglu_t2.so paper_2506_23225_b200/libmglu.so
timeout 100 python bench.py --shape 4096,14336,4,1 --path tcdec --no-cpu-baseline --no-comparator --steps 30 --warmup 5 --clock-window 0 --layers 4 > gpurun_out/trace_t2.log 2>&1
cp /tmp/libmglu_prod.so paper_2506_23225_b200/libmglu.so
