# per-CTA timeline (globaltimer) of the tcgen05 kernel from an instrumented build
cp paper_2506_23225_b200/libmglu.so /tmp/libmglu_prod.so
for e in 8 11; do
  cp tools/probes/libmglu_e$e.so paper_2506_23225_b200/libmglu.so
  timeout 100 python bench.py --workload prefill --no-cpu-baseline --no-comparator --steps 1 --warmup 3 --layers 1 --clock-window 0 > gpurun_out/tctime_e$e.log 2>&1
done
cp /tmp/libmglu_prod.so paper_2506_23225_b200/libmglu.so
