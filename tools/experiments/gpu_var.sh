# compare experiment builds of the decode kernel (tools/experiments/lib/libmglu_<V>.so, MGLU_DEC_ONLY)
set -x
for V in "$@"; do
  export MGLU_LIB=$PWD/tools/experiments/lib/libmglu_$V.so
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "test_bf16_shapes and mma and (n_m1 or -4-) or one_hot_forward_bit_exact and mma and (1-mma or 4-mma)" > gpurun_out/var_${V}_tests.log 2>&1; tail -1 gpurun_out/var_${V}_tests.log
  timeout 300 python -m pytest tests/test_gpu_fullsize.py -q -x -k "test_full_size_sampled_columns" > gpurun_out/var_${V}_full.log 2>&1; tail -1 gpurun_out/var_${V}_full.log
  for r in 1 2; do python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --no-comparator --e2e-streams 0 > gpurun_out/var_${V}_d20_$r.json 2> gpurun_out/var_${V}_d20_$r.err; done
  python bench.py --steps 500 --no-cpu-baseline --no-comparator --e2e-streams 0 > gpurun_out/var_${V}_500.json 2> gpurun_out/var_${V}_500.err
  python bench.py --workload sweep_b1_nm4 --steps 200 --layers 2 --no-cpu-baseline --no-comparator --e2e-streams 0 > gpurun_out/var_${V}_c5.json 2> gpurun_out/var_${V}_c5.err
done
python tools/summ.py gpurun_out/var_*.json
