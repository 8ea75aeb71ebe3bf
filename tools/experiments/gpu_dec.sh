# decode kernel iteration: parity of the MMA path, then the driver's bench command and 500-step runs
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_ffn.py tests/test_gpu_topk.py tests/test_gpu_variants.py tests/test_gpu_shard.py -x -q > gpurun_out/it_tests.log 2>&1; tail -3 gpurun_out/it_tests.log
for r in 1 2; do python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --no-comparator --e2e-streams 1 > gpurun_out/it_d20_$r.json 2> gpurun_out/it_d20_$r.err; done
MGLU_DEC_L2PF=2 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --no-comparator --e2e-streams 1 > gpurun_out/it_d20_pf2.json 2> gpurun_out/it_d20_pf2.err
python bench.py --steps 500 --no-cpu-baseline --no-comparator --e2e-streams 1 > gpurun_out/it500.json 2> gpurun_out/it500.err
for w in decode7b_b1 sweep_b1_nm4 sweep_b1_nm1 sweep_b1_nm8; do python bench.py --workload $w --steps 200 --no-cpu-baseline --no-comparator --e2e-streams 1 --layers 2 > gpurun_out/it_$w.json 2> gpurun_out/it_$w.err; done
for b in 2 4; do python bench.py --shape 4096,14336,4,$b --steps 300 --no-cpu-baseline --no-comparator --e2e-streams 1 > gpurun_out/it_b$b.json 2> gpurun_out/it_b$b.err; done
python tools/summ.py gpurun_out/it_*.json gpurun_out/it500*.json
