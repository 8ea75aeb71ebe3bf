# full GPU suite + smoke + the driver's bench command + per-config decode lines
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/chk_tests.log 2>&1; tail -3 gpurun_out/chk_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/chk_smoke.log 2>&1; tail -1 gpurun_out/chk_smoke.log
for r in 1 2; do python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/chk_d20_$r.json 2> gpurun_out/chk_d20_$r.err; done
python bench.py > gpurun_out/chk_default.json 2> gpurun_out/chk_default.err
for w in decode7b_b1 sweep_b1_nm1 sweep_b1_nm2 sweep_b1_nm4 sweep_b1_nm8; do python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-comparator --layers 2 > gpurun_out/chk_$w.json 2> gpurun_out/chk_$w.err; done
for b in 2 4; do python bench.py --shape 4096,14336,4,$b --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/chk_b$b.json 2> gpurun_out/chk_b$b.err; done
python bench.py --shape 8192,28672,8,1 --path mma --steps 20 --warmup 5 --layers 2 --no-cpu-baseline --no-comparator > gpurun_out/chk_nm8mma.json 2> gpurun_out/chk_nm8mma.err
python tools/summ.py gpurun_out/chk_*.json
