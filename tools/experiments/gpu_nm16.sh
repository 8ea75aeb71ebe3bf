timeout 900 python -m pytest tests/test_gpu_wide_nm.py tests/test_gpu_tcgen05.py -x -q 2>&1 | tail -3
echo "== config 5 shape, n_m = 16 (tile GEMM, 4-CTA clusters) vs n_m = 8"
for nm in 8 16; do timeout 300 python tools/sweep_paths.py --shape 8192,28672,$nm --bs 1,16 --paths auto --steps 50 2>&1 | grep -v Warn; done
for nm in 8 16; do timeout 300 python tools/sweep_paths.py --shape 8192,28672,$nm --bs 2048 --paths auto --steps 10 2>&1 | grep -v Warn; done
