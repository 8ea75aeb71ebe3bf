# row-split tcgen05 GEMV: parity + per-B sweep against the HMMA kernel, the stream-K form and the tile GEMM
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tcdec.py tests/test_gpu_bounds.py -x -q > gpurun_out/rows_tests.log 2>&1; tail -3 gpurun_out/rows_tests.log
echo "== config 3, row split (AUTO rows)"; timeout 300 python tools/sweep_paths.py --shape 4096,14336,4 --bs 1,2,4,8,16,24,32,48,64 --paths mma,tcdec,tcgen05 2>&1 | grep -v Warn
echo "== config 3, stream-K forced"; MGLU_SK_ROWS=0 timeout 300 python tools/sweep_paths.py --shape 4096,14336,4 --bs 1,8,16,32,64 --paths tcdec 2>&1 | grep -v Warn
echo "== config 5 B=1 n_m sweep"; for nm in 1 2 4 8; do timeout 300 python tools/sweep_paths.py --shape 8192,28672,$nm --bs 1 --paths mma,tcdec --steps 100 2>&1 | grep -v Warn; done
echo "== config 2"; timeout 300 python tools/sweep_paths.py --shape 4096,11008,4 --bs 1,8 --paths mma,tcdec 2>&1 | grep -v Warn
