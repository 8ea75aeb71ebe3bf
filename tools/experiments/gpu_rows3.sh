mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv
echo "== config 3"; timeout 300 python tools/sweep_paths.py --shape 4096,14336,4 --bs 1,16,64 --paths mma,tcdec 2>&1 | grep -v Warn
echo "== config 3 stream-K"; MGLU_SK_ROWS=0 timeout 300 python tools/sweep_paths.py --shape 4096,14336,4 --bs 1,16,64 --paths tcdec 2>&1 | grep -v Warn
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv
