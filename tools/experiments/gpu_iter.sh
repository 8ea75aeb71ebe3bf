# iterate: quick tests + decode bench + ncu full profile of the decode kernel
bash tools/gpu_quick.sh
bash tools/gpu_prof.sh iter decode_b1 gemv_mma > /dev/null 2>&1
python3 tools/ncu_summary.py gpurun_out/prof_iter_raw.csv gpurun_out/prof_iter_details.csv > gpurun_out/prof_iter_summary.txt 2>&1
cat gpurun_out/prof_iter_summary.txt
