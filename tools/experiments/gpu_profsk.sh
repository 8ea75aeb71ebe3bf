bash tools/gpu_prof.sh sk8 4096,14336,4,8 gemv_tc > /dev/null 2>&1
python3 tools/ncu_summary.py gpurun_out/prof_sk8_raw.csv gpurun_out/prof_sk8_details.csv > gpurun_out/prof_sk8_summary.txt 2>&1
python3 tools/ncu_src_top.py gpurun_out/prof_sk8_source.csv 40 > gpurun_out/prof_sk8_srctop.txt 2>&1
rm -f gpurun_out/prof_sk8.ncu-rep
