export MGLU_LIB=$PWD/tools/experiments/lib/libmglu_A2.so
bash tools/gpu_prof.sh decA decode_b1 gemv_mma
python3 tools/ncu_summary.py gpurun_out/prof_decA_raw.csv gpurun_out/prof_decA_details.csv > gpurun_out/prof_decA_summary.txt 2>&1
python3 tools/ncu_src_top.py gpurun_out/prof_decA_source.csv > gpurun_out/prof_decA_srctop.txt 2>&1
rm -f gpurun_out/prof_decA.ncu-rep
