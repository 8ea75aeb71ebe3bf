# ncu --set full of the tcgen05 GEMV (row split) at B = 1, 16, 64 + source-level stall tops
mkdir -p gpurun_out
for B in 1 16 64; do
  bash tools/gpu_profx.sh tc_b$B gemv_tc --shape 4096,14336,4,$B --path tcdec > /dev/null 2>&1
  echo "== B=$B"; cat gpurun_out/prof_tc_b${B}_summary.txt
  python3 tools/ncu_src_top.py gpurun_out/prof_tc_b${B}_source.csv 30 > gpurun_out/prof_tc_b${B}_srctop.txt 2>&1; head -32 gpurun_out/prof_tc_b${B}_srctop.txt
done
