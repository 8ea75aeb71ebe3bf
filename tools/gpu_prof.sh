# usage: bash tools/gpu_prof.sh <tag> <workload|d,h,nm,B> <kernel-regex>
tag=$1; wl=${2:-decode_b1}; kre=${3:-gemv_mma}
if [[ "$wl" == *,* ]]; then sel="--shape $wl"; else sel="--workload $wl"; fi
ncu --set full --clock-control none --import-source on -k regex:$kre -s 5 -c 1 -o gpurun_out/prof_$tag python bench.py $sel --steps 10 --warmup 3 --no-comparator --no-cpu-baseline --e2e-streams 0 > gpurun_out/prof_$tag.log 2>&1
ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_$tag.ncu-rep --page details --csv > gpurun_out/prof_${tag}_details.csv 2>/dev/null
ncu -i gpurun_out/prof_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${tag}_source.csv 2>/dev/null
echo prof done
