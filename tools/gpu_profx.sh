# usage: bash tools/gpu_profx.sh <tag> <kernel-regex> <bench args...>   (ncu --set full of one launch + summary)
tag=$1; kre=$2; shift 2
ncu --set full --clock-control none --import-source on -k regex:$kre -s 5 -c 1 -o gpurun_out/prof_$tag python bench.py "$@" --steps 10 --warmup 3 --no-comparator --no-cpu-baseline --clock-window 0 > gpurun_out/prof_$tag.log 2>&1
ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_$tag.ncu-rep --page details --csv > gpurun_out/prof_${tag}_details.csv 2>/dev/null
ncu -i gpurun_out/prof_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${tag}_source.csv 2>/dev/null
python3 tools/ncu_summary.py gpurun_out/prof_${tag}_raw.csv gpurun_out/prof_${tag}_details.csv > gpurun_out/prof_${tag}_summary.txt 2>&1
[ -z "$KEEP_REP" ] && rm -f gpurun_out/prof_$tag.ncu-rep   # gpurun brings back <= 64 MiB
echo "== $tag"; cat gpurun_out/prof_${tag}_summary.txt
