# decode experiment lib with env knobs: MGLU_LIB=<lib> then a list of "ENV=VAL" settings
set -x
export MGLU_LIB=$PWD/tools/experiments/lib/libmglu_$1.so; shift
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
for kv in "$@"; do
  tag=$(echo $kv | tr '=' '_')
  for r in 1 2; do env $kv python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --no-comparator --e2e-streams 0 > gpurun_out/v2_${tag}_d20_$r.json 2> gpurun_out/v2_${tag}_d20_$r.err; done
  env $kv python bench.py --steps 500 --no-cpu-baseline --no-comparator --e2e-streams 0 > gpurun_out/v2_${tag}_500.json 2> gpurun_out/v2_${tag}_500.err
done
python tools/summ.py gpurun_out/v2_*.json
