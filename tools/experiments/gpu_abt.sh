# bash tools/gpu_abt.sh "<ab_time args>" ["<ab_time args>" ...]
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv,noheader
for args in "$@"; do echo "== $args"; python tools/ab_time.py $args; done
