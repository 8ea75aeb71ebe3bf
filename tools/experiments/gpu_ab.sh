# interleaved A/B of experiment libs on ONE box: bash tools/gpu_ab.sh <bench args> -- LIB1 LIB2 ...
set -x
args=(); while [ "$1" != "--" ]; do args+=("$1"); shift; done; shift
python - <<'PY' > gpurun_out/ab_copy.txt 2>&1
import torch
a = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda"); b = torch.empty_like(a)
best = 0
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); b.copy_(a); e1.record(); e1.synchronize()
    best = max(best, 4 * (1 << 30) / (e0.elapsed_time(e1) * 1e-3) / 1e9)
print(f"copy GB/s {best:.0f}")
PY
cat gpurun_out/ab_copy.txt
for r in 1 2; do for V in "$@"; do
  MGLU_LIB=$PWD/tools/experiments/lib/libmglu_$V.so python bench.py "${args[@]}" --no-cpu-baseline --no-comparator --e2e-streams 0 > gpurun_out/ab_${V}_$r.json 2> gpurun_out/ab_${V}_$r.err
done; done
python tools/summ.py gpurun_out/ab_*.json
