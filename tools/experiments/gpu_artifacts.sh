# Round artifacts: default bench line, reference arm, ncu launch list + full capture of the decode kernel
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw,temperature.gpu --format=csv > gpurun_out/nvsmi.txt
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
python bench.py --workload decode_b8 --no-cpu-baseline > gpurun_out/bench_decode_b8.json 2>&1
python bench.py --workload decode7b_b1 --no-cpu-baseline > gpurun_out/bench_decode7b.json 2>&1
for nm in 1 2 4 8; do python bench.py --workload sweep_b1_nm$nm --no-cpu-baseline --layers 2 > gpurun_out/bench_sweep_nm$nm.json 2>&1; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_decode_b1.csv python bench.py --steps 20 --warmup 3 --no-comparator --no-cpu-baseline --clock-window 0 > /dev/null 2>&1
bash tools/gpu_prof.sh decode_b1 decode_b1 gemv_mma
python3 tools/ncu_summary.py gpurun_out/prof_decode_b1_raw.csv gpurun_out/prof_decode_b1_details.csv > gpurun_out/prof_decode_b1_summary.txt
python3 - <<'PY'
import csv, json
rows = list(csv.reader(open("gpurun_out/prof_decode_b1_raw.csv")))
hdr, units, vals = rows[0], rows[1], rows[2]
m = dict(zip(hdr, vals)); u = dict(zip(hdr, units))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd = float(m["dram__bytes_read.sum"]) * scale[u["dram__bytes_read.sum"]]
wr = float(m["dram__bytes_write.sum"]) * scale[u["dram__bytes_write.sum"]]
json.dump({"decode_b1": {"kernel": "gemv_mma_kernel", "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
           "source": "ncu --set full --clock-control none (cold cache, one launch)"}}, open("gpurun_out/ncu_traffic.json", "w"), indent=1)
PY
echo artifacts done
