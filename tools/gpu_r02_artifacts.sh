# Round-2 artifacts: full GPU suite + smoke, bench lines (driver default, 20-step, reference arm,
# prefill, batched decode, config-5 n_m = 8), ncu launch lists and --set full captures of the three
# hot kernels with their DRAM traffic (profiles/ncu_traffic.json)
mkdir -p gpurun_out/r02
O=gpurun_out/r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw,temperature.gpu --format=csv > $O/nvsmi.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 300 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_default_20.json 2> $O/bench_default_20.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
for w in prefill decode_b8 decode_b64 sweep_b1_nm8 sweep_b2048_nm4; do timeout 300 python bench.py --workload $w --no-cpu-baseline --layers 2 > $O/bench_$w.json 2> $O/bench_$w.err; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_decode_b1.csv python bench.py --steps 20 --warmup 3 --no-comparator --no-cpu-baseline --clock-window 0 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_prefill.csv python bench.py --workload prefill --layers 1 --steps 5 --warmup 3 --no-comparator --no-cpu-baseline --clock-window 0 > /dev/null 2>&1
bash tools/gpu_profx.sh decode_b1 gemv_mma --workload decode_b1 > /dev/null 2>&1
bash tools/gpu_profx.sh decode_b8 gemv_tc --workload decode_b8 > /dev/null 2>&1
bash tools/gpu_profx.sh prefill gemm_tc --workload prefill --layers 1 > /dev/null 2>&1
for t in decode_b1 decode_b8 prefill; do cp gpurun_out/prof_${t}_summary.txt $O/ncu_${t}_summary.txt; python3 tools/ncu_src_top.py gpurun_out/prof_${t}_source.csv 25 > $O/ncu_${t}_srctop.txt 2>&1; done
python3 - <<'PY'
import csv, json
out = {}
for tag in ("decode_b1", "decode_b8", "prefill"):
    rows = list(csv.reader(open(f"gpurun_out/prof_{tag}_raw.csv")))
    hdr, units, vals = rows[0], rows[1], rows[2]
    m = dict(zip(hdr, vals)); u = dict(zip(hdr, units))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = float(m["dram__bytes_read.sum"].replace(",", "")) * scale[u["dram__bytes_read.sum"]]
    wr = float(m["dram__bytes_write.sum"].replace(",", "")) * scale[u["dram__bytes_write.sum"]]
    out[tag] = {"kernel": m.get("Kernel Name", m.get("Function Name", "?"))[:80], "dram_bytes_per_launch": rd + wr,
                "dram_read": rd, "dram_write": wr,
                "source": f"ncu --set full --clock-control none (one launch), profiles/r02_ncu_{tag}_summary.txt"}
json.dump(out, open("gpurun_out/r02/ncu_traffic.json", "w"), indent=1)
PY
for f in $O/bench_*.json; do echo "$f: $(python3 -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d.get('us_per_call'), d.get('value'), d.get('unit'), d.get('roofline',{}).get('frac'))" 2>&1 | tail -1)"; done
echo artifacts done
