"""Per-batch timing of the bf16 paths in ONE process on the same data (experiment tool, not the bench):
python tools/sweep_paths.py --shape d,h,n_m --bs 1,2,4,8,16,32,64 --paths mma,tcdec,tcgen05

Each point: `steps` back-to-back mglu_forward calls (PDL launches, one stream) over `layers` distinct
weight copies (inputs larger than L2), timed with CUDA events behind a device-side sleep that lets the
host enqueue ahead; reported as us/call and the fraction of the measured HBM copy bandwidth on the
algorithmic bytes (W + codes + x + y)."""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2506_23225_b200.mglu import Mglu  # noqa: E402
from synth import random_packed_codes  # noqa: E402


ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="4096,14336,4")
ap.add_argument("--bs", default="1,2,4,8,16,32,64")
ap.add_argument("--paths", default="mma,tcdec,tcgen05")
ap.add_argument("--steps", type=int, default=200)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--layers", type=int, default=4)
a = ap.parse_args()
d, h, n_m = (int(v) for v in a.shape.split(","))
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6540.0)
g = torch.Generator(device="cuda").manual_seed(0)
layers = [(((torch.rand(h, d, device="cuda", generator=g) * 2 - 1) / d ** 0.5).to(torch.bfloat16),
           random_packed_codes(li, h, d, n_m, device="cuda")) for li in range(a.layers)]
st = torch.cuda.Stream()
for B in (int(v) for v in a.bs.split(",")):
    x = torch.randn(B, d, device="cuda", generator=g).to(torch.bfloat16)
    y = torch.empty(B, h, device="cuda", dtype=torch.bfloat16)
    nbytes = h * d * 2 + h * d * n_m // 8 + B * d * 2 + B * h * 2
    flops = 2 * B * d * h * (n_m + 1)
    for name in a.paths.split(","):
        layer = Mglu(d, h, n_m, act="swish", dtype="bf16")
        layer.set_path(name)
        ok = True
        times = []
        with torch.cuda.stream(st):
            for rep in range(a.reps + 1):
                torch.cuda._sleep(int(min(a.steps, 64) * 30 * 2000))
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                for k in range(a.steps):
                    Wt, c = layers[k % len(layers)]
                    try:
                        layer.forward(x, Wt, c, out=y)
                    except Exception as ex:  # path refuses the shape
                        ok = False
                        print(f"B={B:3d} {name:8s} refused: {str(ex)[:80]}")
                        break
                if not ok:
                    break
                e1.record(st)
                e1.synchronize()
                if rep:
                    times.append(e0.elapsed_time(e1) * 1e3 / a.steps)
        if ok:
            us = statistics.median(times)
            print(f"B={B:3d} {name:8s} {us:8.2f} us  {nbytes / us / 1e3:7.0f} GB/s  frac {nbytes / us / 1e3 / peak:.3f}"
                  f"  {flops / us / 1e6:7.1f} TFLOP/s  path={layer.last_path()}", flush=True)
        layer.close()
