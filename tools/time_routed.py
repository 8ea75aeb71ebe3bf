"""Routed (Top-K) MGLU timing, row f2 (experiment tool): dense forward vs routed forward on the
interleaved codes vs routed forward on plane-major codes, same data, one process.  G is precomputed
(router launch not timed).  python tools/time_routed.py --shape d,h,n_m --bs 1,2,4 --ks 1,2"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import topk_gate  # noqa: E402  (test infrastructure: draws a valid G, no MGLU arithmetic)
from paper_2506_23225_b200.mglu import Mglu, mglu_pack_planes_device  # noqa: E402
from synth import random_packed_codes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="4096,14336,8")
ap.add_argument("--bs", default="1,2,4")
ap.add_argument("--ks", default="1,2")
ap.add_argument("--steps", type=int, default=200)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--layers", type=int, default=4)
a = ap.parse_args()
d, h, n_m = (int(v) for v in a.shape.split(","))
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6540.0)
g = torch.Generator(device="cuda").manual_seed(0)
layers = []
for li in range(a.layers):
    Wt = ((torch.rand(h, d, device="cuda", generator=g) * 2 - 1) / d ** 0.5).to(torch.bfloat16)
    packed = random_packed_codes(li, h, d, n_m, device="cuda")
    layers.append((Wt, packed, mglu_pack_planes_device(packed, n_m, h, d)))
st = torch.cuda.Stream()
layer = Mglu(d, h, n_m, act="swish", dtype="bf16")


def timeit(fn):
    ts = []
    with torch.cuda.stream(st):
        for rep in range(a.reps + 1):
            torch.cuda._sleep(int(min(a.steps, 64) * 30 * 2000))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for k in range(a.steps):
                fn(*layers[k % len(layers)])
            e1.record(st)
            e1.synchronize()
            if rep:
                ts.append(e0.elapsed_time(e1) * 1e3 / a.steps)
    return statistics.median(ts)


for B in (int(v) for v in a.bs.split(",")):
    x = torch.randn(B, d, device="cuda", generator=g).to(torch.bfloat16)
    y = torch.empty(B, h, device="cuda", dtype=torch.bfloat16)
    io = B * d * 2 + B * h * 2
    us = timeit(lambda W, p, pl: layer.forward(x, W, p, out=y))
    nb = h * d * 2 + h * d * n_m // 8 + io
    print(f"B={B} dense          {us:7.2f} us  {nb / us / 1e3:6.0f} GB/s  frac {nb / us / 1e3 / peak:.3f}", flush=True)
    for K in (int(v) for v in a.ks.split(",")):
        G = topk_gate(np.random.default_rng(B * 10 + K).standard_normal((B, n_m)), K).astype(np.float32)
        nsel = int((G != 0).any(axis=0).sum())
        Gd = torch.from_numpy(G).cuda()
        us_r = timeit(lambda W, p, pl: layer.forward_routed(x, W, p, Gd, K, out=y))
        us_p = timeit(lambda W, p, pl: layer.forward_routed_planes(x, W, pl, Gd, K, out=y))
        nb_p = h * d * 2 + h * d * nsel // 8 + io
        print(f"B={B} K={K} routed R3 {us_r:7.2f} us  (reads W + all {n_m} planes: {nb / us_r / 1e3:6.0f} GB/s)", flush=True)
        print(f"B={B} K={K} planes    {us_p:7.2f} us  (reads W + {nsel} planes: {nb_p / 1e6:.1f} MB, {nb_p / us_p / 1e3:6.0f} GB/s, "
              f"frac {nb_p / us_p / 1e3 / peak:.3f})", flush=True)
