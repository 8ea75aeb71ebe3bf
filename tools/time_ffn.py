"""FFN block timing, row f1 (experiment tool): the fused single launch (mglu_ffn_forward) vs the
two-launch composition (MGLU up-projection, then the dense W_o handle; PDL between them), same
data, one process, 4 rotating layer copies (> L2).  python tools/time_ffn.py --shape d,h,n_m --bs 1,4"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2506_23225_b200.mglu import Mglu, ffn_forward_fused  # noqa: E402
from synth import random_packed_codes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="4096,14336,4")
ap.add_argument("--bs", default="1,2,4")
ap.add_argument("--steps", type=int, default=200)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--layers", type=int, default=4)
a = ap.parse_args()
d, h, n_m = (int(v) for v in a.shape.split(","))
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6540.0)
g = torch.Generator(device="cuda").manual_seed(0)
layers = [(((torch.rand(h, d, device="cuda", generator=g) * 2 - 1) / d ** 0.5).to(torch.bfloat16),
           random_packed_codes(li, h, d, n_m, device="cuda"),
           ((torch.rand(d, h, device="cuda", generator=g) * 2 - 1) / h ** 0.5).to(torch.bfloat16)) for li in range(a.layers)]
up, down = Mglu(d, h, n_m, dtype="bf16"), Mglu(h, d, 0, dtype="bf16")
st = torch.cuda.Stream()


def timeit(fn):
    ts = []
    with torch.cuda.stream(st):
        for rep in range(a.reps + 1):
            torch.cuda._sleep(int(min(a.steps, 64) * 50 * 2000))
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
    ym = torch.empty(B, h, device="cuda", dtype=torch.bfloat16)
    out = torch.empty(B, d, device="cuda", dtype=torch.bfloat16)
    nb = 2 * h * d * 2 + h * d * n_m // 8 + 2 * B * d * 2 + 2 * B * h * 2
    us2 = timeit(lambda W, p, Wo: down.forward(up.forward(x, W, p, out=ym), Wo, None, out=out))
    us1 = timeit(lambda W, p, Wo: ffn_forward_fused(up, down, x, W, p, Wo, y_mid=ym, out=out, stream=st))
    print(f"B={B} two launches {us2:7.2f} us  {nb / us2 / 1e3:6.0f} GB/s  frac {nb / us2 / 1e3 / peak:.3f}", flush=True)
    print(f"B={B} fused        {us1:7.2f} us  {nb / us1 / 1e3:6.0f} GB/s  frac {nb / us1 / 1e3 / peak:.3f}", flush=True)
