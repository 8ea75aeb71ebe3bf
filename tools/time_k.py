"""Fixed vs per-call cost of the bench's timed region (experiment tool): T(K) for K back-to-back
calls after the enqueue-ahead spin, config 3 B=1, 4 rotating layer copies; prints T(K) and T(K)/K."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2506_23225_b200.mglu import Mglu  # noqa: E402
from synth import random_packed_codes  # noqa: E402

d, h, n_m, B = 4096, 14336, 4, 1
g = torch.Generator(device="cuda").manual_seed(0)
layers = [(((torch.rand(h, d, device="cuda", generator=g) * 2 - 1) / d ** 0.5).to(torch.bfloat16),
           random_packed_codes(li, h, d, n_m, device="cuda")) for li in range(4)]
x = torch.randn(B, d, device="cuda", generator=g).to(torch.bfloat16)
y = torch.empty(B, h, device="cuda", dtype=torch.bfloat16)
layer = Mglu(d, h, n_m, dtype="bf16")
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for k in range(20):
        layer.forward(x, *layers[k % 4], out=y)
    st.synchronize()
    for K in (1, 2, 3, 5, 10, 20, 50, 200, 500):
        ts = []
        for rep in range(5):
            torch.cuda._sleep(int((1e3 + 40 * K) * 1965))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for k in range(K):
                layer.forward(x, *layers[k % 4], out=y)
            e1.record(st)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        t = ts[len(ts) // 2]
        print(f"K={K:4d}  T={t:9.2f} us  T/K={t / K:7.2f} us", flush=True)
