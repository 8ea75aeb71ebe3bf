"""Interleaved A/B timing of several libmglu builds in ONE process on the same data (box-to-box
clock/power variance cancels): python tools/ab_time.py --shape d,h,n_m,B --libs A B ... where
each name is tools/experiments/lib/libmglu_<name>.so or 'prod' (the product library)."""
import argparse
import ctypes
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="4096,14336,4,1")
ap.add_argument("--libs", nargs="+", required=True)
ap.add_argument("--steps", type=int, default=200)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--path", type=int, default=0)
a = ap.parse_args()
d, h, n_m, B = (int(v) for v in a.shape.split(","))
from synth import random_packed_codes  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(B, d, device="cuda", generator=g).to(torch.bfloat16)
layers = [(((torch.rand(h, d, device="cuda", generator=g) * 2 - 1) / d ** 0.5).to(torch.bfloat16),
           random_packed_codes(li, h, d, n_m, device="cuda")) for li in range(a.layers)]
y = torch.empty(B, h, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.Stream()
libs = {}
for name in a.libs:
    path = os.path.join(ROOT, "paper_2506_23225_b200", "libmglu.so") if name == "prod" else \
        os.path.join(ROOT, "tools", "experiments", "lib", f"libmglu_{name}.so")
    lib = ctypes.CDLL(path)
    vp = ctypes.c_void_p
    lib.mglu_create.argtypes = [ctypes.POINTER(vp), ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    lib.mglu_forward.argtypes = [vp, vp, ctypes.c_int64, vp, vp, vp, vp]
    lib.mglu_set_path.argtypes = [vp, ctypes.c_int]
    hd = vp()
    assert lib.mglu_create(ctypes.byref(hd), d, h, n_m, 1, 0, 0) == 0
    if a.path:
        lib.mglu_set_path(hd, a.path)
    libs[name] = (lib, hd)


def run(name, K):
    lib, hd = libs[name]
    with torch.cuda.stream(st):
        torch.cuda._sleep(int(min(K, 64) * 25 * 2000))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for k in range(K):
            Wt, c = layers[k % len(layers)]
            r = lib.mglu_forward(hd, x.data_ptr(), B, Wt.data_ptr(), c.data_ptr(), y.data_ptr(), st.cuda_stream)
            assert r == 0, (name, r)
        e1.record(st)
        e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / K


try:
    import pynvml
    pynvml.nvmlInit()
    _nv = pynvml.nvmlDeviceGetHandleByIndex(0)
    clk = lambda: pynvml.nvmlDeviceGetClockInfo(_nv, pynvml.NVML_CLOCK_SM)   # noqa: E731
except Exception:  # noqa: BLE001
    clk = lambda: -1   # noqa: E731
for name in libs:
    run(name, 20)
res = {n: [] for n in libs}
clocks = []
for rep in range(a.reps):
    for name in libs:
        res[name].append(run(name, a.steps))
        clocks.append(clk())
ab = h * d * 2 + h * d * n_m // 8 + B * d * 2 + B * h * 2
for name, v in res.items():
    m = statistics.median(v)
    print(f"{name:24s} median {m:7.2f} us  min {min(v):7.2f}  max {max(v):7.2f}  {ab / m / 1e3:7.0f} GB/s"
          f"  {2 * B * d * h * (n_m + 1) / m / 1e6:7.1f} TFLOP/s  sm_mhz after reps {clocks}")
