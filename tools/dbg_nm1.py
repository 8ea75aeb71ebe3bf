import sys, torch, numpy as np
sys.path.insert(0, '.')
from tests.helpers import gpu_forward, oracle_forward, normwise_err
from synth import make_inputs
for (d,h,B) in [(256,128,1),(256,128,300),(1024,256,500),(8192,256,2048)]:
    inp = make_inputs(1, B=B, d=d, h=h, n_m=1, dtype="bf16")
    try:
        y, used = gpu_forward(inp, "bf16", 1, "swish", path="tcgen05")
        print(d,h,B, used, normwise_err(y, oracle_forward(inp, "bf16", 1, "swish")), flush=True)
    except Exception as e:
        print(d,h,B,'ERR',str(e)[:200], flush=True); break
