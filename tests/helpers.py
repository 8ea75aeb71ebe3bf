"""Shared test helpers: run the CUDA path through the C ABI and the oracle on the same seeded
inputs, and the comparison metric of reading R10."""
from __future__ import annotations

import numpy as np
import torch

from oracle import COracle, decode_bf16
from synth import make_inputs

ACTS = {"identity": 0, "swish": 1, "gelu": 2, "relu": 3, "sigmoid": 4}
TOL = {"bf16": 1e-2, "f32": 1e-5}          # north_star: max relative error, normwise (R10)
TIGHT = {"bf16": 4e-3, "f32": 1e-6}        # regression band (a correct bf16 kernel lands at 1.8-2.3e-3)


def normwise_err(y: np.ndarray, ref: np.ndarray) -> float:
    """Reading R10: per token row, max_j |y - ref| / max_j |ref|; the worst row is returned."""
    y = np.atleast_2d(np.asarray(y, dtype=np.float64))
    ref = np.atleast_2d(np.asarray(ref, dtype=np.float64))
    worst = 0.0
    for b in range(ref.shape[0]):
        scale = np.max(np.abs(ref[b]))
        diff = np.max(np.abs(y[b] - ref[b]))
        if scale == 0.0:
            if diff != 0.0:
                return float("inf")
            continue
        worst = max(worst, diff / scale)
    return worst


def to_device(inp: dict, dtype: str, device="cuda"):
    """x / Wt numpy (uint16 bf16 bits or f32) -> torch tensors on the GPU."""
    if dtype == "bf16":
        x = torch.from_numpy(inp["x"].view(np.int16).copy()).view(torch.bfloat16)
        Wt = torch.from_numpy(inp["Wt"].view(np.int16).copy()).view(torch.bfloat16)
    else:
        x = torch.from_numpy(inp["x"].copy())
        Wt = torch.from_numpy(inp["Wt"].copy())
    return x.to(device).contiguous(), Wt.to(device).contiguous()


def oracle_inputs(inp: dict, dtype: str):
    if dtype == "bf16":
        return decode_bf16(inp["x"]), decode_bf16(inp["Wt"])
    return inp["x"].astype(np.float64), inp["Wt"].astype(np.float64)


_ORACLE = None


def oracle() -> COracle:
    global _ORACLE
    if _ORACLE is None:
        _ORACLE = COracle()
    return _ORACLE


def oracle_forward(inp: dict, dtype: str, n_m: int, act: str, cols=None, want_partials=False):
    """Eq. 3 by the C oracle on the oracle's own packing of the bits."""
    o = oracle()
    x, Wt = oracle_inputs(inp, dtype)
    packed = o.pack(inp["bits"])
    h = Wt.shape[0]
    cols = np.arange(h) if cols is None else np.asarray(cols)
    return o.forward(x, Wt[cols], cols, packed, n_m, ACTS[act], want_partials=want_partials)


def gpu_forward(inp: dict, dtype: str, n_m: int, act: str, path: str = "auto", packed=None):
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    x, Wt = to_device(inp, dtype)
    B, d = x.shape
    h = Wt.shape[0]
    if packed is None:
        packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
    layer = Mglu(d, h, n_m, act=act, dtype=dtype, path=path)
    y = layer.forward(x, Wt, packed)
    torch.cuda.synchronize()
    used = layer.last_path()
    layer.close()
    return y.float().cpu().numpy().astype(np.float64), used


__all__ = ["ACTS", "TOL", "TIGHT", "normwise_err", "to_device", "oracle_inputs", "oracle",
           "oracle_forward", "gpu_forward", "make_inputs"]
