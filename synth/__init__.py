"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic: it draws x, Wt and the 0/1 mask bits and
returns them as plain numpy arrays (bf16 values as uint16 bit patterns).  Packing the bits into
the code layout, and everything after, happens separately on each side (oracle vs library).

Recipe:
  x   ~ N(0, 1)                  -- post-norm activations of a Llama-style model
  Wt  ~ U(-1/sqrt(d), 1/sqrt(d)) -- nn.Linear default init, which MGLU inherits
  M_i = (0.01 * randn > 0)       -- mask-logit init of Alg. 2 binarised with the strict
                                    threshold; i.e. Bernoulli(0.5) per mask and element.
                                    ``density`` != 0.5 draws Bernoulli(density) instead (learned-mask
                                    range 45-55 %) and "ones"/"zeros" give the special masks.
"""
from __future__ import annotations

import numpy as np
import torch


def to_bf16_bits(a: torch.Tensor) -> np.ndarray:
    """float tensor -> bf16 (round-to-nearest-even, torch's cast) bit patterns as uint16."""
    return a.to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16).copy()


def make_inputs(seed: int, B: int, d: int, h: int, n_m: int, dtype: str = "bf16",
                density: float | str = 0.5) -> dict:
    """Returns dict(x, Wt, bits) with x [B][d], Wt [h][d] (uint16 bf16 bits or float32),
    bits [n_m][h][d] uint8 in {0,1}."""
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(B, d, generator=g, dtype=torch.float32)
    bound = 1.0 / float(np.sqrt(d))
    Wt = (torch.rand(h, d, generator=g, dtype=torch.float32) * 2.0 - 1.0) * bound
    if density == "ones":
        bits = torch.ones(n_m, h, d, dtype=torch.uint8)
    elif density == "zeros":
        bits = torch.zeros(n_m, h, d, dtype=torch.uint8)
    elif density == 0.5:
        logits = 0.01 * torch.randn(n_m, h, d, generator=g, dtype=torch.float32)
        bits = (logits > 0).to(torch.uint8)
    else:
        bits = (torch.rand(n_m, h, d, generator=g) < float(density)).to(torch.uint8)
    out = {"bits": bits.numpy()}
    if dtype == "bf16":
        out["x"] = to_bf16_bits(x)
        out["Wt"] = to_bf16_bits(Wt)
    elif dtype == "f32":
        out["x"] = x.numpy()
        out["Wt"] = Wt.numpy()
    else:
        raise ValueError(dtype)
    return out


def make_logits(seed: int, n_m: int, h: int, d: int) -> np.ndarray:
    """Mask logits as Alg. 2 initialises them (0.01 * randn), float32."""
    g = torch.Generator().manual_seed(seed)
    return (0.01 * torch.randn(n_m, h, d, generator=g, dtype=torch.float32)).numpy()


def random_packed_codes(seed: int, h: int, d: int, n_m: int, device: str = "cpu") -> torch.Tensor:
    """Large-config masks drawn directly as uniformly random code bytes (every bit an independent
    Bernoulli(0.5), the same distribution as the recipe above), h*d*n_m/8 bytes.  Used where
    drawing n_m*h*d logits on the host would dominate (prefill shapes); parity at those shapes
    decodes the sampled rows with the oracle's own unpacker."""
    nbytes = (h * d * n_m + 7) // 8
    gen = torch.Generator(device=device).manual_seed(seed)
    return torch.randint(0, 256, (nbytes,), generator=gen, dtype=torch.uint8, device=device)
