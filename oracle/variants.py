"""Partial-mask ablation variants of MGLU -- TEST INFRASTRUCTURE ONLY.

PAPER.md Appendix "Partial Mask Ablation", single-mask definitions:
    NG (no gate mask):  h_NG(x) = g(xW) (.) (x(Mbar (.) W))
    NV (no value mask): h_NV(x) = g(x(M (.) W)) (.) (xW)
    NM (no masks):      h_NM(x) = g(xW) (.) (xW)
Reading R20: for n_m masks each term of Eq. 3 is replaced the same way and summed over i (n_m = 1
is the paper's case).  The streams are the oracle's own, computed independently:
t = xW, gate_i = x(M_i (.) W), value_i = x(Mbar_i (.) W).
"""
from __future__ import annotations

import numpy as np

from .mglu_ref import act_np

VARIANTS = {"standard": 0, "no_gate_mask": 1, "no_value_mask": 2, "no_masks": 3}


def mglu_variant_from_streams(t: np.ndarray, gate: np.ndarray, value: np.ndarray, act: int, variant: int) -> np.ndarray:
    """t [B][h], gate / value [n_m][B][h] -> y [B][h] for the variant (0 = Eq. 3)."""
    n_m = gate.shape[0]
    if variant == 0:
        return np.sum(act_np(act, gate) * value, axis=0)
    if variant == 1:                                           # g(xW) (.) x(Mbar_i W)
        return np.sum(act_np(act, t)[None] * value, axis=0)
    if variant == 2:                                           # g(x(M_i W)) (.) xW
        return np.sum(act_np(act, gate) * t[None], axis=0)
    if variant == 3:                                           # g(xW) (.) xW, once per mask term
        return n_m * act_np(act, t) * t
    raise ValueError(f"unknown variant {variant}")
