"""SwiMGLU FFN block with its down-projection -- TEST INFRASTRUCTURE ONLY.

PAPER.md Sec. 3.1: the FFN's intermediate activation is "mapped back to the hidden size by
an output projection": FFN(x) = MGLU(x) W_o, here with W_o stored like nn.Linear(h, d).weight,
Wo [d][h] (reading R19), so FFN(x) = MGLU(x) @ Wo^T.  Binary64 throughout, the MGLU part by the
oracle's own Eq. 3.
"""
from __future__ import annotations

import numpy as np

from .mglu_ref import mglu_forward_np


def ffn_forward_np(x: np.ndarray, Wt: np.ndarray, bits: np.ndarray, Wo: np.ndarray, act: int) -> np.ndarray:
    """FFN(x) = MGLU(x) Wo^T  (Eq. 3 for MGLU)."""
    y = mglu_forward_np(x, Wt, bits, act)                       # [B][h]
    return y @ np.asarray(Wo, dtype=np.float64).T               # [B][d]


def dense_np(x: np.ndarray, W: np.ndarray) -> np.ndarray:
    """The dense projection x W^T in binary64 (the n_m = 0 handle's definition)."""
    return np.asarray(x, dtype=np.float64) @ np.asarray(W, dtype=np.float64).T
