"""Top-K routed MGLU -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md Appendix B, "Top-K routed MGLU":
    l = x W_r in R^{n_m}                                     (router logits)
    G(x) = Softmax(TopK(l))                                  (keep the K largest logits,
                                                              softmax over those, 0 elsewhere)
    MGLU_TopK(x) = sum_i G(x)_i g(x (M_i (.) W)) (.) x (Mbar_i (.) W)
Readings (R16-R18): W_r is stored like Wt, [n_m][d] (row i = logit i's weights); ties in
TopK go to the lowest index; the softmax runs over the K kept logits only (its weights
sum to 1).  The per-mask terms come from the oracle's own Eq. 3 partials (gate_i and value_i
computed independently), everything in binary64.
"""
from __future__ import annotations

import numpy as np

from .mglu_ref import act_np


def router_logits(x: np.ndarray, Wr: np.ndarray) -> np.ndarray:
    """l[b][i] = sum_k x[b][k] Wr[i][k], binary64."""
    return np.asarray(x, dtype=np.float64) @ np.asarray(Wr, dtype=np.float64).T


def topk_gate(logits: np.ndarray, K: int) -> np.ndarray:
    """G = Softmax(TopK(l)) per row: the K largest logits (ties -> lowest index) get
    softmax weights computed over those K values only; every other entry is exactly 0."""
    l = np.atleast_2d(np.asarray(logits, dtype=np.float64))
    n_m = l.shape[1]
    if not 1 <= K <= n_m:
        raise ValueError("K out of range")
    G = np.zeros_like(l)
    for b in range(l.shape[0]):
        # stable sort of -l: equal logits keep index order, so the lowest index wins ties
        keep = np.argsort(-l[b], kind="stable")[:K]
        z = l[b, keep] - np.max(l[b, keep])
        e = np.exp(z)
        G[b, keep] = e / np.sum(e)
    return G


def mglu_routed_from_partials(gate: np.ndarray, value: np.ndarray, G: np.ndarray, act: int) -> np.ndarray:
    """Eq. of P:724-728 from the per-mask streams: y[b][j] = sum_i G[b][i] g(gate_i[b][j]) value_i[b][j].
    gate, value: [n_m][B][h]; G: [B][n_m]."""
    terms = act_np(act, gate) * value                     # [n_m][B][h]
    return np.einsum("bi,ibj->bj", np.asarray(G, dtype=np.float64), terms)
