"""Training path of MGLU -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md Alg. 2: the forward uses the hard masks ``hard = (soft > 0)`` and the
straight-through estimator ``(hard - soft).detach() + soft`` passes the gradient with respect to
the mask to the soft logits unchanged; W gets the exact gradient of the hard-mask forward
("M is optimized jointly with W via the straight-through estimator").  Reading R21
(DESIGN.md): d_logits_i = dL/dM_i of Eq. 3 with M_i treated as continuous, evaluated at the hard
masks -- the gradient of SPEC's relaxed surrogate at soft = hard.

With the forward streams of Eq. 3, s_i = x (M_i (.) W) and v_i = x (Mbar_i (.) W), and the
upstream gradient dy [B][h]:
    a_i = dy * g'(s_i) * v_i        (dL/ds_i)          c_i = dy * g(s_i)   (dL/dv_i)
    dL/dx     = sum_i a_i (M_i (.) W) + c_i (Mbar_i (.) W)          (as [B][h] @ [h][d])
    dL/dW     = sum_i M_i (.) (a_i^T x) + Mbar_i (.) (c_i^T x)
    dL/dM_i   = W (.) (a_i^T x - c_i^T x)
Each term is written out with explicit masked matrices, in binary64, no reassociation beyond the
matrix products.
"""
from __future__ import annotations

import math

import numpy as np

from .mglu_ref import ACT_GELU, ACT_IDENTITY, ACT_RELU, ACT_SIGMOID, ACT_SWISH, act_np

_erf = np.vectorize(math.erf, otypes=[np.float64])


def act_grad_np(act: int, z: np.ndarray) -> np.ndarray:
    """g'(z): swish' = sigma(z)(1 + z(1 - sigma(z))); gelu' = Phi(z) + z phi(z);
    relu' = 1 for z > 0 else 0 (subgradient 0 at 0); sigmoid' = sigma(1 - sigma)."""
    z = np.asarray(z, dtype=np.float64)
    if act == ACT_IDENTITY:
        return np.ones_like(z)
    if act == ACT_SWISH:
        s = 1.0 / (1.0 + np.exp(-z))
        return s * (1.0 + z * (1.0 - s))
    if act == ACT_GELU:
        return 0.5 * (1.0 + _erf(z / math.sqrt(2.0))) + z * np.exp(-0.5 * z * z) / math.sqrt(2.0 * math.pi)
    if act == ACT_RELU:
        return (z > 0).astype(np.float64)
    if act == ACT_SIGMOID:
        s = 1.0 / (1.0 + np.exp(-z))
        return s * (1.0 - s)
    raise ValueError(f"unknown activation {act}")


def mglu_backward_np(x, Wt, bits, dy, act):
    """(d_x [B][d], d_W [h][d], d_logits [n_m][h][d]) of Eq. 3 under Alg. 2's STE (see module doc)."""
    x = np.asarray(x, dtype=np.float64)
    Wt = np.asarray(Wt, dtype=np.float64)
    M = np.asarray(bits, dtype=np.float64)
    dy = np.asarray(dy, dtype=np.float64)
    dx = np.zeros_like(x)
    dW = np.zeros_like(Wt)
    dl = np.zeros_like(M)
    for i in range(M.shape[0]):
        Wg, Wv = M[i] * Wt, (1.0 - M[i]) * Wt                  # M_i (.) W and Mbar_i (.) W, as [h][d]
        s, v = x @ Wg.T, x @ Wv.T                              # the forward streams [B][h]
        a = dy * act_grad_np(act, s) * v                       # dL/ds_i
        c = dy * act_np(act, s)                                # dL/dv_i
        dx += a @ Wg + c @ Wv
        dW += M[i] * (a.T @ x) + (1.0 - M[i]) * (c.T @ x)
        dl[i] = Wt * (a.T @ x - c.T @ x)
    return dx, dW, dl


def relaxed_forward_np(x, Wt, soft, act):
    """SPEC's relaxed surrogate: Eq. 3 with M_i replaced by the real values soft_i and
    Mbar_i by 1 - soft_i; equals the hard forward when soft is 0/1.  d_logits is its gradient at
    soft = the hard masks (finite-difference oracle of the STE pass-through)."""
    x = np.asarray(x, dtype=np.float64)
    Wt = np.asarray(Wt, dtype=np.float64)
    S = np.asarray(soft, dtype=np.float64)
    y = 0.0
    for i in range(S.shape[0]):
        y = y + act_np(act, x @ (S[i] * Wt).T) * (x @ ((1.0 - S[i]) * Wt).T)
    return y
