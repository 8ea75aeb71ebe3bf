"""numpy float64 twin of the MGLU oracle -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Eq. 3, literally, with explicit masked weight matrices:

    MGLU_{n_m}(x) = sum_{i=1..n_m} g( x (M_i (.) W) ) (.) ( x (Mbar_i (.) W) ),  Mbar_i = 1 - M_i

This is the paper's own "naive" formulation ("n_m separate matrix-vector multiplies"),
evaluated in float64.  Orientation (R2): Wt is [h][d] (row j = output feature j, the
``A`` of Alg. 1), so ``x (M (.) W)`` is ``x @ (M * Wt).T``.
"""
from __future__ import annotations

import math

import numpy as np

# activation codes of the oracle (its own numbering; R5)
ACT_IDENTITY, ACT_SWISH, ACT_GELU, ACT_RELU, ACT_SIGMOID = 0, 1, 2, 3, 4
ACT_NAMES = {"identity": 0, "swish": 1, "gelu": 2, "relu": 3, "sigmoid": 4}

_erf = np.vectorize(math.erf, otypes=[np.float64])


def act_np(act: int, z: np.ndarray) -> np.ndarray:
    """g of Eq. 1/3.  swish(z) = z*sigmoid(z) (beta = 1, reading R5); GELU exact erf form
    (reading R5); relu; sigmoid; identity."""
    z = np.asarray(z, dtype=np.float64)
    if act == ACT_IDENTITY:
        return z.copy()
    if act == ACT_SWISH:
        return z / (1.0 + np.exp(-z))
    if act == ACT_GELU:
        return 0.5 * z * (1.0 + _erf(z / math.sqrt(2.0)))
    if act == ACT_RELU:
        return np.maximum(z, 0.0)
    if act == ACT_SIGMOID:
        return 1.0 / (1.0 + np.exp(-z))
    raise ValueError(f"unknown activation {act}")


def decode_bf16(u16: np.ndarray) -> np.ndarray:
    """bf16 bit pattern u -> the exact float64 value of the float32 with bits (u << 16)."""
    u = np.asarray(u16, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return u.view(np.float32).astype(np.float64)


def _bit_of_column(d: int) -> np.ndarray:
    """Reading R3: column 32g + e of a group sits at bit (e // 2) + 16 * (e % 2) of its word."""
    e = np.arange(d) % 32
    return (e // 2) + 16 * (e % 2)


def unpack_np(packed: np.ndarray, n_m: int, h: int, d: int) -> np.ndarray:
    """Pair-split bit-plane layout (reading R3): for row j, 32-column group g and mask i, one
    little-endian uint32 word (word index (j*(d/32) + g)*n_m + i-1) holds M_i[j, 32g..32g+31], column
    32g+e at bit (e//2) + 16*(e%2).  Mask i is bit (i-1) of the code (Alg. 1).
    Returns bits[i-1][j][k] in {0,1}."""
    if d % 32:
        raise ValueError("d must be a multiple of 32")
    words = np.frombuffer(np.ascontiguousarray(packed, dtype=np.uint8).tobytes(), dtype="<u4")
    words = words[: h * (d // 32) * n_m].reshape(h, d // 32, n_m)      # [j][g][i-1]
    per_col = np.repeat(words, 32, axis=1)                               # [j][k][i-1] (word of column k)
    shifts = _bit_of_column(d).astype(np.uint32)[None, :, None]
    bits = (per_col >> shifts) & np.uint32(1)
    return np.ascontiguousarray(np.transpose(bits, (2, 0, 1)).astype(np.uint8))


def pack_np(bits: np.ndarray) -> np.ndarray:
    """Inverse of :func:`unpack_np`: bits[n_m][h][d] in {0,1} -> packed bytes."""
    bits = np.asarray(bits, dtype=np.uint8)
    if bits.max(initial=0) > 1:
        raise ValueError("mask entries must be 0/1")
    n_m, h, d = bits.shape
    if d % 32:
        raise ValueError("d must be a multiple of 32")
    weights = (np.uint64(1) << _bit_of_column(d).astype(np.uint64))        # value of column k's bit
    contrib = np.transpose(bits, (1, 2, 0)).astype(np.uint64) * weights[None, :, None]   # [j][k][i]
    words = contrib.reshape(h, d // 32, 32, n_m).sum(axis=2).astype("<u4")               # [j][g][i]
    return np.frombuffer(words.tobytes(), dtype=np.uint8).copy()


def mglu_partials_np(x: np.ndarray, Wt: np.ndarray, bits: np.ndarray):
    """Alg. 1's accumulators, each as its own masked product:
    returns t [B][h], gate [n_m][B][h] = x (M_i (.) W), value [n_m][B][h] = x (Mbar_i (.) W)."""
    x = np.asarray(x, dtype=np.float64)
    Wt = np.asarray(Wt, dtype=np.float64)
    M = np.asarray(bits, dtype=np.float64)
    t = x @ Wt.T
    gate = np.stack([x @ (M[i] * Wt).T for i in range(M.shape[0])])
    value = np.stack([x @ ((1.0 - M[i]) * Wt).T for i in range(M.shape[0])])
    return t, gate, value


def mglu_forward_np(x: np.ndarray, Wt: np.ndarray, bits: np.ndarray, act: int) -> np.ndarray:
    """Eq. 3: y = sum_i g(x (M_i (.) W)) (.) x (Mbar_i (.) W); no 1/n_m factor (R6)."""
    _, gate, value = mglu_partials_np(x, Wt, bits)
    return np.sum(act_np(act, gate) * value, axis=0)
