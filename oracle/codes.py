"""Per-element mask codes -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md P:244 (Sec. 4, "Combine the n_m binary masks into a single integer code per weight
element"), Alg. 1's bit test ``mask[row,k] AND (1 << (i-1))``, and the listing's one
uint8 mask per element.  A code stream holds one w-bit field per element of the
[h][d] layer: element (j, k) at bit offset w*(j*d + k), little-endian (bit b of the stream is bit
b mod 8 of byte b div 8); mask i is bit i-1 of the field.  w = n_m is the dense stream of SURVEY
C3; w = 8 is the paper's one-byte-per-element listing.

Written bit by bit from that definition (no vectorised tricks), independent of the product
library's converter.
"""
from __future__ import annotations

import numpy as np


def codes_to_bits_np(stream, w: int, n_m: int, h: int, d: int) -> np.ndarray:
    """Code stream -> masks bits[i-1][j][k] in {0,1}.  Raises on a set field bit >= n_m."""
    if w not in (1, 2, 4, 8, 16) or not 1 <= n_m <= w:
        raise ValueError("bad field width")
    buf = bytes(np.asarray(stream, dtype=np.uint8).tobytes())
    if len(buf) != (h * d * w + 7) // 8:
        raise ValueError("stream size mismatch")
    bits = np.zeros((n_m, h, d), dtype=np.uint8)
    for j in range(h):
        for k in range(d):
            off = w * (j * d + k)
            field = 0
            for b in range(w):                       # gather the field one stream bit at a time
                pos = off + b
                field |= ((buf[pos // 8] >> (pos % 8)) & 1) << b
            if field >> n_m:
                raise ValueError("field bits above n_m are set")
            for i in range(1, n_m + 1):
                bits[i - 1, j, k] = (field >> (i - 1)) & 1        # Alg. 1: mask & (1 << (i-1))
    return bits


def bits_to_codes_np(bits, w: int) -> np.ndarray:
    """Inverse of :func:`codes_to_bits_np`: masks [n_m][h][d] -> a w-bit code stream."""
    bits = np.asarray(bits, dtype=np.uint8)
    n_m, h, d = bits.shape
    if w not in (1, 2, 4, 8, 16) or not 1 <= n_m <= w:
        raise ValueError("bad field width")
    out = bytearray((h * d * w + 7) // 8)
    for j in range(h):
        for k in range(d):
            field = sum(int(bits[i - 1, j, k]) << (i - 1) for i in range(1, n_m + 1))
            off = w * (j * d + k)
            for b in range(w):
                if (field >> b) & 1:
                    pos = off + b
                    out[pos // 8] |= 1 << (pos % 8)
    return np.frombuffer(bytes(out), dtype=np.uint8).copy()
