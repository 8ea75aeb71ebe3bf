"""ctypes loader for ``mglu_oracle.c`` -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

``build_c_oracle()`` compiles ``oracle/libmglu_oracle.so`` with plain ``gcc -O2 -fopenmp``
(no SIMD intrinsics, no -ffast-math: the binary64 loop order is the source order).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mglu_oracle.c")
_LIB = os.path.join(_HERE, "libmglu_oracle.so")


def build_c_oracle(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_P = ctypes.POINTER
_dp = _P(ctypes.c_double)
_u8p = _P(ctypes.c_uint8)
_i64p = _P(ctypes.c_int64)


def _ptr(a, t):
    return a.ctypes.data_as(t) if a is not None else None


class COracle:
    """Thin marshalling around the C oracle.  All arithmetic lives in mglu_oracle.c."""

    def __init__(self):
        lib = ctypes.CDLL(build_c_oracle())
        lib.oracle_pack.argtypes = [_u8p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, _u8p]
        lib.oracle_unpack.argtypes = [_u8p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, _u8p]
        lib.oracle_mglu_forward.argtypes = [_dp, ctypes.c_int64, ctypes.c_int64, _dp, _i64p,
                                            ctypes.c_int64, _u8p, ctypes.c_int, ctypes.c_int,
                                            _dp, _dp, _dp]
        lib.oracle_num_threads.restype = ctypes.c_int
        lib.oracle_set_num_threads.argtypes = [ctypes.c_int]
        self.lib = lib

    def num_threads(self) -> int:
        return int(self.lib.oracle_num_threads())

    def set_num_threads(self, n: int) -> None:
        self.lib.oracle_set_num_threads(int(n))

    def pack(self, bits: np.ndarray) -> np.ndarray:
        bits = np.ascontiguousarray(bits, dtype=np.uint8)
        n_m, h, d = bits.shape
        out = np.zeros((n_m * h * d + 7) // 8, dtype=np.uint8)
        rc = self.lib.oracle_pack(_ptr(bits, _u8p), n_m, h, d, _ptr(out, _u8p))
        if rc:
            raise ValueError(f"oracle_pack rc={rc}")
        return out

    def unpack(self, packed: np.ndarray, n_m: int, h: int, d: int) -> np.ndarray:
        packed = np.ascontiguousarray(packed, dtype=np.uint8)
        out = np.zeros((n_m, h, d), dtype=np.uint8)
        rc = self.lib.oracle_unpack(_ptr(packed, _u8p), n_m, h, d, _ptr(out, _u8p))
        if rc:
            raise ValueError(f"oracle_unpack rc={rc}")
        return out

    def forward(self, x: np.ndarray, Wt_sel: np.ndarray, cols: np.ndarray, packed: np.ndarray,
                n_m: int, act: int, want_partials: bool = False):
        """Eq. 3 for all token rows of ``x`` and the output columns ``cols``.
        ``Wt_sel[c] = Wt[cols[c]]`` (float64).  Returns y [B][ncols] (and z [B][2n_m][ncols],
        t [B][ncols] when ``want_partials``)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.ndim == 1:
            x = x[None]
        B, d = x.shape
        Wt_sel = np.ascontiguousarray(Wt_sel, dtype=np.float64)
        cols = np.ascontiguousarray(cols, dtype=np.int64)
        packed = np.ascontiguousarray(packed, dtype=np.uint8)
        nc = cols.shape[0]
        assert Wt_sel.shape == (nc, d)
        y = np.zeros((B, nc), dtype=np.float64)
        z = np.zeros((B, 2 * n_m, nc), dtype=np.float64) if want_partials else None
        t = np.zeros((B, nc), dtype=np.float64) if want_partials else None
        rc = self.lib.oracle_mglu_forward(_ptr(x, _dp), B, d, _ptr(Wt_sel, _dp), _ptr(cols, _i64p),
                                          nc, _ptr(packed, _u8p), n_m, act, _ptr(y, _dp),
                                          _ptr(z, _dp), _ptr(t, _dp))
        if rc:
            raise ValueError(f"oracle_mglu_forward rc={rc}")
        return (y, z, t) if want_partials else y
