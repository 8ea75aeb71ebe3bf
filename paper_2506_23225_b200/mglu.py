"""Thin Python binding of libmglu (include/mglu.h) -- argument marshalling only.

Every step of the forward pass runs in the CUDA kernels of ``libmglu.so``; this module converts
torch tensors / numpy arrays to raw pointers, picks torch's current stream and turns status codes
into exceptions.  There is no CPU fallback: if the library is missing, importing the binding
raises :class:`MgluLibraryMissing`.

The functions carry the C names (``mglu_create``, ``mglu_forward``, ...); :class:`Mglu` is a
small convenience wrapper owning a handle.
"""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import torch

_PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG_DIR, "libmglu.so")
HEADER_PATH = os.path.join(os.path.dirname(_PKG_DIR), "include", "mglu.h")

MGLU_OK, MGLU_ERR_INVALID_ARG, MGLU_ERR_UNSUPPORTED, MGLU_ERR_MISALIGNED, MGLU_ERR_CUDA, MGLU_ERR_OOM = range(6)
ACT = {"identity": 0, "swish": 1, "gelu": 2, "relu": 3, "sigmoid": 4}
DTYPE = {"bf16": 0, "f32": 1}
PATH = {"auto": 0, "simt": 1, "mma": 2, "tcgen05": 3, "tcdec": 4, "tcrow": 5}
TORCH_DTYPE = {"bf16": torch.bfloat16, "f32": torch.float32}


class MgluLibraryMissing(ImportError):
    pass


class MgluError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


_lib = None


def load_library(path: str | None = None) -> ctypes.CDLL:
    """Load libmglu.so (built in-tree by ``paper_2506_23225_b200.build``; MGLU_LIB points at an
    experiment build instead -- those are never written over the product library)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("MGLU_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise MgluLibraryMissing(
            f"{path} not found: build it with `python -m paper_2506_23225_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    vp, i64, c_int, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
    u8p = ctypes.POINTER(ctypes.c_uint8)
    f32p = ctypes.POINTER(ctypes.c_float)
    sig = {
        "mglu_create": ([ctypes.POINTER(vp), i64, i64, c_int, c_int, c_int, c_int], c_int),
        "mglu_destroy": ([vp], c_int),
        "mglu_set_path": ([vp, c_int], c_int),
        "mglu_set_variant": ([vp, c_int], c_int),
        "mglu_set_debug": ([vp, c_int], c_int),
        "mglu_reserve": ([vp, i64, vp], c_int),
        "mglu_backward": ([vp, vp, i64, vp, vp, vp, vp, vp, vp, vp], c_int),
        "mglu_forward": ([vp, vp, i64, vp, vp, vp, vp], c_int),
        "mglu_forward_partials": ([vp, vp, i64, vp, vp, vp, vp], c_int),
        "mglu_forward_host": ([vp, vp, i64, vp, vp, vp, vp], c_int),
        "mglu_router_topk": ([vp, vp, i64, vp, c_int, vp, vp], c_int),
        "mglu_forward_routed": ([vp, vp, i64, vp, vp, vp, c_int, vp, vp], c_int),
        "mglu_forward_routed_planes": ([vp, vp, i64, vp, vp, vp, c_int, vp, vp], c_int),
        "mglu_ffn_forward": ([vp, vp, vp, i64, vp, vp, vp, vp, vp, vp], c_int),
        "mglu_pack_planes_host": ([vp, c_int, i64, i64, vp], c_int),
        "mglu_pack_planes_device": ([vp, c_int, i64, i64, vp, vp], c_int),
        "mglu_packed_mask_bytes": ([i64, i64, c_int], sz),
        "mglu_pack_masks_host": ([vp, c_int, i64, i64, vp], c_int),
        "mglu_code_stream_bytes": ([i64, i64, c_int], sz),
        "mglu_codes_to_bits_host": ([vp, c_int, c_int, i64, i64, vp], c_int),
        "mglu_pack_codes_host": ([vp, c_int, c_int, i64, i64, vp], c_int),
        "mglu_unpack_codes_host": ([vp, c_int, i64, i64, c_int, vp], c_int),
        "mglu_pack_logits_host": ([vp, c_int, i64, i64, vp], c_int),
        "mglu_unpack_masks_host": ([vp, c_int, i64, i64, vp], c_int),
        "mglu_pack_masks_device": ([vp, c_int, i64, i64, vp, vp], c_int),
        "mglu_pack_logits_device": ([vp, c_int, i64, i64, vp, vp], c_int),
        "mglu_unpack_masks_device": ([vp, c_int, i64, i64, vp, vp], c_int),
        "mglu_last_launch_count": ([vp], c_int),
        "mglu_last_path": ([vp], c_int),
        "mglu_status_string": ([c_int], ctypes.c_char_p),
        "mglu_last_error": ([vp], ctypes.c_char_p),
        "mglu_version": ([], ctypes.c_char_p),
    }
    del u8p, f32p
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def header_functions(path: str = HEADER_PATH) -> list[str]:
    """Names of every function declared in include/mglu.h."""
    text = open(path).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mglu_[a-z_0-9]+)\s*\(", text)))


def _ptr(t) -> int | None:
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        return t.data_ptr()
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    raise TypeError(type(t))


def _stream_ptr(stream, device) -> int:
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return stream.cuda_stream if isinstance(stream, torch.cuda.Stream) else int(stream)


def status_string(status: int) -> str:
    return load_library().mglu_status_string(status).decode()


def _check(status: int, handle=None, what: str = ""):
    if status != MGLU_OK:
        lib = load_library()
        detail = lib.mglu_last_error(handle).decode() if handle else ""
        raise MgluError(status, f"{what}: {status_string(status)} {detail}".strip())


# ------------------------------------------------------------------ C-named entry points
def mglu_create(d: int, h: int, n_m: int, act: int, dtype: int, device: int) -> int:
    lib = load_library()
    hd = ctypes.c_void_p()
    _check(lib.mglu_create(ctypes.byref(hd), d, h, n_m, act, dtype, device), None, "mglu_create")
    return hd.value


def mglu_destroy(handle: int) -> None:
    _check(load_library().mglu_destroy(handle), None, "mglu_destroy")


def mglu_set_path(handle: int, path: int) -> None:
    _check(load_library().mglu_set_path(handle, path), handle, "mglu_set_path")


VARIANT = {"standard": 0, "no_gate_mask": 1, "no_value_mask": 2, "no_masks": 3}


def mglu_set_variant(handle: int, variant: int) -> None:
    _check(load_library().mglu_set_variant(handle, variant), handle, "mglu_set_variant")


def mglu_forward(handle, x, B, Wt, packed, out, stream=None) -> None:
    _check(load_library().mglu_forward(handle, _ptr(x), B, _ptr(Wt), _ptr(packed), _ptr(out),
                                       _stream_ptr(stream, x.device)), handle, "mglu_forward")


def mglu_forward_partials(handle, x, B, Wt, packed, z, stream=None) -> None:
    _check(load_library().mglu_forward_partials(handle, _ptr(x), B, _ptr(Wt), _ptr(packed), _ptr(z),
                                                _stream_ptr(stream, Wt.device)),
           handle, "mglu_forward_partials")


def mglu_forward_host(handle, x_host, B, Wt, packed, out_host, stream=None) -> None:
    _check(load_library().mglu_forward_host(handle, _ptr(x_host), B, _ptr(Wt), _ptr(packed),
                                            _ptr(out_host), _stream_ptr(stream, Wt.device)),
           handle, "mglu_forward_host")


def mglu_router_topk(handle, x, B, Wr, K, G, stream=None) -> None:
    _check(load_library().mglu_router_topk(handle, _ptr(x), B, _ptr(Wr), K, _ptr(G),
                                           _stream_ptr(stream, x.device)), handle, "mglu_router_topk")


def mglu_forward_routed(handle, x, B, Wt, packed, G, K, out, stream=None) -> None:
    _check(load_library().mglu_forward_routed(handle, _ptr(x), B, _ptr(Wt), _ptr(packed), _ptr(G), K, _ptr(out),
                                              _stream_ptr(stream, x.device)), handle, "mglu_forward_routed")


def mglu_packed_mask_bytes(d: int, h: int, n_m: int) -> int:
    return int(load_library().mglu_packed_mask_bytes(d, h, n_m))


def mglu_pack_masks_host(bits: np.ndarray) -> np.ndarray:
    bits = np.ascontiguousarray(bits, dtype=np.uint8)
    n_m, h, d = bits.shape
    out = np.empty(mglu_packed_mask_bytes(d, h, n_m), dtype=np.uint8)
    _check(load_library().mglu_pack_masks_host(_ptr(bits), n_m, h, d, _ptr(out)), None, "pack_masks_host")
    return out


def mglu_pack_logits_host(logits: np.ndarray) -> np.ndarray:
    logits = np.ascontiguousarray(logits, dtype=np.float32)
    n_m, h, d = logits.shape
    out = np.empty(mglu_packed_mask_bytes(d, h, n_m), dtype=np.uint8)
    _check(load_library().mglu_pack_logits_host(_ptr(logits), n_m, h, d, _ptr(out)), None, "pack_logits_host")
    return out


def mglu_unpack_masks_host(packed: np.ndarray, n_m: int, h: int, d: int) -> np.ndarray:
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    out = np.empty((n_m, h, d), dtype=np.uint8)
    _check(load_library().mglu_unpack_masks_host(_ptr(packed), n_m, h, d, _ptr(out)), None, "unpack_masks_host")
    return out


def mglu_code_stream_bytes(d: int, h: int, w: int) -> int:
    return int(load_library().mglu_code_stream_bytes(d, h, w))


def mglu_codes_to_bits_host(codes: np.ndarray, w: int, n_m: int, h: int, d: int) -> np.ndarray:
    """Per-element code stream (w-bit fields, mask i = bit i-1) -> 0/1 masks [n_m][h][d]."""
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    if codes.size != mglu_code_stream_bytes(d, h, w):
        raise MgluError(MGLU_ERR_INVALID_ARG, "code stream size mismatch")
    out = np.empty((n_m, h, d), dtype=np.uint8)
    _check(load_library().mglu_codes_to_bits_host(_ptr(codes), w, n_m, h, d, _ptr(out)), None, "codes_to_bits_host")
    return out


def mglu_pack_codes_host(codes: np.ndarray, w: int, n_m: int, h: int, d: int) -> np.ndarray:
    """Per-element code stream -> this library's packed layout (d % 32 == 0)."""
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    if codes.size != mglu_code_stream_bytes(d, h, w):
        raise MgluError(MGLU_ERR_INVALID_ARG, "code stream size mismatch")
    out = np.empty(mglu_packed_mask_bytes(d, h, n_m), dtype=np.uint8)
    _check(load_library().mglu_pack_codes_host(_ptr(codes), w, n_m, h, d, _ptr(out)), None, "pack_codes_host")
    return out


def mglu_unpack_codes_host(packed: np.ndarray, n_m: int, h: int, d: int, w: int) -> np.ndarray:
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    out = np.empty(mglu_code_stream_bytes(d, h, w), dtype=np.uint8)
    _check(load_library().mglu_unpack_codes_host(_ptr(packed), n_m, h, d, w, _ptr(out)), None, "unpack_codes_host")
    return out


def ffn_forward_fused(up: "Mglu", down: "Mglu", x: torch.Tensor, Wt: torch.Tensor, packed: torch.Tensor,
                      Wo: torch.Tensor, y_mid: torch.Tensor | None = None, out: torch.Tensor | None = None,
                      stream=None) -> torch.Tensor:
    """Row f1 fused: out = MGLU(x) Wo^T in one launch (mglu_ffn_forward).  `up` is the MGLU handle
    (d, h, n_m), `down` a dense handle (h, d_out, 0); y_mid [B][h] receives MGLU(x) (bf16)."""
    up._check_inputs(x, Wt, packed)
    B = x.shape[0]
    if Wo.dtype != torch.bfloat16 or tuple(Wo.shape) != (down.h, up.h) or not Wo.is_contiguous() or Wo.device != x.device:
        raise MgluError(MGLU_ERR_INVALID_ARG, "Wo must be a contiguous bf16 [d_out][h] tensor on x's device")
    if y_mid is None:
        y_mid = torch.empty((B, up.h), dtype=torch.bfloat16, device=x.device)
    if out is None:
        out = torch.empty((B, down.h), dtype=torch.bfloat16, device=x.device)
    for t, shape in ((y_mid, (B, up.h)), (out, (B, down.h))):
        if t.dtype != torch.bfloat16 or tuple(t.shape) != shape or not t.is_contiguous() or t.device != x.device:
            raise MgluError(MGLU_ERR_INVALID_ARG, f"y_mid / out must be contiguous bf16 {shape} tensors on x's device")
    _check(load_library().mglu_ffn_forward(up.handle, down.handle, _ptr(x), B, _ptr(Wt), _ptr(packed), _ptr(Wo),
                                           _ptr(y_mid), _ptr(out), _stream_ptr(stream, x.device)), up.handle,
           "mglu_ffn_forward")
    return out


def mglu_pack_planes_host(packed: np.ndarray, n_m: int, h: int, d: int) -> np.ndarray:
    """Interleaved packed codes -> the plane-major layout (include/mglu.h, row f2)."""
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    if packed.size != mglu_packed_mask_bytes(d, h, n_m):
        raise MgluError(MGLU_ERR_INVALID_ARG, "packed codes size mismatch")
    out = np.empty_like(packed)
    _check(load_library().mglu_pack_planes_host(_ptr(packed), n_m, h, d, _ptr(out)), None, "pack_planes_host")
    return out


def mglu_pack_planes_device(packed: torch.Tensor, n_m: int, h: int, d: int, stream=None) -> torch.Tensor:
    assert packed.is_cuda and packed.dtype == torch.uint8 and packed.is_contiguous()
    if packed.numel() != mglu_packed_mask_bytes(d, h, n_m):
        raise MgluError(MGLU_ERR_INVALID_ARG, "packed codes size mismatch")
    out = torch.empty_like(packed)
    _check(load_library().mglu_pack_planes_device(_ptr(packed), n_m, h, d, _ptr(out),
                                                  _stream_ptr(stream, packed.device)), None, "pack_planes_device")
    return out


def mglu_pack_masks_device(bits: torch.Tensor, stream=None) -> torch.Tensor:
    assert bits.is_cuda and bits.dtype == torch.uint8 and bits.is_contiguous()
    n_m, h, d = bits.shape
    out = torch.empty(mglu_packed_mask_bytes(d, h, n_m), dtype=torch.uint8, device=bits.device)
    _check(load_library().mglu_pack_masks_device(_ptr(bits), n_m, h, d, _ptr(out),
                                                 _stream_ptr(stream, bits.device)), None, "pack_masks_device")
    return out


def mglu_pack_logits_device(logits: torch.Tensor, stream=None) -> torch.Tensor:
    assert logits.is_cuda and logits.dtype == torch.float32 and logits.is_contiguous()
    n_m, h, d = logits.shape
    out = torch.empty(mglu_packed_mask_bytes(d, h, n_m), dtype=torch.uint8, device=logits.device)
    _check(load_library().mglu_pack_logits_device(_ptr(logits), n_m, h, d, _ptr(out),
                                                  _stream_ptr(stream, logits.device)), None, "pack_logits_device")
    return out


def mglu_unpack_masks_device(packed: torch.Tensor, n_m: int, h: int, d: int, stream=None) -> torch.Tensor:
    assert packed.is_cuda and packed.dtype == torch.uint8
    out = torch.empty((n_m, h, d), dtype=torch.uint8, device=packed.device)
    _check(load_library().mglu_unpack_masks_device(_ptr(packed), n_m, h, d, _ptr(out),
                                                   _stream_ptr(stream, packed.device)), None, "unpack_masks_device")
    return out


# ------------------------------------------------------------------ convenience wrapper
class Mglu:
    """One MGLU up-projection layer configuration (d, h, n_m, activation, dtype) on a device.
    Weights and packed codes are passed per call (borrowed, as in the C ABI)."""

    def __init__(self, d: int, h: int, n_m: int, act: str = "swish", dtype: str = "bf16",
                 device: int = 0, path: str = "auto"):
        self.d, self.h, self.n_m, self.act, self.dtype, self.device = d, h, n_m, act, dtype, device
        self.handle = mglu_create(d, h, n_m, ACT[act], DTYPE[dtype], device)
        if path != "auto":
            self.set_path(path)

    def set_path(self, path: str) -> None:
        mglu_set_path(self.handle, PATH[path])

    def backward(self, x: torch.Tensor, Wt: torch.Tensor, packed: torch.Tensor, dy: torch.Tensor,
                 want=("dx", "dW", "dlogits"), stream=None):
        """Gradients of Eq. 3 under Alg. 2's STE (row f4): returns (dx [B][d], dW [h][d],
        dlogits [n_m][h][d]) fp32, None for the ones not in `want`."""
        self._check_inputs(x, Wt, packed)
        B = x.shape[0]
        if dy.dtype != torch.float32 or tuple(dy.shape) != (B, self.h) or not dy.is_contiguous() or dy.device != x.device:
            raise MgluError(MGLU_ERR_INVALID_ARG, "dy must be a contiguous fp32 [B][h] tensor on x's device")
        f32 = dict(dtype=torch.float32, device=x.device)
        dx = torch.empty((B, self.d), **f32) if "dx" in want else None
        dW = torch.empty((self.h, self.d), **f32) if "dW" in want else None
        dl = torch.empty((self.n_m, self.h, self.d), **f32) if "dlogits" in want else None
        _check(load_library().mglu_backward(self.handle, _ptr(x), B, _ptr(Wt), _ptr(packed), _ptr(dy), _ptr(dx), _ptr(dW),
                                            _ptr(dl), _stream_ptr(stream, x.device)), self.handle, "mglu_backward")
        return dx, dW, dl

    def reserve(self, max_B: int, stream=None) -> None:
        """Pre-allocate the batched-decode workspace for batches up to max_B (before graph capture)."""
        _check(load_library().mglu_reserve(self.handle, int(max_B), _stream_ptr(stream, torch.device("cuda", self.device))),
               self.handle, "mglu_reserve")

    def set_debug(self, flags: int) -> None:
        """Test hooks (include/mglu.h): 1 = flip mask 1's bit of element (0, 0) during each call."""
        _check(load_library().mglu_set_debug(self.handle, int(flags)), self.handle, "mglu_set_debug")

    def set_variant(self, variant: str) -> None:
        """Partial-mask ablation variant: standard, no_gate_mask, no_value_mask, no_masks."""
        mglu_set_variant(self.handle, VARIANT[variant])

    def _check_inputs(self, x, Wt, packed):
        td = TORCH_DTYPE[self.dtype]
        if x.dtype != td or Wt.dtype != td:
            raise MgluError(MGLU_ERR_INVALID_ARG, f"x/Wt must be {td}")
        if x.dim() != 2 or tuple(Wt.shape) != (self.h, self.d) or x.shape[1] != self.d:
            raise MgluError(MGLU_ERR_INVALID_ARG, "shape mismatch: x must be [B][d] (flatten leading dims), Wt [h][d]")
        if x.device != Wt.device:
            raise MgluError(MGLU_ERR_INVALID_ARG, "x and Wt must be on the same device")
        if self.n_m == 0 and packed is None:              # dense projection (FFN W_o): no codes
            packed = torch.empty(0, dtype=torch.uint8, device=Wt.device)
        if packed.dtype != torch.uint8 or packed.numel() != mglu_packed_mask_bytes(self.d, self.h, self.n_m):
            raise MgluError(MGLU_ERR_INVALID_ARG, "packed codes size mismatch")
        if not (x.is_contiguous() and Wt.is_contiguous() and packed.is_contiguous()):
            raise MgluError(MGLU_ERR_INVALID_ARG, "tensors must be contiguous")

    def _check_out(self, out, B, x):
        if out.dtype != TORCH_DTYPE[self.dtype] or tuple(out.shape) != (B, self.h) or not out.is_contiguous() \
                or out.device != x.device:
            raise MgluError(MGLU_ERR_INVALID_ARG, f"out must be a contiguous {TORCH_DTYPE[self.dtype]} [B][h] tensor on x's device")

    def forward(self, x: torch.Tensor, Wt: torch.Tensor, packed: torch.Tensor,
                out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """y [..., h] = MGLU(x [..., d]): leading dims of x are flattened into the token count."""
        lead = tuple(x.shape[:-1])
        x2 = x.reshape(-1, x.shape[-1]) if x.dim() != 2 else x
        self._check_inputs(x2, Wt, packed)
        B = x2.shape[0]
        if out is None:
            out = torch.empty((B, self.h), dtype=TORCH_DTYPE[self.dtype], device=x.device)
        else:
            self._check_out(out.reshape(B, self.h) if out.dim() != 2 else out, B, x2)
        mglu_forward(self.handle, x2, B, Wt, packed, out, stream)
        return out.reshape(*lead, self.h) if x.dim() != 2 else out

    __call__ = forward

    def bind(self, x, Wt, packed, out, stream=None):
        """Validate once and return a zero-argument callable that enqueues mglu_forward with
        the pointers pre-marshalled (the per-call host cost is one ctypes call)."""
        self._check_inputs(x, Wt, packed)
        B = x.shape[0]
        self._check_out(out, B, x)
        lib = load_library()
        args = (self.handle, x.data_ptr(), B, Wt.data_ptr(), packed.data_ptr() if packed is not None else None, out.data_ptr(),
                _stream_ptr(stream, x.device))
        fwd = lib.mglu_forward

        def call():
            st = fwd(*args)
            if st != MGLU_OK:
                _check(st, self.handle, "mglu_forward")
        return call

    def router_topk(self, x: torch.Tensor, Wr: torch.Tensor, K: int, stream=None) -> torch.Tensor:
        """G = Softmax(TopK(x W_r)) [B][n_m] fp32 (Appendix B); Wr is [n_m][d] bf16."""
        if Wr.dtype != torch.bfloat16 or tuple(Wr.shape) != (self.n_m, self.d) or not Wr.is_contiguous():
            raise MgluError(MGLU_ERR_INVALID_ARG, "Wr must be a contiguous bf16 [n_m][d] tensor")
        if x.dtype != torch.bfloat16 or x.dim() != 2 or x.shape[1] != self.d or x.device != Wr.device:
            raise MgluError(MGLU_ERR_INVALID_ARG, "x must be a bf16 [B][d] tensor on Wr's device")
        B = x.shape[0]
        G = torch.empty((B, self.n_m), dtype=torch.float32, device=x.device)
        mglu_router_topk(self.handle, x.contiguous(), B, Wr, K, G, stream)
        return G

    def forward_routed(self, x: torch.Tensor, Wt: torch.Tensor, packed: torch.Tensor, G: torch.Tensor,
                       K: int = 0, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """y = sum_i G[:, i] g(s_i) (t - s_i) (Top-K routed MGLU)."""
        self._check_inputs(x, Wt, packed)
        B = x.shape[0]
        if G.dtype != torch.float32 or tuple(G.shape) != (B, self.n_m) or not G.is_contiguous():
            raise MgluError(MGLU_ERR_INVALID_ARG, "G must be a contiguous fp32 [B][n_m] tensor")
        if out is None:
            out = torch.empty((B, self.h), dtype=TORCH_DTYPE[self.dtype], device=x.device)
        else:
            self._check_out(out, B, x)
        mglu_forward_routed(self.handle, x, B, Wt, packed, G, K, out, stream)
        return out

    def forward_routed_planes(self, x: torch.Tensor, Wt: torch.Tensor, planes: torch.Tensor, G: torch.Tensor,
                              K: int, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """forward_routed on plane-major codes (mglu_pack_planes_*): reads W + the selected planes."""
        self._check_inputs(x, Wt, planes)
        B = x.shape[0]
        if G.dtype != torch.float32 or tuple(G.shape) != (B, self.n_m) or not G.is_contiguous():
            raise MgluError(MGLU_ERR_INVALID_ARG, "G must be a contiguous fp32 [B][n_m] tensor")
        if out is None:
            out = torch.empty((B, self.h), dtype=TORCH_DTYPE[self.dtype], device=x.device)
        else:
            self._check_out(out, B, x)
        _check(load_library().mglu_forward_routed_planes(self.handle, _ptr(x), B, _ptr(Wt), _ptr(planes), _ptr(G), K,
                                                         _ptr(out), _stream_ptr(stream, x.device)),
               self.handle, "mglu_forward_routed_planes")
        return out

    def forward_partials(self, x, Wt, packed, stream=None) -> torch.Tensor:
        self._check_inputs(x, Wt, packed)
        B = x.shape[0]
        z = torch.empty((B, 2 * self.n_m, self.h), dtype=torch.float32, device=x.device)
        mglu_forward_partials(self.handle, x, B, Wt, packed, z, stream)
        return z

    def forward_host(self, x_host: torch.Tensor, Wt: torch.Tensor, packed: torch.Tensor,
                     out_host: torch.Tensor, stream=None) -> torch.Tensor:
        td = TORCH_DTYPE[self.dtype]
        if x_host.is_cuda or out_host.is_cuda:
            raise MgluError(MGLU_ERR_INVALID_ARG, "forward_host takes host tensors (pinned for async copies)")
        if x_host.dtype != td or x_host.dim() != 2 or x_host.shape[1] != self.d or not x_host.is_contiguous():
            raise MgluError(MGLU_ERR_INVALID_ARG, f"x_host must be a contiguous {td} [B][d] host tensor")
        B = x_host.shape[0]
        if out_host.dtype != td or tuple(out_host.shape) != (B, self.h) or not out_host.is_contiguous():
            raise MgluError(MGLU_ERR_INVALID_ARG, f"out_host must be a contiguous {td} [B][h] host tensor")
        if Wt.dtype != td or tuple(Wt.shape) != (self.h, self.d) or not Wt.is_cuda:
            raise MgluError(MGLU_ERR_INVALID_ARG, "Wt must be a device [h][d] tensor")
        if self.n_m and (packed is None or packed.numel() != mglu_packed_mask_bytes(self.d, self.h, self.n_m)):
            raise MgluError(MGLU_ERR_INVALID_ARG, "packed codes size mismatch")
        mglu_forward_host(self.handle, x_host, B, Wt, packed, out_host, stream)
        return out_host

    def last_path(self) -> str:
        v = load_library().mglu_last_path(self.handle)
        return {k: p for p, k in PATH.items()}.get(v, str(v))

    def last_launch_count(self) -> int:
        return int(load_library().mglu_last_launch_count(self.handle))

    def close(self) -> None:
        if getattr(self, "handle", None):
            mglu_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
