"""Closed-form accounting of Table 1 and Sec. 4.1 -- TEST INFRASTRUCTURE ONLY.

Letters follow the paper's Table 1 caption: ``h`` hidden, ``d`` intermediate.  Only
products ``h*d`` appear, so the BASELINE naming swap (R2) does not matter here.
"""
from __future__ import annotations


def memory_load_bits(kind: str, h: int, d: int, n_m: int | None = None) -> int:
    """Table 1, memory load per token of the intermediate (up) projection in FP16
    inference: LU 16hd, GLU 32hd, MGLU (16+n_m)hd."""
    if kind == "lu":
        return 16 * h * d
    if kind == "glu":
        return 32 * h * d
    if kind == "mglu":
        if n_m is None:
            raise ValueError("mglu needs n_m")
        return (16 + n_m) * h * d
    raise ValueError(kind)


def reduction_vs_glu(h: int, d: int, n_m: int) -> float:
    """(16*2hd - (16hd + n_m hd)) / (16*2hd); n_m = 1 gives 0.46875."""
    glu = memory_load_bits("glu", h, d)
    return (glu - memory_load_bits("mglu", h, d, n_m)) / glu


def packed_mask_bytes(h: int, d: int, n_m: int) -> int:
    """Dense code layout (R3): n_m bits per weight element, h*d*n_m/8 bytes."""
    bits = h * d * n_m
    return (bits + 7) // 8


def ffn_weight_bytes_fp16(kind: str, h: int, d: int) -> int:
    """Footnote P:289: FFN weights per layer in FP16.  SwiGLU: W_g, W_v, W_o = 3hd;
    MGLU: W, W_o = 2hd."""
    mats = {"glu": 3, "mglu": 2, "lu": 2}[kind]
    return 2 * mats * h * d


def inference_flops_up_proj(B: int, h: int, d: int, n_m: int) -> int:
    """Reading R12: algorithmic FLOPs of the fused up-projection = 2*B*h*d*(n_m+1): one unmasked
    contraction t plus n_m gated contractions s_i (the value streams are t - s_i).  The
    paper's "2(1+n_m)hd multiply-add" is the same count per token."""
    return 2 * B * h * d * (n_m + 1)


def decode_bytes(B: int, h: int, d: int, n_m: int, x_bytes: int = 2, y_bytes: int = 2,
                 w_bytes: int = 2) -> int:
    """Algorithmic HBM bytes of one forward call: W and the packed codes once,
    x read, y written."""
    return h * d * w_bytes + packed_mask_bytes(h, d, n_m) + B * d * x_bytes + B * h * y_bytes


def model_mask_params(layers: int, h: int, d: int, n_m: int) -> int:
    """Table 10 #Masks column: one h x d binary mask per mixture per FFN layer."""
    return layers * h * d * n_m


def storage_mib(n_weights: float, n_mask_bits: float) -> float:
    """Table 10 "Size (MB)": FP16 weights + 1-bit masks, in MiB."""
    return (n_weights * 2 + n_mask_bits / 8) / 2**20
