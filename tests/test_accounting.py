"""Accounting pins (CPU): Table 1, the 47 % / 37.5 % claims, footnote P:289 and Table 10."""
import json
import os

import pytest

from oracle import accounting as acc


@pytest.fixture(scope="module")
def g(golden_dir):
    with open(os.path.join(golden_dir, "accounting.json")) as f:
        return json.load(f)


def test_table1_rows(g):
    h, d = 2048, 8192
    assert acc.memory_load_bits("lu", h, d) == g["table1"]["lu"] * h * d
    assert acc.memory_load_bits("glu", h, d) == g["table1"]["glu"] * h * d
    for n_m in (1, 2, 4, 8, 16):
        assert acc.memory_load_bits("mglu", h, d, n_m) == (g["table1"]["mglu_plus"] + n_m) * h * d


def test_reductions(g):
    assert acc.reduction_vs_glu(2048, 8192, 1) == g["reduction_nm1"]
    assert acc.reduction_vs_glu(4096, 14336, 4) == g["reduction_nm4"]       # P:33 "37.5%"
    assert acc.reduction_vs_glu(768, 3072, g["break_even_nm"]) == 0.0       # S:447 break-even
    vals = [acc.memory_load_bits("mglu", 8, 8, n) for n in range(1, 17)]
    assert vals == sorted(vals) and len(set(vals)) == 16


def test_footnote(g):
    f = g["footnote_llama1b"]
    assert acc.ffn_weight_bytes_fp16("glu", f["h"], f["d"]) == f["glu_ffn_MiB"] * 2**20
    assert acc.ffn_weight_bytes_fp16("mglu", f["h"], f["d"]) == f["mglu_ffn_MiB"] * 2**20
    assert acc.packed_mask_bytes(f["h"], f["d"], 1) == f["mask_MiB_nm1"] * 2**20


def test_table10(g):
    shapes = {"small": (12, 768, 3072), "large": (16, 2048, 8192)}
    for row in g["table10"]["rows"]:
        L, h, d = shapes[row["scale"]]
        masks = acc.model_mask_params(L, h, d, row["n_m"])
        assert abs(masks - row["masks_printed"]) / row["masks_printed"] < 0.005
        # #Weights is printed to 3 significant digits (+-0.5M -> +-0.95 MiB), so allow 1 MiB
        assert abs(acc.storage_mib(row["weights"], masks) - row["size_MiB"]) <= 1.0


def test_packed_bytes_and_decode_bytes():
    # BASELINE config 3 at B=1: W 117.44 MB + codes 29.36 MB + x + y = 146.84 MB
    assert acc.packed_mask_bytes(14336, 4096, 4) == 14336 * 4096 // 2
    b = acc.decode_bytes(1, 14336, 4096, 4)
    assert b == 14336 * 4096 * 2 + 14336 * 4096 // 2 + 4096 * 2 + 14336 * 2
    assert abs(b / 1e6 - 146.84) < 0.01
    # FLOPs (R12): 2 B h d (n_m + 1); prefill config 4 = 9.62 TFLOP
    assert abs(acc.inference_flops_up_proj(4096, 28672, 8192, 4) / 1e12 - 9.62) < 0.005
