"""The bench's algorithmic units: bytes and FLOPs per call for the BASELINE configs,
against the figures derived in SURVEY.md from Table 1's (16 + n_m) bits per element."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_decode_bytes(bench):
    # config 3, B = 1: W 117.44 MB + codes 29.36 MB + x + y = 146.84 MB
    assert bench.algorithmic_bytes(4096, 14336, 4, 1) == 4096 * 14336 * 2 + 4096 * 14336 * 4 // 8 + 4096 * 2 + 14336 * 2
    assert round(bench.algorithmic_bytes(4096, 14336, 4, 1) / 1e6, 2) == 146.84
    # config 2: 112.75 MB
    assert round(bench.algorithmic_bytes(4096, 11008, 4, 1) / 1e6, 2) == 112.75
    # config 5 per GPU at G = 8 (3584 columns): 62.4 / 66.1 / 73.4 / 88.1 MB for n_m = 1 / 2 / 4 / 8
    for n_m, mb in ((1, 62.4), (2, 66.1), (4, 73.4), (8, 88.1)):
        assert round(bench.algorithmic_bytes(8192, 3584, n_m, 1) / 1e6, 1) == mb
    # the dense W_o pass of the FFN block (n_m = 0): W + x + y only
    assert bench.algorithmic_bytes(14336, 4096, 0, 1) == 14336 * 4096 * 2 + 14336 * 2 + 4096 * 2


def test_prefill_flops(bench):
    # config 4: 2 B d h (n_m + 1) = 9.62 TFLOP; config 5 at B = 2048 per GPU of 8
    assert round(bench.algorithmic_flops(8192, 28672, 4, 4096) / 1e12, 2) == 9.62
    for n_m, tf in ((1, 0.24), (2, 0.36), (4, 0.60), (8, 1.08)):
        assert round(bench.algorithmic_flops(8192, 3584, n_m, 2048) / 1e12, 2) == tf


def test_metric_regimes(bench):
    assert bench.work(4096, 14336, 4, 1)[2] == "GB/s"
    assert bench.work(4096, 14336, 4, 64)[2] == "TFLOP/s"
    assert bench.DEFAULT_WORKLOAD == "decode_b1" and bench.WORKLOADS["decode_b1"][:4] == (4096, 14336, 4, 1)
