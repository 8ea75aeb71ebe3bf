"""Pins of the partial-mask ablation variants, row f3."""
import numpy as np

from oracle import ACT_IDENTITY, ACT_SIGMOID, mglu_partials_np, mglu_variant_from_streams


def _streams(x, Wt, bits):
    t, gate, value = mglu_partials_np(x, Wt, bits)
    return t, gate, value


def test_worked_example_each_variant():
    # SPEC 2x2 example: t = [3, 7], gate = [1, 4], value = [2, 3].  By the definitions
    # (identity g): NG = t * value = [6, 21]; NV = gate * t = [3, 28]; NM = t^2 = [9, 49]
    x = np.array([[1.0, 1.0]])
    Wt = np.array([[1.0, 2.0], [3.0, 4.0]])
    bits = np.array([[[1, 0], [0, 1]]], dtype=np.uint8)
    t, gate, value = _streams(x, Wt, bits)
    want = {0: [2.0, 12.0], 1: [6.0, 21.0], 2: [3.0, 28.0], 3: [9.0, 49.0]}
    for v, w in want.items():
        np.testing.assert_array_equal(mglu_variant_from_streams(t, gate, value, ACT_IDENTITY, v), [w])


def test_special_masks():
    rng = np.random.default_rng(2)
    B, d, h, n_m = 2, 32, 6, 3
    x = rng.standard_normal((B, d))
    Wt = rng.standard_normal((h, d))
    ones = np.ones((n_m, h, d), dtype=np.uint8)
    zeros = np.zeros((n_m, h, d), dtype=np.uint8)
    xw = x @ Wt.T
    sig = 1 / (1 + np.exp(-xw))
    # NG with all-ones masks: value = 0 -> 0
    np.testing.assert_array_equal(mglu_variant_from_streams(*_streams(x, Wt, ones), ACT_SIGMOID, 1), 0.0)
    # NV with all-zero masks: gate = 0 -> n_m * g(0) * xW = (n_m / 2) xW for sigmoid
    np.testing.assert_allclose(mglu_variant_from_streams(*_streams(x, Wt, zeros), ACT_SIGMOID, 2), n_m / 2 * xw,
                               rtol=1e-13)
    # NM ignores the masks entirely: n_m g(xW) xW, the same for any masks
    rnd = rng.integers(0, 2, (n_m, h, d)).astype(np.uint8)
    for b in (ones, zeros, rnd):
        np.testing.assert_allclose(mglu_variant_from_streams(*_streams(x, Wt, b), ACT_SIGMOID, 3), n_m * sig * xw,
                                   rtol=1e-13)
    # NG with all-zero masks: value = xW -> n_m g(xW) xW (equals NM)
    np.testing.assert_allclose(mglu_variant_from_streams(*_streams(x, Wt, zeros), ACT_SIGMOID, 1), n_m * sig * xw,
                               rtol=1e-12)
