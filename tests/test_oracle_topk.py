"""Pins of the Top-K routed MGLU oracle (Appendix B)."""
import math

import numpy as np
import pytest

from fractions import Fraction

from oracle import (ACT_SWISH, ACT_SIGMOID, mglu_forward_np, mglu_partials_np, mglu_routed_from_partials,
                    router_logits, topk_gate)


def test_router_logits_hand_example_and_orientation():
    """l = x W_r with W_r stored [n_m][d] (reading R16): x = [1, 2, 3],
    W_r rows [1, 0, -1], [2, 2, 2] -> l = [1 - 3, 2 + 4 + 6] = [-2, 12].  The asymmetric
    B x d / n_m x d shapes make a transposed operand fail."""
    l = router_logits(np.array([[1.0, 2.0, 3.0]]), np.array([[1.0, 0.0, -1.0], [2.0, 2.0, 2.0]]))
    np.testing.assert_array_equal(l, [[-2.0, 12.0]])
    rng = np.random.default_rng(0)
    x, Wr = rng.standard_normal((2, 5)), rng.standard_normal((3, 5))
    assert router_logits(x, Wr).shape == (2, 3)
    for k in range(5):                                    # one-hot x at k picks column k of W_r
        e = np.zeros((1, 5)); e[0, k] = 1.0
        np.testing.assert_array_equal(router_logits(e, Wr)[0], Wr[:, k])


def test_router_logits_exact_rational():
    """Dyadic inputs: every product and partial sum is exact in binary64, so the oracle must equal
    the exact rational sum."""
    rng = np.random.default_rng(1)
    x = rng.integers(-64, 65, (3, 40)) / 16.0
    Wr = rng.integers(-64, 65, (4, 40)) / 32.0
    l = router_logits(x, Wr)
    for b in range(3):
        for i in range(4):
            exact = sum(Fraction(float(x[b, k])) * Fraction(float(Wr[i, k])) for k in range(40))
            assert Fraction(float(l[b, i])) == exact


def test_spec_worked_example_k2():
    # SPEC topk_gate example: l = [0.1, 0.5, 0.3, 0.2], K = 2 -> indices {1, 2}, weights
    # [e^0.5, e^0.3] / (e^0.5 + e^0.3) = [0.549834, 0.450166]
    G = topk_gate(np.array([0.1, 0.5, 0.3, 0.2]), 2)[0]
    a, b = math.exp(0.5), math.exp(0.3)
    np.testing.assert_allclose(G, [0.0, a / (a + b), b / (a + b), 0.0], rtol=0, atol=1e-15)
    np.testing.assert_allclose(G[1:3], [0.549834, 0.450166], atol=5e-7)


def test_k1_is_one_hot_argmax_and_ties_go_low():
    G = topk_gate(np.array([[0.3, -1.0, 2.0, 2.0], [5.0, 5.0, 5.0, 5.0]]), 1)
    np.testing.assert_array_equal(G, [[0, 0, 1.0, 0], [1.0, 0, 0, 0]])   # ties -> lowest index
    G2 = topk_gate(np.array([[1.0, 1.0, 1.0, 0.0]]), 2)
    np.testing.assert_array_equal(G2, [[0.5, 0.5, 0.0, 0.0]])


def test_k_equals_nm_is_full_softmax():
    l = np.array([[0.3, -1.2, 0.7, 2.0, 0.0, -0.4]])
    e = np.exp(l - l.max())
    np.testing.assert_allclose(topk_gate(l, 6), e / e.sum(), rtol=1e-15)
    with pytest.raises(ValueError):
        topk_gate(l, 0)
    with pytest.raises(ValueError):
        topk_gate(l, 7)


def test_uniform_logits_full_k_is_mean_of_terms():
    """K = n_m with equal logits: G = 1/n_m, so MGLU_TopK = (1/n_m) MGLU (Eq. 3)."""
    rng = np.random.default_rng(0)
    n_m, B, d, h = 4, 3, 32, 10
    x = rng.standard_normal((B, d))
    Wt = rng.standard_normal((h, d))
    bits = rng.integers(0, 2, (n_m, h, d)).astype(np.uint8)
    _, gate, value = mglu_partials_np(x, Wt, bits)
    G = topk_gate(np.zeros((B, n_m)), n_m)
    y = mglu_routed_from_partials(gate, value, G, ACT_SWISH)
    np.testing.assert_allclose(y, mglu_forward_np(x, Wt, bits, ACT_SWISH) / n_m, rtol=1e-12, atol=1e-12)


def test_k1_selects_one_term_exactly():
    """K = 1: y = g(x (M_s (.) W)) (.) x (Mbar_s (.) W) for the argmax s, each term by its own
    masked matrix (a dropped or swapped term fails)."""
    rng = np.random.default_rng(1)
    n_m, d, h = 8, 64, 5
    x = rng.standard_normal((1, d))
    Wt = rng.standard_normal((h, d))
    bits = rng.integers(0, 2, (n_m, h, d)).astype(np.uint8)
    l = np.array([[0.1, 0.2, 3.0, -1, 0, 0, 0.5, 2.9]])
    _, gate, value = mglu_partials_np(x, Wt, bits)
    y = mglu_routed_from_partials(gate, value, topk_gate(l, 1), ACT_SIGMOID)
    M = bits[2].astype(np.float64)
    want = (1 / (1 + np.exp(-(x @ (M * Wt).T)))) * (x @ ((1 - M) * Wt).T)
    np.testing.assert_allclose(y, want, rtol=1e-13)
