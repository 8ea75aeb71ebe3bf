"""Pins of the training-path oracle (row f4; Alg. 2; SPEC autograd
S:293-362): the hand-worked 2x2 example, central finite differences of the hard forward (d_x, d_W
with the masks fixed) and of the relaxed surrogate at soft = hard (d_logits, the STE pass-through),
zero upstream, linearity in the upstream gradient, and the identity-g complementarity identity."""
import json
import os

import numpy as np
import pytest

from oracle import (ACT_GELU, ACT_IDENTITY, ACT_RELU, ACT_SIGMOID, ACT_SWISH, act_grad_np, act_np,
                    mglu_backward_np, mglu_forward_np, relaxed_forward_np)

HERE = os.path.dirname(os.path.abspath(__file__))


def test_worked_example():
    g = json.load(open(os.path.join(HERE, "golden", "backward_worked.json")))
    dx, dW, dl = mglu_backward_np(np.array(g["x"], float), np.array(g["Wt"], float), np.array(g["bits"]),
                                  np.array(g["dy"], float), g["act"])
    np.testing.assert_array_equal(dx, g["dx"])
    np.testing.assert_array_equal(dW, g["dW"])
    np.testing.assert_array_equal(dl, g["dlogits"])


@pytest.mark.parametrize("act", [ACT_IDENTITY, ACT_SWISH, ACT_GELU, ACT_SIGMOID])
def test_act_grad_by_central_difference(act):
    z = np.linspace(-4, 4, 81)
    eps = 1e-6
    fd = (act_np(act, z + eps) - act_np(act, z - eps)) / (2 * eps)
    np.testing.assert_allclose(act_grad_np(act, z), fd, rtol=1e-7, atol=1e-8)


def _instance(seed, B, d, h, n_m):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((B, d)), rng.uniform(-1, 1, (h, d)), rng.integers(0, 2, (n_m, h, d)).astype(np.uint8),
            rng.standard_normal((B, h)))


@pytest.mark.parametrize("act,n_m", [(ACT_IDENTITY, 1), (ACT_SWISH, 4), (ACT_GELU, 2), (ACT_SIGMOID, 3)])
def test_dx_dW_match_finite_differences(act, n_m):
    """d_x and d_W are the exact gradients of the hard-mask forward."""
    x, Wt, bits, dy = _instance(10 + n_m, 3, 8, 5, n_m)
    dx, dW, _ = mglu_backward_np(x, Wt, bits, dy, act)
    L = lambda x_, W_: float(np.sum(dy * mglu_forward_np(x_, W_, bits, act)))   # noqa: E731
    eps = 1e-6
    for b in range(3):
        for k in range(8):
            e = np.zeros_like(x); e[b, k] = eps
            assert abs((L(x + e, Wt) - L(x - e, Wt)) / (2 * eps) - dx[b, k]) <= 1e-6 * max(1.0, abs(dx[b, k]))
    for j in range(5):
        for k in range(8):
            e = np.zeros_like(Wt); e[j, k] = eps
            assert abs((L(x, Wt + e) - L(x, Wt - e)) / (2 * eps) - dW[j, k]) <= 1e-6 * max(1.0, abs(dW[j, k]))


@pytest.mark.parametrize("act,n_m", [(ACT_IDENTITY, 1), (ACT_SWISH, 4), (ACT_GELU, 2)])
def test_dlogits_match_relaxed_surrogate(act, n_m):
    """d_logits = gradient of the relaxed forward at soft = hard (the STE pass-through)."""
    x, Wt, bits, dy = _instance(20 + n_m, 2, 6, 4, n_m)
    _, _, dl = mglu_backward_np(x, Wt, bits, dy, act)
    soft = bits.astype(np.float64)
    np.testing.assert_allclose(relaxed_forward_np(x, Wt, soft, act), mglu_forward_np(x, Wt, bits, act), rtol=0, atol=1e-12)
    eps = 1e-6
    for i in range(n_m):
        for j in range(4):
            for k in range(6):
                e = np.zeros_like(soft); e[i, j, k] = eps
                fd = (np.sum(dy * relaxed_forward_np(x, Wt, soft + e, act)) -
                      np.sum(dy * relaxed_forward_np(x, Wt, soft - e, act))) / (2 * eps)
                assert abs(fd - dl[i, j, k]) <= 1e-6 * max(1.0, abs(dl[i, j, k]))


def test_zero_upstream_and_linearity():
    x, Wt, bits, dy = _instance(3, 4, 16, 6, 2)
    for g in mglu_backward_np(x, Wt, bits, np.zeros_like(dy), ACT_SWISH):
        assert not np.any(g)
    g1 = mglu_backward_np(x, Wt, bits, dy, ACT_SWISH)
    g3 = mglu_backward_np(x, Wt, bits, -2.5 * dy, ACT_SWISH)
    for a, b in zip(g1, g3):
        np.testing.assert_allclose(b, -2.5 * a, rtol=1e-12, atol=1e-12)


def test_relu_subgradient_zero_at_zero():
    assert act_grad_np(ACT_RELU, np.array([0.0]))[0] == 0.0 and act_grad_np(ACT_RELU, np.array([1e-300]))[0] == 1.0


def test_identity_complementarity_identity():
    """Identity g, n_m = 1, all-zero masks: y = 0 * (xW) and the value-stream gradient alone is
    left: d_W = (dy * 0)^T x + ... i.e. only c = dy * s = 0 contributes -> d_W = 0, and with
    all-ones masks s = xW, v = 0: d_W = (dy v)^T x = 0 as well, while d_logits = W (.) (a - c)^T x
    with a = dy v = 0, c = dy s: d_logits = -W (.) ((dy * xW)^T x)."""
    x, Wt, _, dy = _instance(5, 3, 8, 4, 1)
    ones = np.ones((1, 4, 8), dtype=np.uint8)
    dx, dW, dl = mglu_backward_np(x, Wt, ones, dy, ACT_IDENTITY)
    assert not np.any(dx) and not np.any(dW)
    np.testing.assert_allclose(dl[0], -Wt * ((dy * (x @ Wt.T)).T @ x), rtol=1e-13, atol=1e-13)
