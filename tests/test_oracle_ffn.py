"""Pins of the FFN oracle (P:100 output projection) and of its row-parallel split."""
import numpy as np

from oracle import ACT_IDENTITY, ACT_SWISH, dense_np, ffn_forward_np, mglu_forward_np


def test_identity_down_projection_is_mglu():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((2, 32))
    Wt = rng.standard_normal((32, 32))
    bits = rng.integers(0, 2, (2, 32, 32)).astype(np.uint8)
    np.testing.assert_allclose(ffn_forward_np(x, Wt, bits, np.eye(32), ACT_SWISH),
                               mglu_forward_np(x, Wt, bits, ACT_SWISH), rtol=1e-14)


def test_worked_example_down_projection():
    # SPEC 2x2 example: y_identity = [2, 12]; with Wo = [[1, 1], [1, -1]] the FFN gives
    # [2 + 12, 2 - 12] = [14, -10] exactly
    x = np.array([[1.0, 1.0]])
    Wt = np.array([[1.0, 2.0], [3.0, 4.0]])
    bits = np.array([[[1, 0], [0, 1]]], dtype=np.uint8)
    out = ffn_forward_np(x, Wt, bits, np.array([[1.0, 1.0], [1.0, -1.0]]), ACT_IDENTITY)
    np.testing.assert_array_equal(out, [[14.0, -10.0]])


def test_row_parallel_split_sums_to_full():
    """Column shard of the up-projection + row (reduction) shard of W_o: the per-rank partial
    outputs sum to the full FFN (the all-reduce of SURVEY 8(e)/(f1)), for uneven shards too."""
    rng = np.random.default_rng(1)
    B, d, h, n_m = 3, 64, 37, 2
    x = rng.standard_normal((B, d))
    Wt = rng.standard_normal((h, d))
    Wo = rng.standard_normal((d, h))
    bits = rng.integers(0, 2, (n_m, h, d)).astype(np.uint8)
    full = ffn_forward_np(x, Wt, bits, Wo, ACT_SWISH)
    for G in (2, 3, 5):
        parts = []
        for r in range(G):
            lo, hi = r * h // G, (r + 1) * h // G
            y_r = mglu_forward_np(x, Wt[lo:hi], bits[:, lo:hi], ACT_SWISH)
            parts.append(dense_np(y_r, Wo[:, lo:hi]))
        np.testing.assert_allclose(np.sum(parts, axis=0), full, rtol=1e-12, atol=1e-12)
