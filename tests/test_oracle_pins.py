"""Pins of the CPU oracle to things other than itself (CPU only, no GPU).

Each test pins both oracle implementations (numpy twin ``mglu_forward_np`` and the C loops
``COracle``) against: values printed in SPEC/PAPER worked examples (tests/golden/), closed forms,
exhaustive enumeration of codes, exact rational brute force, and special masks.  A plausible
mistake -- dropped term, wrong sign, swapped gate/value, off-by-one bit index, transposed
operand, a 1/n_m factor -- fails at least one of these (see the comment on each test).
"""
import itertools
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import (ACT_GELU, ACT_IDENTITY, ACT_NAMES, ACT_RELU, ACT_SIGMOID, ACT_SWISH, act_np,
                    decode_bf16, mglu_forward_np, mglu_partials_np, pack_np, unpack_np)
from synth import make_inputs, make_logits

pytestmark = pytest.mark.cpu


def _load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


def _pad32(x, Wt, bits):
    """Zero-pad the reduction dim to a multiple of 32 (the packed layout's group, reading R3):
    zero columns of W and x add exact zeros to every sum, so Eq. 3 is unchanged."""
    d = Wt.shape[1]
    dp = -(-d // 32) * 32
    if dp == d:
        return x, Wt, bits
    pad = dp - d
    return (np.pad(x, ((0, 0), (0, pad))), np.pad(Wt, ((0, 0), (0, pad))),
            np.pad(bits, ((0, 0), (0, 0), (0, pad))))


def _forward_both(c_oracle, x, Wt, bits, act):
    """y from the numpy twin (on the unpadded inputs) and from the C oracle (which sees only the
    packed layout, on zero-padded inputs when d % 32 != 0)."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    Wt = np.asarray(Wt, dtype=np.float64)
    bits = np.asarray(bits, dtype=np.uint8)
    y_np = mglu_forward_np(x, Wt, bits, act)
    xp, Wp, bp = _pad32(x, Wt, bits)
    packed = c_oracle.pack(bp)
    h = Wt.shape[0]
    y_c = c_oracle.forward(xp, Wp, np.arange(h), packed, bits.shape[0], act)
    return y_np, y_c


# ---------------------------------------------------------------- worked example (P1)
@pytest.mark.parametrize("act_name", ["identity", "relu", "swish", "sigmoid", "gelu"])
def test_worked_example_2x2(c_oracle, golden_dir, act_name):
    """SPEC S:160/S:246/S:256 example.  Pins orientation (A = Wt, row = output), which stream is
    activated (swapping gate/value changes the swish/sigmoid/gelu values), and the complement."""
    g = _load(golden_dir, "p1_worked_example.json")
    bits = np.array([g["mask"]], dtype=np.uint8)
    act = ACT_NAMES[act_name]
    for y in _forward_both(c_oracle, g["x"], g["Wt"], bits, act):
        np.testing.assert_allclose(y[0], g["y"][act_name], rtol=1e-15, atol=0)
    t, gate, value = mglu_partials_np(np.array([g["x"]], float), np.array(g["Wt"], float), bits)
    assert t[0].tolist() == g["t"] and gate[0, 0].tolist() == g["gate"] and value[0, 0].tolist() == g["value"]
    xp, Wp, bp = _pad32(np.array([g["x"]], float), np.array(g["Wt"], float), bits)
    y, z, tc = c_oracle.forward(xp, Wp, np.arange(2), c_oracle.pack(bp), 1, act, want_partials=True)
    assert z[0, 0].tolist() == g["gate"] and z[0, 1].tolist() == g["value"] and tc[0].tolist() == g["t"]


def test_worked_example_not_swapped(c_oracle, golden_dir):
    """Reading R1: bit = 1 -> gate (activated).  The swapped orientation must not come out."""
    g = _load(golden_dir, "p1_worked_example.json")
    bits = np.array([g["mask"]], dtype=np.uint8)
    for y in _forward_both(c_oracle, g["x"], g["Wt"], bits, ACT_SWISH):
        assert not np.allclose(y[0], g["y_swish_swapped"], rtol=1e-6)


@pytest.mark.parametrize("act_name", ["identity", "swish"])
def test_worked_example_nm2_complement(c_oracle, golden_dir, act_name):
    """n_m=2 with M2 = Mbar1 doubles the identity output; pins the sum over i
    (a 1/n_m normalisation, reading R6, would halve it)."""
    g = _load(golden_dir, "p1_worked_example.json")
    bits = np.array([g["mask"], g["n_m2_complement"]["mask2"]], dtype=np.uint8)
    for y in _forward_both(c_oracle, g["x"], g["Wt"], bits, ACT_NAMES[act_name]):
        np.testing.assert_allclose(y[0], g["n_m2_complement"]["y"][act_name], rtol=1e-15)


def test_activation_closed_forms(golden_dir):
    """swish(1); gelu(z) = z*Phi(z) at z = 1, 2 with Phi from the standard normal table
    value Phi(1) = 0.8413447460685429, Phi(2) = 0.9772498680518208; relu, sigmoid(0) = 1/2."""
    g = _load(golden_dir, "p1_worked_example.json")
    assert act_np(ACT_SWISH, np.array([1.0]))[0] == pytest.approx(g["swish_at_1"], rel=1e-15)
    assert act_np(ACT_GELU, np.array([1.0, 2.0])).tolist() == pytest.approx(
        [0.8413447460685429, 2 * 0.9772498680518208], rel=1e-14)
    assert act_np(ACT_RELU, np.array([-1.0, 0.0, 2.5])).tolist() == [0.0, 0.0, 2.5]
    assert act_np(ACT_SIGMOID, np.array([0.0]))[0] == 0.5
    assert act_np(ACT_SWISH, np.array([0.0]))[0] == 0.0


# ---------------------------------------------------------------- exhaustive codes
@pytest.mark.parametrize("n_m", [1, 2, 4, 8])
def test_exhaustive_code_pairs_identity(c_oracle, n_m):
    """d = 2, one output: with identity g, Eq. 3 reduces to the closed form
    y = popcount(c0 XOR c1) * p0 * p1 (p_k = x_k w_k): each mask contributes p0*p1 exactly when
    the two elements land in different streams.  Enumerates every code pair (all 2^(2 n_m) for
    n_m <= 4, a seeded 2000-pair sample for n_m = 8).  Pins bit indexing and the plain sum."""
    rng = np.random.default_rng(n_m)
    pairs = list(itertools.product(range(2 ** n_m), repeat=2)) if n_m <= 4 else \
        [tuple(p) for p in rng.integers(0, 2 ** n_m, size=(2000, 2))]
    x = np.array([[1.5, -0.75]])
    Wt = np.array([[0.5, 2.0]])
    p0, p1 = 1.5 * 0.5, -0.75 * 2.0
    # all pairs in one call: h = len(pairs) rows, each row its own code pair
    h = len(pairs)
    bits = np.zeros((n_m, h, 2), dtype=np.uint8)
    for j, (c0, c1) in enumerate(pairs):
        for i in range(n_m):
            bits[i, j, 0] = (c0 >> i) & 1
            bits[i, j, 1] = (c1 >> i) & 1
    Wt_rep = np.repeat(Wt, h, axis=0)
    expect = np.array([bin(c0 ^ c1).count("1") * p0 * p1 for c0, c1 in pairs])
    for y in _forward_both(c_oracle, x, Wt_rep, bits, ACT_IDENTITY):
        np.testing.assert_allclose(y[0], expect, rtol=0, atol=1e-15)


@pytest.mark.parametrize("n_m", [1, 2, 4, 8])
def test_single_element_sigmoid_counts_zero_bits(c_oracle, n_m):
    """d = 1: each mask puts the single product p either in the gate (value = 0) or in the value
    (gate = 0, sigmoid(0) = 1/2), so y = (n_m - popcount(c)) * p / 2 for every code c."""
    codes = np.arange(2 ** n_m)
    h = len(codes)
    bits = np.array([[[(c >> i) & 1] for c in codes] for i in range(n_m)], dtype=np.uint8)
    p = 0.8125 * -1.25
    Wt = np.full((h, 1), -1.25)
    x = np.array([[0.8125]])
    expect = np.array([(n_m - bin(c).count("1")) * p / 2 for c in codes])
    for y in _forward_both(c_oracle, x, Wt, bits, ACT_SIGMOID):
        np.testing.assert_allclose(y[0], expect, rtol=0, atol=1e-15)


# ---------------------------------------------------------------- exact rational brute force
def _brute_fraction(x, Wt, bits, act):
    """Eq. 3 with Python Fractions (exact) for identity/relu, pure loops."""
    n_m, h, d = bits.shape
    B = len(x)
    out = [[Fraction(0)] * h for _ in range(B)]
    for b in range(B):
        for j in range(h):
            acc = Fraction(0)
            for i in range(n_m):
                gate = sum((Fraction(x[b][k]) * Fraction(Wt[j][k]) for k in range(d) if bits[i][j][k]), Fraction(0))
                value = sum((Fraction(x[b][k]) * Fraction(Wt[j][k]) for k in range(d) if not bits[i][j][k]), Fraction(0))
                gval = gate if act == ACT_IDENTITY else max(gate, Fraction(0))
                acc += gval * value
            out[b][j] = acc
    return out


@pytest.mark.parametrize("n_m,act", [(1, ACT_IDENTITY), (2, ACT_RELU), (4, ACT_IDENTITY), (8, ACT_RELU)])
def test_exact_rational_bruteforce(c_oracle, n_m, act):
    """Dyadic inputs (exact in binary64), B=3, h=5, d=7 -- asymmetric so a transposed operand
    fails.  The oracle must equal the exact rational result up to binary64 rounding."""
    rng = np.random.default_rng(100 + n_m)
    B, h, d = 3, 5, 7
    x = rng.integers(-16, 17, size=(B, d)) / 8.0
    Wt = rng.integers(-16, 17, size=(h, d)) / 16.0
    bits = rng.integers(0, 2, size=(n_m, h, d)).astype(np.uint8)
    exact = np.array([[float(v) for v in row] for row in _brute_fraction(x, Wt, bits, act)])
    for y in _forward_both(c_oracle, x, Wt, bits, act):
        np.testing.assert_allclose(y, exact, rtol=1e-13, atol=1e-13)


def test_pure_python_loops_swish_gelu(c_oracle):
    """Smooth activations: a pure-Python loop evaluation (math.fsum, math.exp/erf) vs both
    oracles on seeded float inputs, B=2, h=9, d=13, n_m=4."""
    rng = np.random.default_rng(7)
    B, h, d, n_m = 2, 9, 13, 4
    x = rng.standard_normal((B, d))
    Wt = rng.uniform(-0.3, 0.3, (h, d))
    bits = rng.integers(0, 2, size=(n_m, h, d)).astype(np.uint8)
    for act, g in ((ACT_SWISH, lambda z: z / (1 + math.exp(-z))),
                   (ACT_GELU, lambda z: 0.5 * z * (1 + math.erf(z / math.sqrt(2))))):
        ref = np.zeros((B, h))
        for b in range(B):
            for j in range(h):
                tot = []
                for i in range(n_m):
                    gate = math.fsum(x[b, k] * Wt[j, k] for k in range(d) if bits[i, j, k])
                    value = math.fsum(x[b, k] * Wt[j, k] for k in range(d) if not bits[i, j, k])
                    tot.append(g(gate) * value)
                ref[b, j] = math.fsum(tot)
        for y in _forward_both(c_oracle, x, Wt, bits, act):
            np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-14)


# ---------------------------------------------------------------- special masks / invariants
@pytest.mark.parametrize("act_name", list(ACT_NAMES))
def test_all_ones_mask_gives_zero(c_oracle, act_name):
    """M_i = 1 everywhere -> value_i = x(0 (.) W) = 0 -> y = 0 exactly for every g."""
    inp = make_inputs(3, B=2, d=64, h=16, n_m=4, dtype="f32", density="ones")
    for y in _forward_both(c_oracle, inp["x"], inp["Wt"], inp["bits"], ACT_NAMES[act_name]):
        assert np.all(y == 0.0)


@pytest.mark.parametrize("n_m", [1, 2, 4, 8])
def test_all_zeros_mask_sigmoid_is_plain_projection(c_oracle, n_m):
    """M_i = 0 -> gate_i = 0, value_i = xW -> y = n_m * sigmoid(0) * xW = (n_m/2) xW: a plain
    ungated projection (north_star), checked against math.fsum dot products."""
    inp = make_inputs(4, B=2, d=64, h=16, n_m=n_m, dtype="f32", density="zeros")
    x = inp["x"].astype(np.float64)
    Wt = inp["Wt"].astype(np.float64)
    ref = np.array([[n_m / 2 * math.fsum(x[b] * Wt[j]) for j in range(16)] for b in range(2)])
    for y in _forward_both(c_oracle, x, Wt, inp["bits"], ACT_SIGMOID):
        np.testing.assert_allclose(y, ref, rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("n_m", [1, 2, 4, 8])
def test_complementarity(c_oracle, n_m):
    """gate_i + value_i = t.  value_i is computed from Mbar
    independently in both oracles, so this is a real check (to binary64 reassociation)."""
    inp = make_inputs(5, B=3, d=96, h=24, n_m=n_m, dtype="f32")
    x, Wt, bits = inp["x"].astype(float), inp["Wt"].astype(float), inp["bits"]
    t, gate, value = mglu_partials_np(x, Wt, bits)
    np.testing.assert_allclose(gate + value, np.broadcast_to(t, gate.shape), rtol=1e-13, atol=1e-14)
    _, z, tc = c_oracle.forward(x, Wt, np.arange(24), c_oracle.pack(bits), n_m, ACT_SWISH,
                                want_partials=True)     # d = 96: a multiple of the 32-column group
    np.testing.assert_allclose(z[:, :n_m] + z[:, n_m:], np.repeat(tc[:, None], n_m, 1), rtol=1e-13, atol=1e-14)
    np.testing.assert_allclose(tc, t, rtol=1e-13, atol=1e-14)


def test_glu_on_disjoint_supports(c_oracle):
    """MGLU(n_m=1) equals GLU g(xW_g) (.) xW_v with W_g = M (.) W, W_v = Mbar (.) W,
    evaluated here as textbook fsum dot products of the two explicit matrices."""
    inp = make_inputs(6, B=2, d=32, h=8, n_m=1, dtype="f32")
    x, Wt, M = inp["x"].astype(float), inp["Wt"].astype(float), inp["bits"][0].astype(float)
    Wg, Wv = M * Wt, (1 - M) * Wt
    ref = np.array([[(lambda a, v: a / (1 + math.exp(-a)) * v)(math.fsum(x[b] * Wg[j]), math.fsum(x[b] * Wv[j]))
                     for j in range(8)] for b in range(2)])
    for y in _forward_both(c_oracle, x, Wt, inp["bits"], ACT_SWISH):
        np.testing.assert_allclose(y, ref, rtol=1e-13)


def test_token_rows_independent(c_oracle):
    """Reading R15: each token row is its own Eq. 3 instance."""
    inp = make_inputs(8, B=4, d=32, h=8, n_m=2, dtype="f32")
    x, Wt, bits = inp["x"].astype(float), inp["Wt"].astype(float), inp["bits"]
    full = mglu_forward_np(x, Wt, bits, ACT_SWISH)
    for b in range(4):
        np.testing.assert_allclose(mglu_forward_np(x[b:b + 1], Wt, bits, ACT_SWISH)[0], full[b],
                                   rtol=1e-13, atol=1e-15)


def test_c_and_numpy_agree_on_seeded_bf16(c_oracle):
    """The two oracle implementations (numpy matmul on masked matrices vs C loops on the packed
    stream) agree on a bf16-decoded seeded instance spanning several n_m."""
    for n_m in (1, 2, 4, 8):
        inp = make_inputs(9, B=2, d=128, h=48, n_m=n_m, dtype="bf16")
        x, Wt = decode_bf16(inp["x"]), decode_bf16(inp["Wt"])
        y_np, y_c = _forward_both(c_oracle, x, Wt, inp["bits"], ACT_SWISH)
        np.testing.assert_allclose(y_c, y_np, rtol=1e-12, atol=1e-14)


def test_decode_bf16_exact():
    """bf16 bit patterns decode to the documented values (1.0 = 0x3f80, -2.0 = 0xc000,
    2^-133 subnormal = 0x0001, 0x7f7f = 3.3895313892515355e38)."""
    got = decode_bf16(np.array([0x3F80, 0xC000, 0x0001, 0x7F7F], dtype=np.uint16))
    assert got.tolist() == [1.0, -2.0, 2.0 ** -133, 3.3895313892515355e38]


# ---------------------------------------------------------------- packing (a1)
def _golden_bits(case):
    bits = np.zeros((case["n_m"], case["h"], case["d"]), dtype=np.uint8)
    for i, j, k in case["ones"]:
        bits[i - 1, j, k] = 1
    return bits


def test_pack_golden_vectors(c_oracle, golden_dir):
    for case in _load(golden_dir, "pack_golden.json")["cases"]:
        bits = _golden_bits(case)
        want = bytes.fromhex(case["packed_hex"])
        assert bytes(pack_np(bits)) == want
        assert bytes(c_oracle.pack(bits)) == want
        np.testing.assert_array_equal(unpack_np(np.frombuffer(want, np.uint8), case["n_m"], case["h"], case["d"]), bits)
        np.testing.assert_array_equal(c_oracle.unpack(np.frombuffer(want, np.uint8), case["n_m"], case["h"], case["d"]), bits)


@pytest.mark.parametrize("n_m", [1, 2, 4, 8])
def test_pack_round_trip(c_oracle, n_m):
    """pack(unpack(p)) = p for random streams; numpy and C unpackers agree."""
    rng = np.random.default_rng(n_m)
    h, d = 6, 96
    packed = rng.integers(0, 256, size=h * d * n_m // 8, dtype=np.uint8)
    b1 = unpack_np(packed, n_m, h, d)
    b2 = c_oracle.unpack(packed, n_m, h, d)
    np.testing.assert_array_equal(b1, b2)
    np.testing.assert_array_equal(pack_np(b1), packed)
    np.testing.assert_array_equal(c_oracle.pack(b2), packed)


def test_binarize_strict_threshold():
    """Alg. 2 '(soft_mask > 0)' and S:67: logit 0.0 -> 0; the synthetic recipe gives
    ~50 % ones (P:1045 init 0.01*randn)."""
    logits = np.array([0.3, -0.2, 0.0, -0.0, 1e-30])
    assert ((logits > 0).astype(int)).tolist() == [1, 0, 0, 0, 1]
    lg = make_logits(0, 2, 64, 64)
    frac = float((lg > 0).mean())
    assert abs(frac - 0.5) < 0.02


@pytest.mark.parametrize("n_m", [1, 4])
def test_layout_bit_positions(c_oracle, n_m):
    """Reading R3, enumerated: a word with the single bit p set marks exactly column
    2*(p % 16) + p // 16 of its group (bits 0..15 even columns, 16..31 odd), for every p, every
    mask word and a second group -- both unpackers."""
    h, d = 1, 64
    for g in range(2):
        for i in range(n_m):
            for pbit in range(32):
                words = np.zeros(h * (d // 32) * n_m, dtype="<u4")
                words[g * n_m + i] = np.uint32(1) << np.uint32(pbit)
                packed = np.frombuffer(words.tobytes(), dtype=np.uint8)
                want = np.zeros((n_m, h, d), dtype=np.uint8)
                want[i, 0, 32 * g + 2 * (pbit % 16) + pbit // 16] = 1
                np.testing.assert_array_equal(unpack_np(packed, n_m, h, d), want)
                np.testing.assert_array_equal(c_oracle.unpack(packed, n_m, h, d), want)


@pytest.mark.parametrize("n_m", [3, 5, 6, 7, 16])
def test_wider_and_odd_mask_counts(n_m):
    """Row f3 ("Scaling n_m to 16"): the layout and Eq. 3 for any n_m up to 16 -- the C
    oracle's own unpacker and sum equal the numpy twin's explicit masked matrices, and the
    all-zeros masks reduce to the plain projection n_m * g(0) * xW (sigmoid: n_m/2 * xW)."""
    from oracle import ACT_SIGMOID, ACT_SWISH, COracle, mglu_forward_np, pack_np, unpack_np
    rng = np.random.default_rng(n_m)
    B, d, h = 2, 64, 9
    x = rng.standard_normal((B, d))
    Wt = rng.standard_normal((h, d))
    bits = rng.integers(0, 2, (n_m, h, d)).astype(np.uint8)
    o = COracle()
    packed = o.pack(bits)
    assert packed.size == h * d * n_m // 8
    np.testing.assert_array_equal(packed, pack_np(bits))
    np.testing.assert_array_equal(unpack_np(packed, n_m, h, d), bits)
    y = o.forward(x, Wt, np.arange(h), packed, n_m, ACT_SWISH)
    np.testing.assert_allclose(y, mglu_forward_np(x, Wt, bits, ACT_SWISH), rtol=1e-11, atol=1e-11)
    zeros = o.pack(np.zeros_like(bits))
    np.testing.assert_allclose(o.forward(x, Wt, np.arange(h), zeros, n_m, ACT_SIGMOID), n_m / 2 * x @ Wt.T,
                               rtol=1e-12, atol=1e-12)
