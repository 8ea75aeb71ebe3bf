"""Per-element mask code streams: the oracle's
bit-by-bit reader pinned by SURVEY's golden vectors, then the library's converters
(mglu_codes_to_bits_host / mglu_pack_codes_host / mglu_unpack_codes_host) against the oracle and
the packed layout.  CPU only: no compute call."""
import json
import os

import numpy as np
import pytest

from oracle import bits_to_codes_np, codes_to_bits_np, pack_np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "c3_golden.json")))["cases"]


def _golden_masks(c):
    if "masks" in c:
        return np.array(c["masks"], dtype=np.uint8)
    codes = np.array(c["codes"], dtype=np.int64)
    return np.stack([(codes >> i) & 1 for i in range(c["n_m"])]).astype(np.uint8)


@pytest.mark.parametrize("case", range(len(GOLD)))
def test_oracle_reads_golden_vectors(case):
    c = GOLD[case]
    stream = np.frombuffer(bytes.fromhex(c["hex"]), dtype=np.uint8)
    bits = codes_to_bits_np(stream, c["w"], c["n_m"], c["h"], c["d"])
    np.testing.assert_array_equal(bits, _golden_masks(c))
    np.testing.assert_array_equal(bits_to_codes_np(bits, c["w"]), stream)


def test_oracle_rejects_high_bits_and_wide_fields():
    with pytest.raises(ValueError):                       # code 0x10 with n_m = 4 in a byte field
        codes_to_bits_np(np.array([0x10], dtype=np.uint8), 8, 4, 1, 1)
    with pytest.raises(ValueError):
        codes_to_bits_np(np.array([0], dtype=np.uint8), 2, 4, 1, 1)


def test_oracle_int8_per_element_equals_dense_stream():
    """The listing's uint8-per-element codes and the dense n_m-bit stream describe the
    same masks: reading both gives identical bits."""
    rng = np.random.default_rng(3)
    for n_m in (1, 2, 4):
        bits = rng.integers(0, 2, (n_m, 3, 8)).astype(np.uint8)
        dense = bits_to_codes_np(bits, n_m)
        byte = bits_to_codes_np(bits, 8)
        assert byte.size == 24 and dense.size == 24 * n_m // 8
        np.testing.assert_array_equal(byte, (bits * (1 << np.arange(n_m))[:, None, None]).sum(0).ravel())
        np.testing.assert_array_equal(codes_to_bits_np(dense, n_m, n_m, 3, 8), codes_to_bits_np(byte, 8, n_m, 3, 8))


# ------------------------------------------------------------------ the library's converters
@pytest.fixture(scope="module")
def M():
    from paper_2506_23225_b200 import mglu as M
    from paper_2506_23225_b200.build import build
    build()
    M.load_library()
    return M


@pytest.mark.parametrize("case", range(len(GOLD)))
def test_library_reads_golden_vectors(M, case):
    c = GOLD[case]
    stream = np.frombuffer(bytes.fromhex(c["hex"]), dtype=np.uint8)
    np.testing.assert_array_equal(M.mglu_codes_to_bits_host(stream, c["w"], c["n_m"], c["h"], c["d"]),
                                  _golden_masks(c))


@pytest.mark.parametrize("n_m,w", [(1, 1), (2, 2), (4, 4), (8, 8), (16, 16), (3, 8), (4, 8), (1, 8), (5, 16)])
def test_library_pack_codes_matches_oracle(M, n_m, w):
    rng = np.random.default_rng(n_m * 31 + w)
    h, d = 5, 64
    bits = rng.integers(0, 2, (n_m, h, d)).astype(np.uint8)
    stream = bits_to_codes_np(bits, w)
    assert stream.size == M.mglu_code_stream_bytes(d, h, w)
    packed = M.mglu_pack_codes_host(stream, w, n_m, h, d)
    np.testing.assert_array_equal(packed, pack_np(bits))                         # == packing the masks
    np.testing.assert_array_equal(M.mglu_codes_to_bits_host(stream, w, n_m, h, d), codes_to_bits_np(stream, w, n_m, h, d))
    np.testing.assert_array_equal(M.mglu_unpack_codes_host(packed, n_m, h, d, w), stream)   # round trip


def test_library_rejects_contaminated_fields(M):
    stream = np.zeros(32, dtype=np.uint8)
    stream[5] = 0x10                                       # bit 4 of a byte field with n_m = 4
    with pytest.raises(M.MgluError) as e:
        M.mglu_pack_codes_host(stream, 8, 4, 1, 32)
    assert e.value.status == M.MGLU_ERR_INVALID_ARG
    with pytest.raises(M.MgluError) as e:
        M.mglu_codes_to_bits_host(stream, 8, 4, 1, 32)
    assert e.value.status == M.MGLU_ERR_INVALID_ARG
    with pytest.raises(M.MgluError) as e:                  # field narrower than n_m
        M.mglu_pack_codes_host(np.zeros(16, dtype=np.uint8), 2, 4, 1, 64)
    assert e.value.status == M.MGLU_ERR_UNSUPPORTED
