"""Plane-major code layout (row f2; include/mglu.h): the host converter against the layout
written out here from its definition -- plane i, row j, 32-column group g is one little-endian u32
word at word index (i h + j) d/32 + g whose bit (e >> 1) + 16 (e & 1) is M_{i+1}[j, 32 g + e].
CPU only (host functions of the library, no compute call)."""
import numpy as np
import pytest

from paper_2506_23225_b200.mglu import mglu_pack_masks_host, mglu_pack_planes_host


def _planes_by_definition(bits):
    n_m, h, d = bits.shape
    words = np.zeros((n_m, h, d // 32), dtype=np.uint64)
    for e in range(32):
        pos = (e >> 1) + 16 * (e & 1)
        words |= bits[:, :, e::32].astype(np.uint64) << np.uint64(pos)
    return words.astype("<u4").tobytes()


@pytest.mark.parametrize("n_m,h,d", [(1, 3, 32), (2, 5, 64), (4, 7, 96), (8, 2, 256), (16, 3, 64), (3, 4, 128)])
def test_host_planes_match_definition(n_m, h, d):
    rng = np.random.default_rng(n_m * 100 + h + d)
    bits = (rng.random((n_m, h, d)) < 0.5).astype(np.uint8)
    planes = mglu_pack_planes_host(mglu_pack_masks_host(bits), n_m, h, d)
    assert planes.tobytes() == _planes_by_definition(bits)


def test_single_bit_lands_in_its_plane_word():
    n_m, h, d = 4, 3, 64
    bits = np.zeros((n_m, h, d), dtype=np.uint8)
    bits[2, 1, 37] = 1                                   # mask 3, row 1, group 1, e = 5 -> bit 2 + 16
    planes = np.frombuffer(mglu_pack_planes_host(mglu_pack_masks_host(bits), n_m, h, d).tobytes(), dtype="<u4")
    want = np.zeros(n_m * h * d // 32, dtype=np.uint32)
    want[(2 * h + 1) * (d // 32) + 1] = 1 << 18
    np.testing.assert_array_equal(planes, want)
