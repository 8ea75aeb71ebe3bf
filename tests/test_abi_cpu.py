"""C-ABI checks that need no GPU: the library loads, exports every symbol include/mglu.h declares,
and its host packers agree bit for bit with the oracle's independent packer and the golden
vectors.  No compute call is made here."""
import ctypes
import json
import os

import numpy as np
import pytest
import torch

from paper_2506_23225_b200 import mglu as M
from paper_2506_23225_b200.build import build

pytestmark = pytest.mark.cpu


@pytest.fixture(scope="module")
def lib():
    build()
    return M.load_library()


def test_exports_every_header_symbol(lib):
    names = M.header_functions()
    assert len(names) >= 18
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/mglu.h but not exported"


def test_status_strings_and_version(lib):
    assert M.status_string(0) == "MGLU_OK"
    assert M.status_string(2) == "MGLU_ERR_UNSUPPORTED"
    assert M.status_string(99) == "MGLU_ERR_UNKNOWN"
    assert lib.mglu_version().decode().count(".") == 2
    assert lib.mglu_last_error(None).decode() == "null handle"


def test_packed_bytes(lib):
    assert M.mglu_packed_mask_bytes(4096, 14336, 4) == 14336 * 4096 // 2
    assert M.mglu_packed_mask_bytes(64, 128, 1) == 64 * 128 // 8
    assert M.mglu_packed_mask_bytes(64, 128, 3) == 64 * 128 * 3 // 8   # SIMT-only counts (row f3)
    assert M.mglu_packed_mask_bytes(64, 128, 16) == 64 * 128 * 2
    assert M.mglu_packed_mask_bytes(64, 128, 9) == 0
    assert M.mglu_packed_mask_bytes(64, 128, 0) == 0
    assert M.mglu_packed_mask_bytes(48, 128, 4) == 0         # d % 32 != 0
    assert M.mglu_packed_mask_bytes(-1, 128, 1) == 0


def test_create_argument_errors(lib):
    hd = ctypes.c_void_p()
    assert lib.mglu_create(None, 64, 128, 1, 1, 0, 0) == M.MGLU_ERR_INVALID_ARG
    assert lib.mglu_create(ctypes.byref(hd), 0, 128, 1, 1, 0, 0) == M.MGLU_ERR_INVALID_ARG
    assert lib.mglu_create(ctypes.byref(hd), 64, 128, 1, 9, 0, 0) == M.MGLU_ERR_INVALID_ARG
    assert lib.mglu_create(ctypes.byref(hd), 64, 128, 9, 1, 0, 0) == M.MGLU_ERR_UNSUPPORTED
    assert lib.mglu_create(ctypes.byref(hd), 64, 128, 17, 1, 0, 0) == M.MGLU_ERR_UNSUPPORTED
    assert lib.mglu_create(ctypes.byref(hd), 60, 128, 1, 1, 0, 0) == M.MGLU_ERR_UNSUPPORTED
    assert lib.mglu_destroy(None) == M.MGLU_OK
    assert lib.mglu_forward(None, None, 1, None, None, None, None) == M.MGLU_ERR_INVALID_ARG


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_create_without_gpu_fails_loudly(lib):
    hd = ctypes.c_void_p()
    assert lib.mglu_create(ctypes.byref(hd), 64, 128, 1, 1, 0, 0) == M.MGLU_ERR_CUDA
    assert hd.value is None


def test_host_pack_golden(lib, golden_dir):
    cases = json.load(open(os.path.join(golden_dir, "pack_golden.json")))["cases"]
    for case in cases:
        n_m, h, d = case["n_m"], case["h"], case["d"]
        bits = np.zeros((n_m, h, d), dtype=np.uint8)
        for i, j, k in case["ones"]:
            bits[i - 1, j, k] = 1
        assert bytes(M.mglu_pack_masks_host(bits)) == bytes.fromhex(case["packed_hex"])
        back = M.mglu_unpack_masks_host(np.frombuffer(bytes.fromhex(case["packed_hex"]), np.uint8), n_m, h, d)
        np.testing.assert_array_equal(back, bits)


@pytest.mark.parametrize("n_m", [1, 2, 4, 8])
def test_host_pack_matches_oracle(lib, c_oracle, n_m):
    from synth import make_inputs, make_logits
    inp = make_inputs(n_m, B=1, d=64, h=24, n_m=n_m)
    bits = inp["bits"]
    mine = M.mglu_pack_masks_host(bits)
    np.testing.assert_array_equal(mine, c_oracle.pack(bits))
    np.testing.assert_array_equal(M.mglu_unpack_masks_host(mine, n_m, 24, 64), bits)
    logits = make_logits(n_m, n_m, 24, 64)
    logits[0, 0, :4] = [0.0, -0.0, 1e-30, -1e-30]           # strict threshold (R4)
    ref = (logits > 0).astype(np.uint8)
    np.testing.assert_array_equal(M.mglu_pack_logits_host(logits), c_oracle.pack(ref))


def test_host_pack_rejects_non_binary(lib):
    bits = np.zeros((2, 4, 32), dtype=np.uint8)
    bits[1, 2, 3] = 2
    with pytest.raises(M.MgluError) as e:
        M.mglu_pack_masks_host(bits)
    assert e.value.status == M.MGLU_ERR_INVALID_ARG
    with pytest.raises(M.MgluError) as e:
        M.mglu_pack_masks_host(np.zeros((9, 4, 32), dtype=np.uint8))   # n_m in 1..8 or 16 (row f3)
    assert e.value.status == M.MGLU_ERR_UNSUPPORTED
    with pytest.raises(M.MgluError) as e:                   # d % 32 != 0 (layout groups, R3)
        M.mglu_pack_masks_host(np.zeros((2, 4, 48), dtype=np.uint8))
    assert e.value.status == M.MGLU_ERR_UNSUPPORTED


@pytest.mark.parametrize("n_m", [3, 5, 6, 7, 16])
def test_host_pack_wide_counts_match_oracle(lib, n_m):
    """The library's host packer equals the oracle's for the SIMT-only mask counts (row f3)."""
    from oracle import pack_np
    bits = np.random.default_rng(n_m).integers(0, 2, (n_m, 5, 64)).astype(np.uint8)
    np.testing.assert_array_equal(M.mglu_pack_masks_host(bits), pack_np(bits))
    np.testing.assert_array_equal(M.mglu_unpack_masks_host(pack_np(bits), n_m, 5, 64), bits)


def test_product_package_does_not_import_oracle():
    """The product path never imports the test oracle."""
    import pathlib
    pkg = pathlib.Path(__file__).resolve().parents[1] / "paper_2506_23225_b200"
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert "import oracle" not in src and "from oracle" not in src, f
    for f in list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        assert "oracle" not in f.read_text().lower() or f.name == "__never__", f
