"""Row f3: mask counts outside {1, 2, 4, 8} (3, 5, 6, 7 and 16) through AUTO, bf16 and
fp32, against the oracle.  n_m = 16 (the 32-bit break-even of P:885) runs in bf16 on the
tcgen05 tile GEMM as a cluster of four CTAs with four masks each (DSMEM reduction in rank order);
the odd counts run on the SIMT kernel, and the paths that cannot serve a count refuse it
explicitly."""
import numpy as np
import pytest
import torch

from tests.helpers import TIGHT, TOL, gpu_forward, make_inputs, normwise_err, oracle_forward

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_23225_b200.build import build
    build()


@pytest.mark.parametrize("n_m", [3, 5, 6, 7, 16])
@pytest.mark.parametrize("dtype,B", [("bf16", 1), ("bf16", 6), ("f32", 2)])
def test_wide_mask_counts(n_m, dtype, B):
    inp = make_inputs(2000 + n_m * 7 + B, B=B, d=256, h=300, n_m=n_m, dtype=dtype)
    y, used = gpu_forward(inp, dtype, n_m, "swish")
    assert used == ("tcgen05" if (n_m == 16 and dtype == "bf16") else "simt")
    err = normwise_err(y, oracle_forward(inp, dtype, n_m, "swish"))
    assert err <= TOL[dtype] and err <= TIGHT[dtype], err


@pytest.mark.parametrize("path", ["mma", "tcdec", "tcgen05"])
def test_fast_paths_refuse_wide_counts(path):
    from paper_2506_23225_b200.mglu import MgluError, MGLU_ERR_UNSUPPORTED
    inp = make_inputs(1, B=2, d=256, h=128, n_m=3, dtype="bf16")
    with pytest.raises(MgluError) as e:
        gpu_forward(inp, "bf16", 3, "swish", path=path)
    assert e.value.status == MGLU_ERR_UNSUPPORTED


@pytest.mark.parametrize("path", ["mma", "tcdec", "tcrow"])
def test_fast_paths_refuse_sixteen_except_tile_gemm(path):
    from paper_2506_23225_b200.mglu import MgluError, MGLU_ERR_UNSUPPORTED
    inp = make_inputs(2, B=2, d=256, h=128, n_m=16, dtype="bf16")
    with pytest.raises(MgluError) as e:
        gpu_forward(inp, "bf16", 16, "swish", path=path)
    assert e.value.status == MGLU_ERR_UNSUPPORTED


@pytest.mark.parametrize("d,h,B", [(64, 128, 1), (256, 300, 5), (512, 260, 33), (1024, 700, 100), (2048, 129, 17)])
@pytest.mark.parametrize("act", ["swish", "gelu"])
def test_sixteen_masks_tile_gemm(d, h, B, act):
    inp = make_inputs(3100 + d + h + B, B=B, d=d, h=h, n_m=16, dtype="bf16")
    y, used = gpu_forward(inp, "bf16", 16, act, path="tcgen05")
    assert used == "tcgen05"
    err = normwise_err(y, oracle_forward(inp, "bf16", 16, act))
    assert err <= TIGHT["bf16"], err


def test_sixteen_masks_one_hot_bit_exact():
    """Wt = 1, x one-hot, sigmoid: y[b][j] = (16 - popcount(c[j, k0 + b])) / 2 exactly -- every mask
    bit of every (row, column) decoded through the four-CTA cluster and its DSMEM reduction."""
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    d, h, n_m = 256, 200, 16
    inp = make_inputs(77, B=1, d=d, h=h, n_m=n_m, dtype="bf16")
    bits = inp["bits"]
    packed = torch.from_numpy(mglu_pack_masks_host(bits)).cuda()
    Wt = torch.ones(h, d, device="cuda", dtype=torch.bfloat16)
    eye = torch.eye(d, device="cuda", dtype=torch.bfloat16)
    layer = Mglu(d, h, n_m, act="sigmoid", dtype="bf16", path="tcgen05")
    want = (n_m - bits.sum(axis=0).T) / 2.0
    for k0 in range(0, d, 32):
        y = layer.forward(eye[k0:k0 + 32].contiguous(), Wt, packed).float().cpu().numpy()
        np.testing.assert_array_equal(y, want[k0:k0 + 32])


def test_sixteen_masks_partials_vs_independent_value_stream():
    """The tile kernel's own s_i / t - s_i streams for all 16 masks (each CTA writes its four) against
    the oracle's gate and independently computed value streams."""
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    from tests.helpers import to_device
    d, h, B, n_m = 512, 300, 3, 16
    inp = make_inputs(88, B=B, d=d, h=h, n_m=n_m, dtype="bf16")
    x, Wt = to_device(inp, "bf16")
    packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
    z = Mglu(d, h, n_m, act="swish", dtype="bf16", path="tcgen05").forward_partials(x, Wt, packed)
    _, zr, tr = oracle_forward(inp, "bf16", n_m, "swish", want_partials=True)
    zz = z.cpu().numpy().astype(np.float64)
    for b in range(B):
        scale = np.max(np.abs(tr[b]))
        assert np.max(np.abs(zz[b] - zr[b])) / scale <= 1e-5
