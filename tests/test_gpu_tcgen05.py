"""GPU parity of the tcgen05/TMEM masked GEMM (the prefill / large-batch regime)
against the CPU oracle on identical seeded inputs.

Shapes span several 128-row M tiles and BN-token N tiles (BN = 224/128/64/32 for n_m = 1/2/4/8)
with ragged tails in every dimension, including a final half K-block (d % 64 == 32); shapes whose
mask-word rows are not 16-byte multiples (d * n_m % 128 != 0) must be refused as UNSUPPORTED."""
import numpy as np
import pytest
import torch

from tests.helpers import TIGHT, TOL, gpu_forward, make_inputs, normwise_err, oracle_forward, oracle_inputs, to_device

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_23225_b200.build import build
    build()


TC_SHAPES = [  # (d, h, B)
    (64, 128, 1), (128, 200, 65), (96, 130, 17), (256, 333, 130), (1024, 256, 300), (4096, 384, 257),
    (2080, 129, 40), (2112, 140, 230), (192, 64, 480),
]


@pytest.mark.parametrize("n_m", [1, 2, 4, 8])
@pytest.mark.parametrize("d,h,B", TC_SHAPES)
def test_tc_shapes(n_m, d, h, B):
    inp = make_inputs(5000 + 13 * n_m + d + h + B, B=B, d=d, h=h, n_m=n_m, dtype="bf16")
    if (d // 32 * n_m) % 4:
        # the mask-word rows are fetched by TMA: d * n_m must be a multiple of 128
        from paper_2506_23225_b200.mglu import MgluError, MGLU_ERR_UNSUPPORTED
        with pytest.raises(MgluError) as e:
            gpu_forward(inp, "bf16", n_m, "swish", path="tcgen05")
        assert e.value.status == MGLU_ERR_UNSUPPORTED
        return
    y, used = gpu_forward(inp, "bf16", n_m, "swish", path="tcgen05")
    assert used == "tcgen05"
    ref = oracle_forward(inp, "bf16", n_m, "swish")
    err = normwise_err(y, ref)
    assert err <= TOL["bf16"] and err <= TIGHT["bf16"], err


@pytest.mark.parametrize("act", ["identity", "swish", "gelu", "relu", "sigmoid"])
def test_tc_activations(act):
    inp = make_inputs(88, B=100, d=512, h=256, n_m=4, dtype="bf16")
    y, _ = gpu_forward(inp, "bf16", 4, act, path="tcgen05")
    assert normwise_err(y, oracle_forward(inp, "bf16", 4, act)) <= TIGHT["bf16"]


@pytest.mark.parametrize("n_m", [1, 2, 4, 8])
def test_tc_one_hot_bit_exact(n_m):
    """Wt = 1 and x = I (token k one-hot at column k, B = d tokens in one call): with sigmoid g
    every accumulator is a small integer, so y[k][j] = (n_m - popcount(c[j,k])) / 2 exactly --
    the mask decode of every (row, column) checked bit-exactly through the tensor-core path."""
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    d, h = 384, 200
    inp = make_inputs(61 + n_m, B=1, d=d, h=h, n_m=n_m, dtype="bf16")
    bits = inp["bits"]
    packed = torch.from_numpy(mglu_pack_masks_host(bits)).cuda()
    Wt = torch.ones(h, d, device="cuda", dtype=torch.bfloat16)
    x = torch.eye(d, device="cuda", dtype=torch.bfloat16)
    layer = Mglu(d, h, n_m, act="sigmoid", dtype="bf16", path="tcgen05")
    y = layer.forward(x, Wt, packed).float().cpu().numpy()
    assert layer.last_path() == "tcgen05"
    want = (n_m - bits.sum(axis=0).T) / 2.0                        # [d tokens][h]
    np.testing.assert_array_equal(y, want)


def test_tc_all_ones_mask_zero():
    inp = make_inputs(3, B=70, d=256, h=192, n_m=4, dtype="bf16", density="ones")
    y, _ = gpu_forward(inp, "bf16", 4, "swish", path="tcgen05")
    assert np.all(y == 0.0)


def test_tc_all_zeros_mask_plain_projection():
    inp = make_inputs(4, B=90, d=256, h=192, n_m=2, dtype="bf16", density="zeros")
    y, _ = gpu_forward(inp, "bf16", 2, "sigmoid", path="tcgen05")
    x, Wt = oracle_inputs(inp, "bf16")
    assert normwise_err(y, (2 / 2) * x @ Wt.T) <= TIGHT["bf16"]


def test_tc_deterministic_and_auto():
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    inp = make_inputs(9, B=200, d=1024, h=300, n_m=4, dtype="bf16")
    x, Wt = to_device(inp, "bf16")
    packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
    layer = Mglu(1024, 300, 4, dtype="bf16")
    y0 = layer.forward(x, Wt, packed).clone()
    assert layer.last_path() == "tcgen05"                          # AUTO: B > 24 -> tile GEMM
    for _ in range(3):
        assert torch.equal(layer.forward(x, Wt, packed), y0)


def test_tc_back_to_back_pdl():
    """Two dependent launches on one stream (PDL): the second reads the first's output as x."""
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    d = h = 512
    inp = make_inputs(12, B=130, d=d, h=h, n_m=4, dtype="bf16")
    x, Wt = to_device(inp, "bf16")
    packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
    layer = Mglu(d, h, 4, act="identity", dtype="bf16", path="tcgen05")
    y1 = layer.forward(x, Wt, packed)
    y2 = layer.forward(y1, Wt, packed)
    torch.cuda.synchronize()
    y2_ref = layer.forward(y1.clone(), Wt, packed)
    torch.cuda.synchronize()
    assert torch.equal(y2, y2_ref)
