"""Row f2's bandwidth half ("only those K masked projections need be evaluated -- reducing
memory traffic"): the routed forward on PLANE-MAJOR codes (mglu_forward_routed_planes), which
streams W and only the selected planes.  Checked bit for bit against the routed forward on the
interleaved codes (same kernel arithmetic, other operand source), against the oracle's routed sum
built from its independent gate/value streams, and the device converter against the host one."""
import numpy as np
import pytest
import torch

from tests.helpers import TIGHT, make_inputs, normwise_err, to_device
from tests.test_gpu_topk import _oracle_routed

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_23225_b200.build import build
    build()


def _topk_gate(rng, B, n_m, K):
    from oracle import topk_gate
    return topk_gate(rng.standard_normal((B, n_m)), K).astype(np.float32)


@pytest.mark.parametrize("n_m,h,d", [(1, 300, 512), (2, 1000, 1024), (4, 300, 512), (8, 1000, 1024), (8, 130, 2048)])
def test_device_planes_equal_host(n_m, h, d):
    from paper_2506_23225_b200.mglu import mglu_pack_masks_host, mglu_pack_planes_device, mglu_pack_planes_host
    rng = np.random.default_rng(n_m + h)
    bits = (rng.random((n_m, h, d)) < 0.5).astype(np.uint8)
    packed = mglu_pack_masks_host(bits)
    dev = mglu_pack_planes_device(torch.from_numpy(packed).cuda(), n_m, h, d).cpu().numpy()
    np.testing.assert_array_equal(dev, mglu_pack_planes_host(packed, n_m, h, d))


@pytest.mark.parametrize("n_m", [1, 2, 4, 8])
@pytest.mark.parametrize("B,K", [(1, 1), (1, 2), (2, 1), (3, 2), (4, 2)])
@pytest.mark.parametrize("d,h", [(512, 300), (1024, 1000)])
def test_routed_planes_bit_identical_and_oracle(n_m, B, K, d, h):
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host, mglu_pack_planes_device
    if K > n_m:
        pytest.skip("K > n_m")
    inp = make_inputs(4000 + 31 * n_m + 7 * B + K + d, B=B, d=d, h=h, n_m=n_m, dtype="bf16")
    x, Wt = to_device(inp, "bf16")
    packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
    planes = mglu_pack_planes_device(packed, n_m, h, d)
    G = _topk_gate(np.random.default_rng(B * 10 + K), B, n_m, K)
    Gd = torch.from_numpy(G).cuda()
    layer = Mglu(d, h, n_m, act="swish", dtype="bf16")
    y_pl = layer.forward_routed_planes(x, Wt, planes, Gd, K)
    y_r3 = layer.forward_routed(x, Wt, packed, Gd, K)
    torch.cuda.synchronize()
    assert layer.last_path() == "mma"
    assert torch.equal(y_pl, y_r3)
    ref = _oracle_routed(inp, n_m, 1, G.astype(np.float64))
    assert normwise_err(y_pl.float().cpu().numpy().astype(np.float64), ref) <= TIGHT["bf16"]


def test_routed_planes_full_size_config3_nm8():
    """d = 4096, h = 14336, n_m = 8, Top-2 at B = 1 (the bench's routed workload), sampled vs oracle
    and bit-identical to the interleaved routed call."""
    from oracle import decode_bf16
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_planes_device
    from synth import random_packed_codes
    from tests.helpers import oracle
    from oracle import mglu_routed_from_partials
    d, h, n_m, K = 4096, 14336, 8, 2
    g = torch.Generator(device="cuda").manual_seed(8)
    x = torch.randn(1, d, device="cuda", generator=g).to(torch.bfloat16)
    Wt = ((torch.rand(h, d, device="cuda", generator=g) * 2 - 1) / d ** 0.5).to(torch.bfloat16)
    packed = random_packed_codes(9, h, d, n_m, device="cuda")
    planes = mglu_pack_planes_device(packed, n_m, h, d)
    G = _topk_gate(np.random.default_rng(3), 1, n_m, K)
    Gd = torch.from_numpy(G).cuda()
    layer = Mglu(d, h, n_m, act="swish", dtype="bf16")
    y = layer.forward_routed_planes(x, Wt, planes, Gd, K)
    assert torch.equal(y, layer.forward_routed(x, Wt, packed, Gd, K))
    cols = np.sort(np.random.default_rng(4).choice(h, 200, replace=False))
    xo = decode_bf16(x.view(torch.int16).cpu().numpy().view(np.uint16))
    Wo = decode_bf16(Wt[torch.from_numpy(cols).cuda()].view(torch.int16).cpu().numpy().view(np.uint16))
    _, z, _ = oracle().forward(xo, Wo, cols, packed.cpu().numpy(), n_m, 1, want_partials=True)
    ref = mglu_routed_from_partials(np.transpose(z[:, :n_m], (1, 0, 2)), np.transpose(z[:, n_m:], (1, 0, 2)),
                                    G.astype(np.float64), 1)
    assert normwise_err(y[:, torch.from_numpy(cols).cuda()].float().cpu().numpy().astype(np.float64), ref) <= TIGHT["bf16"]


@pytest.mark.parametrize("case", ["B5", "gelu", "variant", "path"])
def test_routed_planes_refuses_unsupported(case):
    from paper_2506_23225_b200.mglu import Mglu, MgluError, MGLU_ERR_UNSUPPORTED, mglu_pack_masks_host
    d, h, n_m = 512, 300, 4
    B = 5 if case == "B5" else 2
    inp = make_inputs(5, B=B, d=d, h=h, n_m=n_m, dtype="bf16")
    x, Wt = to_device(inp, "bf16")
    packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
    Gd = torch.from_numpy(_topk_gate(np.random.default_rng(1), B, n_m, 2)).cuda()
    layer = Mglu(d, h, n_m, act="gelu" if case == "gelu" else "swish", dtype="bf16")
    if case == "variant":
        layer.set_variant("no_gate_mask")
    if case == "path":
        layer.set_path("tcdec")
    with pytest.raises(MgluError) as e:
        layer.forward_routed_planes(x, Wt, packed, Gd, 2)
    assert e.value.status == MGLU_ERR_UNSUPPORTED
