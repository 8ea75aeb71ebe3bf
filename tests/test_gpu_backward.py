"""GPU parity of the training path (row f4, mglu_backward through the C ABI) against the oracle's
Alg. 2 STE gradients (oracle/backward.py, pinned by tests/test_oracle_backward.py): fp32 and bf16
handles, every activation, n_m in {1, 2, 4, 8}, ragged tiles; the forward streams come from each
fast forward kernel's partials mode (paths mma / tcdec / tcgen05 / simt); optional outputs."""
import numpy as np
import pytest
import torch

from tests.helpers import make_inputs, normwise_err, oracle_inputs, to_device

pytestmark = pytest.mark.gpu

ACTS = {"identity": 0, "swish": 1, "gelu": 2, "relu": 3, "sigmoid": 4}


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_23225_b200.build import build
    build()


def _run(dtype, n_m, act, B, d, h, path="auto", seed=0):
    from oracle import mglu_backward_np
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    inp = make_inputs(700 + seed + n_m + B, B=B, d=d, h=h, n_m=n_m, dtype=dtype)
    x, Wt = to_device(inp, dtype)
    packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
    dy = torch.from_numpy(np.random.default_rng(seed + 5).standard_normal((B, h)).astype(np.float32)).cuda()
    layer = Mglu(d, h, n_m, act=act, dtype=dtype, path=path)
    dx, dW, dl = layer.backward(x, Wt, packed, dy)
    torch.cuda.synchronize()
    xo, Wo = oracle_inputs(inp, dtype)
    rdx, rdW, rdl = mglu_backward_np(xo, Wo, inp["bits"], dy.cpu().numpy().astype(np.float64), ACTS[act])
    return (dx, dW, dl), (rdx, rdW, rdl), layer


def _err(a, ref):
    a = a.cpu().numpy().astype(np.float64).reshape(ref.shape[0], -1)
    return normwise_err(a, ref.reshape(ref.shape[0], -1))


# fp32 accumulation of exact products against binary64: ~1e-6 normwise; the bf16-input handles
# add the forward streams' fp32 rounding before g / g' (same order): held to 1e-4
TOL = {"f32": 2e-5, "bf16": 1e-4}


@pytest.mark.parametrize("act", list(ACTS))
@pytest.mark.parametrize("n_m", [1, 4])
def test_backward_f32_every_activation(act, n_m):
    got, ref, _ = _run("f32", n_m, act, B=5, d=96, h=70)
    for g, r in zip(got, ref):
        assert _err(g, r) <= TOL["f32"], (act, n_m)


@pytest.mark.parametrize("n_m", [1, 2, 4, 8])
@pytest.mark.parametrize("path,B", [("auto", 3), ("mma", 2), ("tcdec", 9), ("tcrow", 11), ("tcgen05", 40), ("simt", 4)])
def test_backward_bf16_paths(n_m, path, B):
    if path == "mma" and n_m >= 4 and B > 4:
        pytest.skip("one token group on the MMA path")
    got, ref, layer = _run("bf16", n_m, "swish", B=B, d=256, h=200, path=path)
    for g, r in zip(got, ref):
        assert _err(g, r) <= TOL["bf16"], (path, n_m)


def test_backward_optional_outputs_and_zero_upstream():
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    d, h, n_m, B = 128, 64, 2, 3
    inp = make_inputs(9, B=B, d=d, h=h, n_m=n_m, dtype="bf16")
    x, Wt = to_device(inp, "bf16")
    packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
    layer = Mglu(d, h, n_m, dtype="bf16")
    dx, dW, dl = layer.backward(x, Wt, packed, torch.zeros(B, h, device="cuda"))
    assert not dx.any() and not dW.any() and not dl.any()
    dx2, dW2, dl2 = layer.backward(x, Wt, packed, torch.ones(B, h, device="cuda"), want=("dW",))
    assert dx2 is None and dl2 is None and dW2.abs().sum() > 0


def test_backward_deterministic():
    got1, _, _ = _run("bf16", 4, "swish", B=20, d=512, h=300, path="tcdec", seed=3)
    got2, _, _ = _run("bf16", 4, "swish", B=20, d=512, h=300, path="tcdec", seed=3)
    for a, b in zip(got1, got2):
        assert torch.equal(a, b)
