"""Test hooks and interop through the real kernels (-m gpu):
  * the mask-corruption hook: with one mask bit flipped, the bit-exact decode probe
    must fail at exactly that element on every fast path, and pass again once the hook is cleared;
  * forward from per-element code streams (P:244 dense C3 stream, P:1084 one byte per element):
    codes -> mglu_pack_codes_host -> forward, against the oracle reading the stream itself."""
import numpy as np
import pytest
import torch

from tests.helpers import TIGHT, make_inputs, normwise_err, oracle, oracle_inputs, to_device

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_23225_b200.build import build
    build()


def _one_hot_probe(layer, Wt, packed, d, T):
    """y for x = e_k, Wt = 1, sigmoid g: (n_m - popcount(code[j, k])) / 2 for every k."""
    out = []
    for k0 in range(0, d, T):
        x = torch.zeros(T, d, device="cuda", dtype=torch.bfloat16)
        x[torch.arange(T), torch.arange(k0, k0 + T)] = 1.0
        out.append(layer.forward(x, Wt, packed).float().cpu().numpy())
    return np.concatenate(out)                            # [d][h]


@pytest.mark.parametrize("path,T", [("mma", 4), ("tcdec", 8), ("tcrow", 16), ("tcgen05", 32), ("simt", 8)])
def test_mask_corruption_hook_is_detected(path, T):
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    d, h, n_m = 256, 200, 4
    inp = make_inputs(61, B=1, d=d, h=h, n_m=n_m, dtype="bf16")
    bits = inp["bits"]
    packed = torch.from_numpy(mglu_pack_masks_host(bits)).cuda()
    before = packed.clone()
    Wt = torch.ones(h, d, device="cuda", dtype=torch.bfloat16)
    layer = Mglu(d, h, n_m, act="sigmoid", dtype="bf16", path=path)
    want = ((n_m - bits.sum(axis=0)) / 2.0).T             # [d][h]
    layer.set_debug(1)
    y = _one_hot_probe(layer, Wt, packed, d, T)
    torch.cuda.synchronize()
    bad = np.argwhere(y != want)
    # exactly element (row 0, column 0): mask 1's bit flipped changes popcount by one
    assert bad.tolist() == [[0, 0]], bad[:10]
    assert abs(y[0, 0] - want[0, 0]) == 0.5
    assert torch.equal(packed, before)                    # the hook restores the caller's codes
    layer.set_debug(0)
    np.testing.assert_array_equal(_one_hot_probe(layer, Wt, packed, d, T), want)


@pytest.mark.parametrize("w,n_m", [(4, 4), (8, 4), (1, 1), (8, 8), (2, 2)])
def test_forward_from_code_stream(w, n_m):
    from oracle import bits_to_codes_np, codes_to_bits_np
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_codes_host
    d, h, B = 512, 160, 2
    inp = make_inputs(90 + w + n_m, B=B, d=d, h=h, n_m=n_m, dtype="bf16")
    stream = bits_to_codes_np(inp["bits"], w)              # the caller's per-element codes
    x, Wt = to_device(inp, "bf16")
    packed = torch.from_numpy(mglu_pack_codes_host(stream, w, n_m, h, d)).cuda()
    y = Mglu(d, h, n_m, act="swish", dtype="bf16").forward(x, Wt, packed)
    xo, Wo = oracle_inputs(inp, "bf16")
    o = oracle()
    ref = o.forward(xo, Wo, np.arange(h), o.pack(codes_to_bits_np(stream, w, n_m, h, d)), n_m, 1)
    assert normwise_err(y.float().cpu().numpy().astype(np.float64), ref) <= TIGHT["bf16"]
