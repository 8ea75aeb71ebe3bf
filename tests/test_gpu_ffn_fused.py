"""Row f1, fused (mglu_ffn_forward): the SwiMGLU FFN block out = MGLU(x) Wo^T (R19) in one
launch -- bit for bit the two-launch composition (up.forward, then the dense handle on its bf16
output), and against the binary64 oracle; repeated calls and CUDA-graph replays (the grid barrier
resets itself); unsupported configurations refused."""
import numpy as np
import pytest
import torch

from tests.helpers import TIGHT, make_inputs, normwise_err, oracle_inputs, to_device

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_23225_b200.build import build
    build()


def _wo(seed, d, h):
    g = torch.Generator().manual_seed(seed)
    return ((torch.rand(d, h, generator=g) * 2 - 1) / h ** 0.5).to(torch.bfloat16)


def _setup(seed, d, h, n_m, B, act="swish", d_out=None):
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    d_out = d if d_out is None else d_out
    inp = make_inputs(seed, B=B, d=d, h=h, n_m=n_m, dtype="bf16")
    x, Wt = to_device(inp, "bf16")
    packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
    Wo = _wo(seed + 1, d_out, h).cuda()
    up = Mglu(d, h, n_m, act=act, dtype="bf16")
    down = Mglu(h, d_out, 0, dtype="bf16")
    return inp, x, Wt, packed, Wo, up, down


@pytest.mark.parametrize("n_m", [1, 2, 4, 8])
@pytest.mark.parametrize("d,h,B", [(512, 1024, 1), (1024, 4096, 3), (256, 2048, 4), (2048, 1152, 2)])
def test_fused_ffn_equals_two_launches_and_oracle(n_m, d, h, B):
    from oracle import ffn_forward_np
    from paper_2506_23225_b200.mglu import ffn_forward_fused
    inp, x, Wt, packed, Wo, up, down = _setup(700 + n_m + d + B, d, h, n_m, B)
    ymid = torch.empty(B, h, dtype=torch.bfloat16, device="cuda")
    out = ffn_forward_fused(up, down, x, Wt, packed, Wo, y_mid=ymid)
    y2 = up.forward(x, Wt, packed)
    out2 = down.forward(y2, Wo, None)
    torch.cuda.synchronize()
    assert torch.equal(ymid, y2)
    assert torch.equal(out, out2)
    xo, Wto = oracle_inputs(inp, "bf16")
    ref = ffn_forward_np(xo, Wto, inp["bits"], Wo.float().cpu().numpy().astype(np.float64), 1)
    assert normwise_err(out.float().cpu().numpy().astype(np.float64), ref) <= TIGHT["bf16"]


@pytest.mark.parametrize("B", [1, 4])
def test_fused_ffn_config3_full_size(B):
    """Llama-3-8B FFN (d = 4096, h = 14336, n_m = 4): fused == two launches bit for bit, repeated
    calls and a CUDA-graph replay give the same output."""
    from paper_2506_23225_b200.mglu import ffn_forward_fused
    from synth import random_packed_codes
    from paper_2506_23225_b200.mglu import Mglu
    d, h, n_m = 4096, 14336, 4
    g = torch.Generator(device="cuda").manual_seed(B)
    x = torch.randn(B, d, device="cuda", generator=g).to(torch.bfloat16)
    Wt = ((torch.rand(h, d, device="cuda", generator=g) * 2 - 1) / d ** 0.5).to(torch.bfloat16)
    Wo = ((torch.rand(d, h, device="cuda", generator=g) * 2 - 1) / h ** 0.5).to(torch.bfloat16)
    packed = random_packed_codes(5, h, d, n_m, device="cuda")
    up, down = Mglu(d, h, n_m, dtype="bf16"), Mglu(h, d, 0, dtype="bf16")
    ref = down.forward(up.forward(x, Wt, packed), Wo, None)
    out = ffn_forward_fused(up, down, x, Wt, packed, Wo)
    assert torch.equal(out, ref)
    for _ in range(3):
        assert torch.equal(ffn_forward_fused(up, down, x, Wt, packed, Wo), ref)
    s = torch.cuda.Stream()
    ymid = torch.empty(B, h, dtype=torch.bfloat16, device="cuda")
    o = torch.empty(B, d, dtype=torch.bfloat16, device="cuda")
    with torch.cuda.stream(s):
        ffn_forward_fused(up, down, x, Wt, packed, Wo, y_mid=ymid, out=o, stream=s)
        s.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            ffn_forward_fused(up, down, x, Wt, packed, Wo, y_mid=ymid, out=o, stream=s)
            ffn_forward_fused(up, down, x, Wt, packed, Wo, y_mid=ymid, out=o, stream=s)
    for _ in range(3):
        o.zero_()
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(o, ref)


def test_fused_ffn_other_activation_and_output_width():
    from oracle import ffn_forward_np
    from paper_2506_23225_b200.mglu import ffn_forward_fused
    inp, x, Wt, packed, Wo, up, down = _setup(91, 1024, 2048, 4, 2, act="gelu", d_out=640)
    out = ffn_forward_fused(up, down, x, Wt, packed, Wo)
    assert torch.equal(out, down.forward(up.forward(x, Wt, packed), Wo, None))
    xo, Wto = oracle_inputs(inp, "bf16")
    ref = ffn_forward_np(xo, Wto, inp["bits"], Wo.float().cpu().numpy().astype(np.float64), 2)
    assert normwise_err(out.float().cpu().numpy().astype(np.float64), ref) <= TIGHT["bf16"]


@pytest.mark.parametrize("case", ["B5", "nm8_gelu", "mismatch", "alias"])
def test_fused_ffn_refuses(case):
    from paper_2506_23225_b200.mglu import Mglu, MgluError, MGLU_ERR_INVALID_ARG, MGLU_ERR_UNSUPPORTED, ffn_forward_fused
    n_m = 8 if case == "nm8_gelu" else 4
    B = 5 if case == "B5" else 2
    inp, x, Wt, packed, Wo, up, down = _setup(3, 512, 1024, n_m, B, act="gelu" if case == "nm8_gelu" else "swish")
    if case == "mismatch":
        down = Mglu(2048, 512, 0, dtype="bf16")
        Wo = torch.zeros(512, 1024, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(MgluError) as e:
        if case == "alias":                               # out aliasing y_mid: refused, not corrupted
            ym = torch.empty(2, 1024, dtype=torch.bfloat16, device="cuda")
            from paper_2506_23225_b200.mglu import _check, _ptr, _stream_ptr, load_library
            _check(load_library().mglu_ffn_forward(up.handle, down.handle, _ptr(x), 2, _ptr(Wt), _ptr(packed), _ptr(Wo),
                                                   _ptr(ym), _ptr(ym), _stream_ptr(None, x.device)), up.handle, "ffn")
        else:
            ffn_forward_fused(up, down, x, Wt, packed, Wo)
    want = MGLU_ERR_INVALID_ARG if case in ("mismatch", "alias") else MGLU_ERR_UNSUPPORTED
    assert e.value.status == want
