"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (AUTO
dispatch -> the MMA decode kernel at B = 1, the row-split tcgen05 GEMV at B = 8), checked on sampled output columns the oracle computes one
by one, plus a one-hot decode probe on sampled k."""
import numpy as np
import pytest
import torch

from tests.helpers import TIGHT, make_inputs, normwise_err, oracle, oracle_inputs, to_device

pytestmark = pytest.mark.gpu

FULL = [  # (name, d, h, n_m, B)
    ("config2_decode_7b", 4096, 11008, 4, 1),
    ("config3_llama3_8b_b1", 4096, 14336, 4, 1),
    ("config3_llama3_8b_b8", 4096, 14336, 4, 8),
]


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_23225_b200.build import build
    build()


@pytest.mark.parametrize("name,d,h,n_m,B", FULL)
def test_full_size_sampled_columns(name, d, h, n_m, B):
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    inp = make_inputs(0, B=B, d=d, h=h, n_m=n_m, dtype="bf16")
    x, Wt = to_device(inp, "bf16")
    packed_np = mglu_pack_masks_host(inp["bits"])
    packed = torch.from_numpy(packed_np).cuda()
    layer = Mglu(d, h, n_m, act="swish", dtype="bf16")
    y = layer.forward(x, Wt, packed).float().cpu().numpy().astype(np.float64)
    assert layer.last_path() == ("mma" if B <= 4 else "tcrow")     # AUTO crossovers
    rng = np.random.default_rng(1)
    cols = np.unique(np.concatenate([[0, 1, h // 2, h - 2, h - 1], rng.choice(h, 384, replace=False)]))
    xo, Wo = oracle_inputs(inp, "bf16")
    o = oracle()
    ref = o.forward(xo, Wo[cols], cols, o.pack(inp["bits"]), n_m, 1)   # oracle packs the bits itself
    err = normwise_err(y[:, cols], ref)
    assert err <= TIGHT["bf16"], (name, err)
    assert np.all(np.isfinite(y))


@pytest.mark.parametrize("n_m", [1, 2, 4, 8])
def test_config5_shape_sampled(n_m):
    """Config 5 shapes (d=8192, h=28672) at B=1 for every n_m.  Inputs are drawn on the device
    (synth.random_packed_codes: i.i.d. Bernoulli(0.5) code bits) and the sampled rows copied to
    the host for the oracle, which decodes them with its own unpacker."""
    from paper_2506_23225_b200.mglu import Mglu
    from synth import random_packed_codes
    d, h = 8192, 28672
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(1, d, device="cuda", generator=g).to(torch.bfloat16)
    Wt = ((torch.rand(h, d, device="cuda", generator=g) * 2 - 1) / d ** 0.5).to(torch.bfloat16)
    packed = random_packed_codes(7 + n_m, h, d, n_m, device="cuda")
    layer = Mglu(d, h, n_m, act="swish", dtype="bf16")
    y = layer.forward(x, Wt, packed).float().cpu().numpy().astype(np.float64)
    rng = np.random.default_rng(n_m)
    cols = np.sort(rng.choice(h, 256, replace=False))
    from oracle import decode_bf16
    xo = decode_bf16(x.view(torch.int16).cpu().numpy().view(np.uint16))
    Wo = decode_bf16(Wt[torch.from_numpy(cols).cuda()].view(torch.int16).cpu().numpy().view(np.uint16))
    ref = oracle().forward(xo, Wo, cols, packed.cpu().numpy(), n_m, 1)
    assert normwise_err(y[:, cols], ref) <= TIGHT["bf16"]


def test_full_size_one_hot_decode():
    """Bit-exact decode at the config-3 shape through the bench kernel: Wt = 1, x one-hot at
    sampled k, sigmoid -> y[j] = (n_m - popcount(c[j,k])) / 2 exactly, all 14336 rows."""
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    d, h, n_m = 4096, 14336, 4
    inp = make_inputs(3, B=1, d=d, h=h, n_m=n_m, dtype="bf16")
    packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
    Wt = torch.ones(h, d, device="cuda", dtype=torch.bfloat16)
    layer = Mglu(d, h, n_m, act="sigmoid", dtype="bf16")
    pop = inp["bits"].sum(axis=0)
    ks = [0, 1, 7, 8, 15, 16, 63, 64, 255, 1000, 2047, 2048, 4030, 4095, 17, 3333]
    for k0 in range(0, len(ks), 8):
        kk = ks[k0:k0 + 8]
        x = torch.zeros(len(kk), d, device="cuda", dtype=torch.bfloat16)
        x[torch.arange(len(kk)), torch.tensor(kk)] = 1.0
        y = layer.forward(x, Wt, packed).float().cpu().numpy()
        np.testing.assert_array_equal(y, (n_m - pop[:, kk].T) / 2.0)


PREFILL_FULL = [  # (name, d, h, n_m, B): the tensor-core workloads bench.py times, AUTO dispatch
    ("config4_prefill", 8192, 28672, 4, 4096),
    ("config5_b2048_nm8", 8192, 28672, 8, 2048),
    ("config5_b2048_nm1", 8192, 28672, 1, 2048),
    ("config3_b64", 4096, 14336, 4, 64),
    ("config3_b16", 4096, 14336, 4, 16),
]


@pytest.mark.parametrize("name,d,h,n_m,B", PREFILL_FULL)
def test_full_size_tensor_core_sampled(name, d, h, n_m, B):
    """BASELINE configs 3 (B = 16, 64), 4 and 5 (B = 2048) at full size through AUTO (tcgen05 tile
    GEMM / stream-K GEMV), device-drawn inputs as bench.py draws them; the oracle computes 48 sampled
    tokens x 96 sampled output columns one by one (its own unpacker on the sampled rows)."""
    from oracle import decode_bf16
    from paper_2506_23225_b200.mglu import Mglu
    from synth import random_packed_codes
    g = torch.Generator(device="cuda").manual_seed(11)
    x = torch.randn(B, d, device="cuda", generator=g).to(torch.bfloat16)
    Wt = ((torch.rand(h, d, device="cuda", generator=g) * 2 - 1) / d ** 0.5).to(torch.bfloat16)
    packed = random_packed_codes(13 + n_m, h, d, n_m, device="cuda")
    layer = Mglu(d, h, n_m, act="swish", dtype="bf16")
    y = layer.forward(x, Wt, packed)
    torch.cuda.synchronize()
    wide = h >= torch.cuda.get_device_properties(0).multi_processor_count * 64
    want = "tcrow" if (5 <= B <= 32 and n_m <= 4 and wide) else ("tcdec" if B <= 16 else "tcgen05")
    assert layer.last_path() == want                               # AUTO crossovers
    rng = np.random.default_rng(B + n_m)
    toks = np.unique(np.concatenate([[0, B - 1], rng.choice(B, min(B, 46), replace=False)]))
    cols = np.unique(np.concatenate([[0, 127, 128, h - 1], rng.choice(h, 92, replace=False)]))
    ys = y[torch.from_numpy(toks).cuda()][:, torch.from_numpy(cols).cuda()].float().cpu().numpy().astype(np.float64)
    xo = decode_bf16(x[torch.from_numpy(toks).cuda()].view(torch.int16).cpu().numpy().view(np.uint16))
    Wo = decode_bf16(Wt[torch.from_numpy(cols).cuda()].view(torch.int16).cpu().numpy().view(np.uint16))
    ref = oracle().forward(xo, Wo, cols, packed.cpu().numpy(), n_m, 1)
    assert normwise_err(ys, ref) <= TIGHT["bf16"], name
    del x, Wt, packed, y
    torch.cuda.empty_cache()
