"""GPU parity: the CUDA path through the C ABI vs the CPU oracle on identical seeded inputs.

Tolerances (north_star; normwise reading R10): bf16 1e-2, fp32 1e-5, plus a tighter regression
band.  Mask decoding is checked bit-exactly through the real kernels (one-hot probes)."""
import numpy as np
import pytest
import torch

from tests.helpers import (TIGHT, TOL, gpu_forward, make_inputs, normwise_err, oracle,
                           oracle_forward, oracle_inputs, to_device)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_23225_b200.build import build
    build()


# ---------------------------------------------------------------- config 1 (tiny, fp32)
@pytest.mark.parametrize("seed", range(5))
def test_tiny_config_f32(seed):
    """BASELINE config 1: d=64, h=128, n_m=1, B=1, fp32, Swish -> 1e-5."""
    inp = make_inputs(seed, B=1, d=64, h=128, n_m=1, dtype="f32")
    y, path = gpu_forward(inp, "f32", 1, "swish")
    ref = oracle_forward(inp, "f32", 1, "swish")
    assert path == "simt"
    err = normwise_err(y, ref)
    assert err <= TOL["f32"] and err <= TIGHT["f32"], err


# ---------------------------------------------------------------- bf16 shapes, both decode regimes
SHAPES = [  # (d, h, B) -- several tiles, ragged row tails, B up to the MMA group
    (64, 16, 1), (256, 100, 1), (512, 1000, 3), (1024, 333, 8), (2048, 160, 5), (4096, 300, 2),
]


@pytest.mark.parametrize("n_m", [1, 2, 4, 8])
@pytest.mark.parametrize("d,h,B", SHAPES)
@pytest.mark.parametrize("path", ["mma", "simt"])
def test_bf16_shapes(n_m, d, h, B, path):
    inp = make_inputs(1000 + n_m * 7 + d + h + B, B=B, d=d, h=h, n_m=n_m, dtype="bf16")
    if path == "mma" and (d % 128 or (n_m >= 4 and B > 4)):
        # the MMA path tiles rows in 128-column code blocks (16 * n_m bytes): d % 128 == 0; with
        # n_m >= 4 it serves one token group (B <= 4), larger batches go to the tcgen05 paths
        from paper_2506_23225_b200.mglu import MgluError, MGLU_ERR_UNSUPPORTED
        with pytest.raises(MgluError) as e:
            gpu_forward(inp, "bf16", n_m, "swish", path=path)
        assert e.value.status == MGLU_ERR_UNSUPPORTED
        return
    y, used = gpu_forward(inp, "bf16", n_m, "swish", path=path)
    assert used == path
    ref = oracle_forward(inp, "bf16", n_m, "swish")
    err = normwise_err(y, ref)
    assert err <= TIGHT["bf16"], err


@pytest.mark.parametrize("act", ["identity", "swish", "gelu", "relu", "sigmoid"])
@pytest.mark.parametrize("path", ["mma", "simt"])
def test_activations(act, path):
    inp = make_inputs(77, B=4, d=512, h=200, n_m=4, dtype="bf16")
    y, _ = gpu_forward(inp, "bf16", 4, act, path=path)
    ref = oracle_forward(inp, "bf16", 4, act)
    assert normwise_err(y, ref) <= TIGHT["bf16"]


@pytest.mark.parametrize("act", ["identity", "swish", "gelu", "relu", "sigmoid"])
@pytest.mark.parametrize("n_m", [1, 2, 4, 8])
def test_f32_simt_all(act, n_m):
    inp = make_inputs(5 + n_m, B=3, d=128, h=96, n_m=n_m, dtype="f32")
    y, _ = gpu_forward(inp, "f32", n_m, act)
    ref = oracle_forward(inp, "f32", n_m, act)
    assert normwise_err(y, ref) <= TOL["f32"]


@pytest.mark.parametrize("seed", range(5))
@pytest.mark.parametrize("density", [0.45, 0.55])
def test_mask_density_sensitivity(seed, density):
    """Learned-mask range 45-55 %."""
    inp = make_inputs(seed, B=1, d=1024, h=256, n_m=4, dtype="bf16", density=density)
    y, _ = gpu_forward(inp, "bf16", 4, "swish", path="mma")
    assert normwise_err(y, oracle_forward(inp, "bf16", 4, "swish")) <= TIGHT["bf16"]


# ---------------------------------------------------------------- partial sums (Alg. 1's z)
@pytest.mark.parametrize("n_m", [1, 2, 4, 8])
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_partials_vs_independent_value_stream(n_m, dtype):
    """z[gate_i] and z[value_i] vs the oracle, whose value stream is computed from Mbar
    independently (complementarity P2 checked across the two implementations)."""
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    inp = make_inputs(11 + n_m, B=2, d=256, h=72, n_m=n_m, dtype=dtype)
    x, Wt = to_device(inp, dtype)
    packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
    layer = Mglu(256, 72, n_m, act="swish", dtype=dtype)
    z = layer.forward_partials(x, Wt, packed).cpu().numpy().astype(np.float64)
    _, zr, tr = oracle_forward(inp, dtype, n_m, "swish", want_partials=True)
    for b in range(2):
        scale = np.max(np.abs(tr[b]))
        assert np.max(np.abs(z[b] - zr[b])) / scale <= 1e-5
        np.testing.assert_allclose(z[b, :n_m] + z[b, n_m:], np.repeat(tr[b][None], n_m, 0),
                                   rtol=0, atol=1e-5 * scale)


@pytest.mark.parametrize("n_m", [1, 2, 4, 8])
@pytest.mark.parametrize("path,B", [("mma", 1), ("mma", 3), ("tcdec", 1), ("tcdec", 9), ("tcrow", 1), ("tcrow", 17), ("tcgen05", 2), ("tcgen05", 70)])
def test_fast_path_partials_vs_independent_value_stream(n_m, path, B):
    """The fast kernels' own value streams (each kernel's epilogue writes s_i = (t + u_i) / 2 and
    t - s_i instead of y when the partials entry selects it): checked against the oracle's gate and
    INDEPENDENTLY computed value streams (P2 across implementations, rows a5/a6 on every path)."""
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    d, h = 1024, 300                                   # several tiles, ragged rows
    inp = make_inputs(400 + 13 * n_m + B, B=B, d=d, h=h, n_m=n_m, dtype="bf16")
    x, Wt = to_device(inp, "bf16")
    packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
    layer = Mglu(d, h, n_m, act="swish", dtype="bf16", path=path)
    z = layer.forward_partials(x, Wt, packed).cpu().numpy().astype(np.float64)
    assert layer.last_path() == path
    _, zr, tr = oracle_forward(inp, "bf16", n_m, "swish", want_partials=True)
    for b in range(B):
        scale = np.max(np.abs(tr[b]))
        # fp32 accumulation of exact bf16 products, order differing from the oracle's: ~1e-6
        assert np.max(np.abs(z[b] - zr[b])) / scale <= 1e-5, (b, np.max(np.abs(z[b] - zr[b])) / scale)


# ---------------------------------------------------------------- bit-exact decoding (P7)
@pytest.mark.parametrize("n_m", [1, 2, 4, 8])
def test_one_hot_partials_bit_exact(n_m):
    """Wt = 1, x one-hot at k: gate_i[j] = M_i[j,k] and value_i[j] = 1 - M_i[j,k] exactly."""
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    d, h = 64, 40
    inp = make_inputs(21, B=1, d=d, h=h, n_m=n_m, dtype="f32")
    bits = inp["bits"]
    packed = torch.from_numpy(mglu_pack_masks_host(bits)).cuda()
    Wt = torch.ones(h, d, device="cuda")
    x = torch.eye(d, device="cuda")        # B = d tokens, token k one-hot at k
    layer = Mglu(d, h, n_m, act="identity", dtype="f32")
    z = layer.forward_partials(x, Wt, packed).cpu().numpy()
    for k in range(d):
        np.testing.assert_array_equal(z[k, :n_m], bits[:, :, k].astype(np.float32))
        np.testing.assert_array_equal(z[k, n_m:], 1.0 - bits[:, :, k].astype(np.float32))


@pytest.mark.parametrize("n_m", [1, 2, 4, 8])
@pytest.mark.parametrize("path", ["mma", "simt"])
def test_one_hot_forward_bit_exact(n_m, path):
    """Through the fused bf16 forward: Wt = 1, x one-hot at k, sigmoid g gives
    y[j] = (n_m - popcount(c[j,k])) / 2 exactly (each mask: bit 1 -> sigmoid(1)*0, bit 0 ->
    sigmoid(0)*1).  Eight (or four) tokens per call, every k of d = 256 covered."""
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    d, h = 256, 200
    inp = make_inputs(31 + n_m, B=1, d=d, h=h, n_m=n_m, dtype="bf16")
    bits = inp["bits"]
    packed = torch.from_numpy(mglu_pack_masks_host(bits)).cuda()
    Wt = torch.ones(h, d, device="cuda", dtype=torch.bfloat16)
    layer = Mglu(d, h, n_m, act="sigmoid", dtype="bf16", path=path)
    pop = bits.sum(axis=0)                                         # [h][d]
    T = 4 if (path == "mma" and n_m >= 4) else 8                   # (one MMA token group for n_m >= 4)
    for k0 in range(0, d, T):
        x = torch.zeros(T, d, device="cuda", dtype=torch.bfloat16)
        x[torch.arange(T), torch.arange(k0, k0 + T)] = 1.0
        y = layer.forward(x, Wt, packed).float().cpu().numpy()
        want = (n_m - pop[:, k0:k0 + T].T) / 2.0
        np.testing.assert_array_equal(y, want)


# ---------------------------------------------------------------- special masks, empty, ragged
@pytest.mark.parametrize("path", ["mma", "simt"])
def test_all_ones_mask_zero(path):
    inp = make_inputs(3, B=2, d=256, h=64, n_m=4, dtype="bf16", density="ones")
    y, _ = gpu_forward(inp, "bf16", 4, "swish", path=path)
    assert np.all(y == 0.0)


@pytest.mark.parametrize("path", ["mma", "simt"])
def test_all_zeros_mask_plain_projection(path):
    inp = make_inputs(4, B=2, d=256, h=64, n_m=2, dtype="bf16", density="zeros")
    y, _ = gpu_forward(inp, "bf16", 2, "sigmoid", path=path)
    x, Wt = oracle_inputs(inp, "bf16")
    ref = (2 / 2) * x @ Wt.T                     # (n_m/2) x W
    assert normwise_err(y, ref) <= TIGHT["bf16"]


def test_empty_batch():
    from paper_2506_23225_b200.mglu import Mglu, mglu_forward
    layer = Mglu(64, 32, 2, dtype="bf16")
    x = torch.zeros(1, 64, device="cuda", dtype=torch.bfloat16)
    Wt = torch.zeros(32, 64, device="cuda", dtype=torch.bfloat16)
    packed = torch.zeros(32 * 64 * 2 // 8, device="cuda", dtype=torch.uint8)
    out = torch.full((1, 32), 7.0, device="cuda", dtype=torch.bfloat16)
    mglu_forward(layer.handle, x, 0, Wt, packed, out)
    torch.cuda.synchronize()
    assert layer.last_launch_count() == 0
    assert torch.all(out == 7.0)


@pytest.mark.parametrize("path", ["mma", "simt"])
def test_deterministic_repeats(path):
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    inp = make_inputs(9, B=4, d=1024, h=777, n_m=4, dtype="bf16")
    x, Wt = to_device(inp, "bf16")
    packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
    layer = Mglu(1024, 777, 4, dtype="bf16", path=path)
    y0 = layer.forward(x, Wt, packed).clone()
    for _ in range(5):
        assert torch.equal(layer.forward(x, Wt, packed), y0)


# ---------------------------------------------------------------- packing on the device
@pytest.mark.parametrize("n_m", [1, 2, 4, 8])
def test_device_pack_unpack(n_m):
    from paper_2506_23225_b200 import mglu as M
    from synth import make_logits
    inp = make_inputs(50 + n_m, B=1, d=128, h=48, n_m=n_m)
    bits = inp["bits"]
    dev = M.mglu_pack_masks_device(torch.from_numpy(bits).cuda()).cpu().numpy()
    np.testing.assert_array_equal(dev, M.mglu_pack_masks_host(bits))
    np.testing.assert_array_equal(dev, oracle().pack(bits))
    back = M.mglu_unpack_masks_device(torch.from_numpy(dev).cuda(), n_m, 48, 128).cpu().numpy()
    np.testing.assert_array_equal(back, bits)
    logits = make_logits(n_m, n_m, 48, 128)
    devl = M.mglu_pack_logits_device(torch.from_numpy(logits).cuda()).cpu().numpy()
    np.testing.assert_array_equal(devl, oracle().pack((logits > 0).astype(np.uint8)))


# ---------------------------------------------------------------- ABI errors on a live device
def test_abi_errors_live():
    from paper_2506_23225_b200 import mglu as M
    layer = M.Mglu(256, 64, 4, dtype="bf16")
    x = torch.zeros(9, 256, device="cuda", dtype=torch.bfloat16)
    Wt = torch.zeros(64, 256, device="cuda", dtype=torch.bfloat16)
    packed = torch.zeros(64 * 256 // 2, device="cuda", dtype=torch.uint8)
    layer.set_path("mma")
    with pytest.raises(M.MgluError) as e:
        layer.forward(x, Wt, packed)                  # B = 9 > 8 on the MMA path
    assert e.value.status == M.MGLU_ERR_UNSUPPORTED
    buf = torch.zeros(256 * 2 + 16, device="cuda", dtype=torch.uint8)
    mis = buf[2:2 + 512].view(torch.bfloat16)
    with pytest.raises(M.MgluError) as e:
        M.mglu_forward(layer.handle, mis, 1, Wt, packed, x)
    assert e.value.status == M.MGLU_ERR_MISALIGNED
    f32 = M.Mglu(256, 64, 4, dtype="f32", path="mma")
    with pytest.raises(M.MgluError) as e:
        f32.forward(x.float()[:1].contiguous(), Wt.float(), packed)
    assert e.value.status == M.MGLU_ERR_UNSUPPORTED


# ---------------------------------------------------------------- e2e host-buffer entry
def test_forward_host_matches_device():
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    inp = make_inputs(12, B=2, d=512, h=300, n_m=4, dtype="bf16")
    x, Wt = to_device(inp, "bf16")
    packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
    layer = Mglu(512, 300, 4, dtype="bf16")
    y = layer.forward(x, Wt, packed)
    xh = x.cpu().pin_memory()
    yh = torch.empty(2, 300, dtype=torch.bfloat16).pin_memory()
    layer.forward_host(xh, Wt, packed, yh)
    torch.cuda.synchronize()
    assert torch.equal(yh, y.cpu())


@pytest.mark.parametrize("pinned", [True, False])
@pytest.mark.parametrize("B,d,h", [(1, 4096, 14336), (3, 512, 300), (8, 1024, 1000)])
def test_forward_host_copy_paths(pinned, B, d, h):
    """mglu_forward_host's two copy paths: page-locked (device-mapped) buffers go through the
    PDL-chained copy kernels, pageable ones through cudaMemcpyAsync; both give the device result
    bit for bit, repeated back to back on one stream (the copy-in of call i+1 must not overtake the
    copy-out of call i)."""
    from paper_2506_23225_b200.mglu import Mglu
    from synth import random_packed_codes
    g = torch.Generator(device="cuda").manual_seed(B + d)
    x = torch.randn(B, d, device="cuda", generator=g).to(torch.bfloat16)
    Wt = ((torch.rand(h, d, device="cuda", generator=g) * 2 - 1) / d ** 0.5).to(torch.bfloat16)
    packed = random_packed_codes(B, h, d, 4, device="cuda")
    layer = Mglu(d, h, 4, dtype="bf16")
    xs = [torch.randn(B, d, generator=torch.Generator().manual_seed(k)).to(torch.bfloat16) for k in range(4)]
    want = [layer.forward(xk.cuda(), Wt, packed).cpu() for xk in xs]
    if pinned:
        xs = [xk.pin_memory() for xk in xs]
    outs = [torch.empty(B, h, dtype=torch.bfloat16) for _ in xs]
    if pinned:
        outs = [o.pin_memory() for o in outs]
    for xk, o in zip(xs, outs):
        layer.forward_host(xk, Wt, packed, o)
    torch.cuda.synchronize()
    for o, w in zip(outs, want):
        assert torch.equal(o, w)
