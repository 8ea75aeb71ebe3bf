"""GPU parity of the decode-regime tcgen05 kernel (MGLU_PATH_TCDEC: persistent, stream-K balanced
masked GEMV, SURVEY rows a2-a7 for 1 <= B <= 64) against the CPU oracle on identical seeded
inputs.

The shapes are chosen to exercise the stream-K decomposition: tiles cut by one, two and many CTA
range boundaries (small h with large d spreads one 128-row tile over dozens of CTAs, whose
partials the owner sums in CTA order), ragged last tiles (h % 128 != 0), every token tile
(16 / 32 / 64) with ragged token counts, and every n_m."""
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


SHAPES = [  # (d, h, B)
    (64, 128, 1),        # one unit, one CTA
    (128, 200, 3),       # two ragged tiles
    (4096, 300, 1),      # 3 tiles x 64 units over 148 CTAs: ~50 contributors per owner
    (2048, 1000, 8),     # 8 tiles, each cut once or twice
    (1024, 4000, 16),    # 32 tiles (fewer units than two per CTA)
    (4096, 2944, 17),    # BN = 32, ragged tokens
    (1984, 640, 5),      # d % 128 == 64: a final half unit of zero-filled boxes
    (512, 9000, 33),     # BN = 64, many tiles per CTA, ragged last tile
    (256, 20000, 64),    # BN = 64, full token tile
]


@pytest.mark.parametrize("n_m", [1, 2, 4, 8])
@pytest.mark.parametrize("d,h,B", SHAPES)
def test_tcdec_shapes(n_m, d, h, B):
    inp = make_inputs(7000 + 17 * n_m + d + h + B, B=B, d=d, h=h, n_m=n_m, dtype="bf16")
    from paper_2506_23225_b200.mglu import MgluError, MGLU_ERR_UNSUPPORTED
    if (d // 32 * n_m) % 4 or (n_m == 8 and B > 32):
        with pytest.raises(MgluError) as e:
            gpu_forward(inp, "bf16", n_m, "swish", path="tcdec")
        assert e.value.status == MGLU_ERR_UNSUPPORTED
        return
    y, used = gpu_forward(inp, "bf16", n_m, "swish", path="tcdec")
    assert used == "tcdec"
    ref = oracle_forward(inp, "bf16", n_m, "swish")
    err = normwise_err(y, ref)
    assert err <= TOL["bf16"] and err <= TIGHT["bf16"], err


@pytest.mark.parametrize("act", ["identity", "swish", "gelu", "relu", "sigmoid"])
def test_tcdec_activations(act):
    inp = make_inputs(91, B=5, d=1024, h=700, n_m=4, dtype="bf16")
    y, _ = gpu_forward(inp, "bf16", 4, act, path="tcdec")
    assert normwise_err(y, oracle_forward(inp, "bf16", 4, act)) <= TIGHT["bf16"]


@pytest.mark.parametrize("n_m", [1, 2, 4, 8])
def test_tcdec_one_hot_bit_exact(n_m):
    """Wt = 1 and x one-hot (token b at column k0 + b, 16 tokens per call, every k covered): with
    sigmoid g every accumulator is a small integer, so y[b][j] = (n_m - popcount(c[j, k0 + b])) / 2
    exactly -- the mask decode of every (row, column) checked bit-exactly through this kernel,
    including rows of tiles finished by the stream-K fix-up."""
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    d, h = 1024, 200
    inp = make_inputs(71 + n_m, B=1, d=d, h=h, n_m=n_m, dtype="bf16")
    bits = inp["bits"]
    packed = torch.from_numpy(mglu_pack_masks_host(bits)).cuda()
    Wt = torch.ones(h, d, device="cuda", dtype=torch.bfloat16)
    eye = torch.eye(d, device="cuda", dtype=torch.bfloat16)
    layer = Mglu(d, h, n_m, act="sigmoid", dtype="bf16", path="tcdec")
    want = (n_m - bits.sum(axis=0).T) / 2.0                        # [d][h]
    for k0 in range(0, d, 16):
        y = layer.forward(eye[k0:k0 + 16].contiguous(), Wt, packed).float().cpu().numpy()
        assert layer.last_path() == "tcdec"
        np.testing.assert_array_equal(y, want[k0:k0 + 16])


def test_tcdec_all_ones_and_zeros():
    inp = make_inputs(3, B=4, d=2048, h=500, n_m=4, dtype="bf16", density="ones")
    y, _ = gpu_forward(inp, "bf16", 4, "swish", path="tcdec")
    assert np.all(y == 0.0)
    inp = make_inputs(4, B=9, d=2048, h=500, n_m=2, dtype="bf16", density="zeros")
    y, _ = gpu_forward(inp, "bf16", 2, "sigmoid", path="tcdec")
    x, Wt = oracle_inputs(inp, "bf16")
    assert normwise_err(y, (2 / 2) * x @ Wt.T) <= TIGHT["bf16"]


def test_tcdec_deterministic_back_to_back_and_graph():
    """Repeats are bit-identical (fixed fix-up order); dependent PDL launches (the second reads the
    first's output as x) and CUDA-graph replays see re-armed flags every call."""
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    d = h = 4096
    inp = make_inputs(12, B=2, d=d, h=h, n_m=4, dtype="bf16")
    x, Wt = to_device(inp, "bf16")
    packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
    layer = Mglu(d, h, 4, act="identity", dtype="bf16", path="tcdec")
    y0 = layer.forward(x, Wt, packed).clone()
    for _ in range(3):
        assert torch.equal(layer.forward(x, Wt, packed), y0)
    y1 = layer.forward(x, Wt, packed)
    y2 = layer.forward(y1, Wt, packed)
    torch.cuda.synchronize()
    assert torch.equal(y2, layer.forward(y1.clone(), Wt, packed))
    s = torch.cuda.Stream()
    out = torch.empty_like(y0)
    call = layer.bind(x, Wt, packed, out, stream=s)
    with torch.cuda.stream(s):
        call()
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            call()
            call()
    for _ in range(3):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, y0)


def test_tcdec_matches_mma_path_sampled_full_size():
    """Config 3 at B = 1 and 8 through TCDEC agrees with the oracle on sampled columns."""
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    from tests.helpers import oracle
    d, h, n_m = 4096, 14336, 4
    for B in (1, 8):
        inp = make_inputs(0, B=B, d=d, h=h, n_m=n_m, dtype="bf16")
        x, Wt = to_device(inp, "bf16")
        packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
        layer = Mglu(d, h, n_m, act="swish", dtype="bf16", path="tcdec")
        y = layer.forward(x, Wt, packed).float().cpu().numpy().astype(np.float64)
        rng = np.random.default_rng(2)
        cols = np.unique(np.concatenate([[0, 127, 128, h - 1], rng.choice(h, 256, replace=False)]))
        xo, Wo = oracle_inputs(inp, "bf16")
        o = oracle()
        ref = o.forward(xo, Wo[cols], cols, o.pack(inp["bits"]), n_m, 1)
        assert normwise_err(y[:, cols], ref) <= TIGHT["bf16"]


# row split (MGLU_PATH_TCROW): every CTA owns whole tiles of tr_base or tr_base + 1 rows over all of d
ROW_SHAPES = [  # (d, h, B)
    (4096, 9472, 1),     # exactly 64 rows per CTA
    (1024, 9601, 5),     # 64 / 65-row tiles (two TMA box heights)
    (512, 19000, 24),    # two tiles per CTA, 64 / 65 rows
    (2048, 14336, 40),   # the config-3 split (96 / 97 rows), BN = 64, ragged tokens
    (256, 38000, 64),    # three tiles per CTA, full token tile
]


@pytest.mark.parametrize("n_m", [1, 2, 4, 8])
@pytest.mark.parametrize("d,h,B", ROW_SHAPES)
def test_tcdec_row_split_shapes(n_m, d, h, B):
    from paper_2506_23225_b200.mglu import MgluError, MGLU_ERR_UNSUPPORTED
    inp = make_inputs(9100 + 13 * n_m + d + h + B, B=B, d=d, h=h, n_m=n_m, dtype="bf16")
    if n_m == 8 and B > 32:
        with pytest.raises(MgluError) as e:
            gpu_forward(inp, "bf16", n_m, "swish", path="tcrow")
        assert e.value.status == MGLU_ERR_UNSUPPORTED
        return
    y, used = gpu_forward(inp, "bf16", n_m, "swish", path="tcrow")
    assert used == "tcrow"
    rng = np.random.default_rng(h + B)
    cols = np.unique(np.concatenate([[0, 63, 64, 65, 96, 97, h // 2, h - 2, h - 1], rng.choice(h, 300, replace=False)]))
    ref = oracle_forward(inp, "bf16", n_m, "swish", cols=cols)
    assert normwise_err(y[:, cols], ref) <= TIGHT["bf16"]


@pytest.mark.parametrize("n_m", [1, 4, 8])
def test_tcdec_row_split_one_hot_bit_exact(n_m):
    """The one-hot decode probe through the row split (MGLU_PATH_TCROW): every (row, column) of a layer with 64- and
    65-row tiles, bit-exact."""
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    d, h = 256, 9601
    inp = make_inputs(171 + n_m, B=1, d=d, h=h, n_m=n_m, dtype="bf16")
    bits = inp["bits"]
    packed = torch.from_numpy(mglu_pack_masks_host(bits)).cuda()
    Wt = torch.ones(h, d, device="cuda", dtype=torch.bfloat16)
    eye = torch.eye(d, device="cuda", dtype=torch.bfloat16)
    layer = Mglu(d, h, n_m, act="sigmoid", dtype="bf16", path="tcrow")
    want = (n_m - bits.sum(axis=0).T) / 2.0                        # [d][h]
    for k0 in range(0, d, 16):
        y = layer.forward(eye[k0:k0 + 16].contiguous(), Wt, packed).float().cpu().numpy()
        np.testing.assert_array_equal(y, want[k0:k0 + 16])


def test_tcdec_row_split_shard_bit_identical():
    """P8 on the row split: a row's k-order does not depend on which CTA or tile holds it, so an
    h-shard (pointer offsets into Wt and the codes) reproduces the unsharded output bit for bit."""
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    d, h, n_m, B = 2048, 19200, 4, 8
    inp = make_inputs(44, B=B, d=d, h=h, n_m=n_m, dtype="bf16")
    x, Wt = to_device(inp, "bf16")
    packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
    full = Mglu(d, h, n_m, act="swish", dtype="bf16", path="tcrow").forward(x, Wt, packed)
    row_bytes = d * n_m // 8
    for lo, hi in ((0, 9600), (9600, 19200), (4800, 14400)):
        part = Mglu(d, hi - lo, n_m, act="swish", dtype="bf16", path="tcrow")
        y = part.forward(x, Wt[lo:hi], packed[lo * row_bytes:hi * row_bytes])
        assert torch.equal(y, full[:, lo:hi]), (lo, hi)
