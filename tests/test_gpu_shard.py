"""Column-shard parity on one GPU: G handles Mglu(d, h/G) each run on their row
slice (pointer offsets into Wt and the packed codes, paper_2506_23225_b200.shard) and the
concatenated outputs equal the unsharded layer (P8) -- bit-identically on the tcgen05 tile
GEMM and on the row-split tcgen05 GEMV (MGLU_PATH_TCROW, AUTO for 5 <= B <= 32): on both a row's
k-order is unit by unit, k16 step by k16 step, whatever tile or CTA holds it.  The HMMA decode
kernel (AUTO for B <= 4) re-splits a stage's columns over 2..16 warps by the CTA's row count for
throughput, so its shards are held to the bf16 bound against the oracle instead (R21)."""
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


def _sharded(x, Wt, packed, n_m, G, path="auto"):
    from paper_2506_23225_b200.mglu import Mglu
    from paper_2506_23225_b200.shard import shard_bounds, shard_layer
    h, d = Wt.shape
    outs = []
    for r in range(G):
        W_r, p_r = shard_layer(Wt, packed, n_m, G, r)
        lo, hi = shard_bounds(h, G, r)
        layer = Mglu(d, hi - lo, n_m, act="swish", dtype="bf16", path=path)
        outs.append(layer.forward(x, W_r, p_r))
        layer.close()
    return torch.cat(outs, dim=1)


@pytest.mark.parametrize("G", [2, 4, 8])
def test_tile_path_shards_bit_identical(G):
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    d, h, n_m, B = 1024, 1024, 4, 200
    inp = make_inputs(40 + G, B=B, d=d, h=h, n_m=n_m, dtype="bf16")
    x, Wt = to_device(inp, "bf16")
    packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
    full = Mglu(d, h, n_m, act="swish", dtype="bf16", path="tcgen05").forward(x, Wt, packed)
    assert torch.equal(_sharded(x, Wt, packed, n_m, G, path="tcgen05"), full)


@pytest.mark.parametrize("G", [2, 4, 8])
def test_decode_shards_match_oracle(G):
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    d, h, n_m, B = 4096, 14336, 4, 1
    inp = make_inputs(0, B=B, d=d, h=h, n_m=n_m, dtype="bf16")
    x, Wt = to_device(inp, "bf16")
    packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
    y = _sharded(x, Wt, packed, n_m, G).float().cpu().numpy().astype(np.float64)
    full = Mglu(d, h, n_m, act="swish", dtype="bf16").forward(x, Wt, packed).float().cpu().numpy()
    rng = np.random.default_rng(G)
    # every shard boundary and a random sample
    bounds = [r * h // G for r in range(G)]
    cols = np.unique(np.concatenate([bounds, np.array(bounds[1:]) - 1, [h - 1], rng.choice(h, 256, replace=False)]))
    xo, Wo = oracle_inputs(inp, "bf16")
    o = oracle()
    ref = o.forward(xo, Wo[cols], cols, o.pack(inp["bits"]), n_m, 1)
    assert normwise_err(y[:, cols], ref) <= TIGHT["bf16"]
    assert normwise_err(y, full) <= TIGHT["bf16"]


@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("B", [1, 8, 40])
def test_row_split_decode_shards_bit_identical(G, B):
    """Config 3 (d = 4096, h = 14336, n_m = 4) through the row-split GEMV: every G-shard's output
    equals the unsharded layer's columns bit for bit."""
    from paper_2506_23225_b200.mglu import Mglu
    from synth import random_packed_codes
    d, h, n_m = 4096, 14336, 4
    g = torch.Generator(device="cuda").manual_seed(100 + G + B)
    x = torch.randn(B, d, device="cuda", generator=g).to(torch.bfloat16)
    Wt = ((torch.rand(h, d, device="cuda", generator=g) * 2 - 1) / d ** 0.5).to(torch.bfloat16)
    packed = random_packed_codes(21 + G, h, d, n_m, device="cuda")
    full = Mglu(d, h, n_m, act="swish", dtype="bf16", path="tcrow").forward(x, Wt, packed)
    assert torch.equal(_sharded(x, Wt, packed, n_m, G, path="tcrow"), full)
