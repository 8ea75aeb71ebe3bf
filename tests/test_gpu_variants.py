"""GPU parity of the partial-mask ablation variants NG / NV / NM (row f3) on the MMA and
SIMT paths against the oracle's variant of Eq. 3 built from its independent streams."""
import numpy as np
import pytest
import torch

from tests.helpers import TIGHT, TOL, make_inputs, normwise_err, oracle, oracle_inputs, to_device

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_23225_b200.build import build
    build()


def _oracle_variant(inp, n_m, act_code, variant):
    from oracle import mglu_variant_from_streams
    xo, Wo = oracle_inputs(inp, "bf16")
    o = oracle()
    h = Wo.shape[0]
    _, z, t = o.forward(xo, Wo, np.arange(h), o.pack(inp["bits"]), n_m, act_code, want_partials=True)
    gate = np.transpose(z[:, :n_m, :], (1, 0, 2))
    value = np.transpose(z[:, n_m:, :], (1, 0, 2))
    return mglu_variant_from_streams(t, gate, value, act_code, variant)


@pytest.mark.parametrize("variant", ["no_gate_mask", "no_value_mask", "no_masks"])
@pytest.mark.parametrize("n_m,B,path", [(1, 1, "mma"), (4, 3, "mma"), (1, 10, "auto"), (2, 2, "simt"),
                                         (4, 7, "tcdec"), (2, 12, "tcrow"), (1, 100, "tcgen05"), (8, 70, "tcgen05")])
def test_variant_matches_oracle(variant, n_m, B, path):
    from oracle import VARIANTS
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    d, h = 1024, 500
    inp = make_inputs(1200 + n_m + B + VARIANTS[variant], B=B, d=d, h=h, n_m=n_m, dtype="bf16")
    x, Wt = to_device(inp, "bf16")
    packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
    layer = Mglu(d, h, n_m, act="swish", dtype="bf16", path=path)
    layer.set_variant(variant)
    y = layer.forward(x, Wt, packed)
    torch.cuda.synchronize()
    assert layer.last_path() == path or path == "auto"
    ref = _oracle_variant(inp, n_m, 1, VARIANTS[variant])
    err = normwise_err(y.float().cpu().numpy().astype(np.float64), ref)
    assert err <= TOL["bf16"] and err <= TIGHT["bf16"], err


def test_variant_reset():
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    from tests.helpers import oracle_forward
    d, h, n_m = 512, 256, 4
    inp = make_inputs(5, B=2, d=d, h=h, n_m=n_m, dtype="bf16")
    x, Wt = to_device(inp, "bf16")
    packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
    layer = Mglu(d, h, n_m, dtype="bf16", path="tcgen05")
    layer.set_variant("no_masks")
    layer.forward(x, Wt, packed)
    layer.set_variant("standard")
    y = layer.forward(x, Wt, packed)                      # back to Eq. 3
    assert normwise_err(y.float().cpu().numpy().astype(np.float64), oracle_forward(inp, "bf16", n_m, "swish")) <= TIGHT["bf16"]
