"""Row f1 on the GPU: the dense projection (n_m = 0 handle, the FFN down-projection W_o) and the
SwiMGLU FFN block, single GPU and tensor-parallel G = 2/4/8 (handles on one GPU, the all-reduce
replaced by a host sum), against the binary64 oracle (Eq. 3)."""
import numpy as np
import pytest
import torch

from tests.helpers import TIGHT, TOL, make_inputs, normwise_err, oracle_inputs, to_device

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


@pytest.mark.parametrize("K,N,B", [(128, 200, 1), (1792, 4096, 1), (14336, 4096, 2), (1792, 4096, 8), (4096, 333, 8), (256, 64, 3)])
def test_dense_projection(K, N, B):
    from oracle import dense_np
    from paper_2506_23225_b200.mglu import Mglu
    g = torch.Generator().manual_seed(K + N + B)
    x = torch.randn(B, K, generator=g).to(torch.bfloat16)
    W = _wo(K + N, N, K)
    layer = Mglu(K, N, 0, dtype="bf16")
    y = layer.forward(x.cuda(), W.cuda(), None)
    torch.cuda.synchronize()
    assert layer.last_path() == "mma"
    ref = dense_np(x.float().numpy(), W.float().numpy())
    err = normwise_err(y.float().cpu().numpy().astype(np.float64), ref)
    assert err <= TIGHT["bf16"], err


def test_dense_projection_refuses_other_paths():
    from paper_2506_23225_b200.mglu import Mglu, MgluError, MGLU_ERR_UNSUPPORTED
    layer = Mglu(256, 128, 0, dtype="bf16")
    x = torch.zeros(9, 256, dtype=torch.bfloat16, device="cuda")      # B > 8
    with pytest.raises(MgluError) as e:
        layer.forward(x, torch.zeros(128, 256, dtype=torch.bfloat16, device="cuda"), None)
    assert e.value.status == MGLU_ERR_UNSUPPORTED


@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_ffn_tensor_parallel(G):
    from oracle import ACT_SWISH, ffn_forward_np
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    from paper_2506_23225_b200.shard import ffn_forward_tp, shard_bounds, shard_down, shard_layer
    d, h, n_m, B = 1024, 4096, 4, 2
    inp = make_inputs(60 + G, B=B, d=d, h=h, n_m=n_m, dtype="bf16")
    x, Wt = to_device(inp, "bf16")
    packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
    Wo = _wo(G, d, h).cuda()
    total = torch.zeros(B, d, dtype=torch.float32, device="cuda")
    for r in range(G):                                   # G ranks on one GPU; host-side sum = all-reduce
        lo, hi = shard_bounds(h, G, r)
        W_g, p_g = shard_layer(Wt, packed, n_m, G, r)
        up = Mglu(d, hi - lo, n_m, act="swish", dtype="bf16")
        down = Mglu(hi - lo, d, 0, dtype="bf16")
        total += ffn_forward_tp(up, down, x, W_g, p_g, shard_down(Wo, G, r))
    xo, Wto = oracle_inputs(inp, "bf16")
    ref = ffn_forward_np(xo, Wto, inp["bits"], Wo.float().cpu().numpy().astype(np.float64), ACT_SWISH)
    err = normwise_err(total.cpu().numpy().astype(np.float64), ref)
    assert err <= TOL["bf16"] and err <= TIGHT["bf16"], err
