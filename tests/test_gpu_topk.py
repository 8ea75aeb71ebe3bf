"""GPU parity of the Top-K routed MGLU (Appendix B) through the C
ABI: the router (mglu_router_topk: fp32 logits, TopK with ties to the lowest index, softmax over the
kept logits) against the oracle's topk_gate, and the routed forward (mglu_forward_routed) against
the oracle's routed sum built from its independent per-mask gate/value streams -- on the MMA path
(which skips masks no token selected) and the SIMT path."""
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


def _router_weights(seed, n_m, d):
    g = torch.Generator().manual_seed(seed)
    return (torch.randn(n_m, d, generator=g) / d ** 0.5).to(torch.bfloat16)


def _oracle_routed(inp, n_m, act_code, G):
    from oracle import mglu_routed_from_partials
    xo, Wo = oracle_inputs(inp, "bf16")
    o = oracle()
    h = Wo.shape[0]
    _, z, _ = o.forward(xo, Wo, np.arange(h), o.pack(inp["bits"]), n_m, act_code, want_partials=True)
    gate = np.transpose(z[:, :n_m, :], (1, 0, 2))
    value = np.transpose(z[:, n_m:, :], (1, 0, 2))
    return mglu_routed_from_partials(gate, value, G, act_code)


LOGIT_TOL = 1e-4     # fp32 rounding of a d-term logit sum (d <= 4096, |l| = O(1)) -- generous


def _check_selection(g, l, g_ref, K):
    """The GPU takes TopK in fp32, so near ties (within LOGIT_TOL) may legitimately go either way.
    Every selection must be VALID: K entries, none of the unselected logits exceeds a selected one
    by more than LOGIT_TOL (in exact arithmetic), and the weights are the softmax of the oracle's
    logits over the selected set.  Where no near tie exists the set equals the oracle's."""
    sel = np.flatnonzero(g != 0)
    assert sel.size == K, (g, K)
    uns = np.setdiff1d(np.arange(l.size), sel)
    if uns.size:
        assert l[uns].max() <= l[sel].min() + LOGIT_TOL, (l, sel)
    e = np.exp(l[sel] - l[sel].max())
    np.testing.assert_allclose(g[sel], e / e.sum(), rtol=0, atol=2e-6)
    srt = np.sort(l)[::-1]
    if K == l.size or srt[K - 1] - srt[K] > LOGIT_TOL:
        np.testing.assert_array_equal(g != 0, g_ref != 0)


def test_router_near_ties_give_valid_selections():
    """Logits engineered into exact and near ties (equal router rows, rows differing in one
    low bit): whatever the GPU picks must be a valid TopK set with the matching softmax."""
    from oracle import router_logits, topk_gate
    from paper_2506_23225_b200.mglu import Mglu
    d, n_m, B = 512, 8, 16
    inp = make_inputs(77, B=B, d=d, h=128, n_m=n_m, dtype="bf16")
    x, _ = to_device(inp, "bf16")
    base = _router_weights(3, n_m, d)
    Wr = base.clone()
    Wr[1] = Wr[0]                                          # exact tie between logits 0 and 1
    Wr[3] = Wr[2]
    Wr[3, 5] = (Wr[3, 5].float() * (1 + 2 ** -7)).to(torch.bfloat16)   # near tie 2 vs 3
    xo, _ = oracle_inputs(inp, "bf16")
    l = router_logits(xo, Wr.float().numpy().astype(np.float64))
    layer = Mglu(d, 128, n_m, dtype="bf16")
    for K in (1, 2, 3, 4):
        G = layer.router_topk(x, Wr.cuda(), K).cpu().numpy()
        G_ref = topk_gate(l, K)
        for b in range(B):
            _check_selection(G[b], l[b], G_ref[b], K)


@pytest.mark.parametrize("n_m,K", [(4, 1), (4, 2), (8, 2), (8, 4), (8, 8)])
@pytest.mark.parametrize("B", [1, 3, 8])
def test_router_matches_oracle(n_m, K, B):
    from oracle import router_logits, topk_gate
    from paper_2506_23225_b200.mglu import Mglu
    d = 1024
    inp = make_inputs(300 + n_m + K + B, B=B, d=d, h=128, n_m=n_m, dtype="bf16")
    x, _ = to_device(inp, "bf16")
    Wr = _router_weights(7 + n_m, n_m, d)
    layer = Mglu(d, 128, n_m, dtype="bf16")
    G = layer.router_topk(x, Wr.cuda(), K).cpu().numpy()
    xo, _ = oracle_inputs(inp, "bf16")
    l = router_logits(xo, Wr.float().numpy().astype(np.float64))
    G_ref = topk_gate(l, K)
    for b in range(B):
        _check_selection(G[b], l[b], G_ref[b], K)
    assert np.allclose(G.sum(axis=1), 1.0, atol=1e-6)


@pytest.mark.parametrize("path", ["mma", "simt", "tcdec", "tcrow", "tcgen05"])
@pytest.mark.parametrize("n_m,K,B", [(4, 1, 1), (4, 2, 3), (8, 2, 1), (8, 3, 5), (8, 8, 8), (2, 1, 2), (8, 1, 2),
                                     (8, 4, 1), (8, 2, 2)])
def test_routed_forward_matches_oracle(path, n_m, K, B):
    from oracle import topk_gate
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    d, h = 2048, 700
    inp = make_inputs(500 + n_m * 10 + K + B, B=B, d=d, h=h, n_m=n_m, dtype="bf16")
    x, Wt = to_device(inp, "bf16")
    packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
    rng = np.random.default_rng(K + B)
    G = topk_gate(rng.standard_normal((B, n_m)), K)
    layer = Mglu(d, h, n_m, act="swish", dtype="bf16", path=path)
    if path == "mma" and n_m >= 4 and B > 4:         # one token group on the MMA path for n_m >= 4
        from paper_2506_23225_b200.mglu import MGLU_ERR_UNSUPPORTED, MgluError
        with pytest.raises(MgluError) as e:
            layer.forward_routed(x, Wt, packed, torch.from_numpy(G.astype(np.float32)).cuda(), K)
        assert e.value.status == MGLU_ERR_UNSUPPORTED
        return
    y = layer.forward_routed(x, Wt, packed, torch.from_numpy(G.astype(np.float32)).cuda(), K)
    torch.cuda.synchronize()
    assert layer.last_path() == path
    ref = _oracle_routed(inp, n_m, 1, G.astype(np.float32).astype(np.float64))
    err = normwise_err(y.float().cpu().numpy().astype(np.float64), ref)
    assert err <= TOL["bf16"] and err <= TIGHT["bf16"], err


def test_routed_forward_no_promise_and_other_activation():
    """K = 0 (no sparsity promise: every mask evaluated) and a non-Swish activation (weights in the
    epilogue only) give the same routed sum as the oracle."""
    from oracle import topk_gate
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    d, h, n_m, B = 1024, 300, 8, 2
    inp = make_inputs(901, B=B, d=d, h=h, n_m=n_m, dtype="bf16")
    x, Wt = to_device(inp, "bf16")
    packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
    G = topk_gate(np.random.default_rng(5).standard_normal((B, n_m)), 2).astype(np.float32)
    for act, code, K in (("swish", 1, 0), ("gelu", 2, 2), ("sigmoid", 4, 2)):
        layer = Mglu(d, h, n_m, act=act, dtype="bf16", path="mma")
        y = layer.forward_routed(x, Wt, packed, torch.from_numpy(G).cuda(), K)
        ref = _oracle_routed(inp, n_m, code, G.astype(np.float64))
        assert normwise_err(y.float().cpu().numpy().astype(np.float64), ref) <= TIGHT["bf16"], act


def test_router_then_routed_forward_chain():
    """router -> routed forward on one stream (PDL chain), config-3 shape, B = 1, n_m = 8, K = 2;
    the oracle applies the GPU's gate weights (the discrete TopK decision is checked above)."""
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    d, h, n_m, K = 4096, 1024, 8, 2
    inp = make_inputs(77, B=1, d=d, h=h, n_m=n_m, dtype="bf16")
    x, Wt = to_device(inp, "bf16")
    packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
    Wr = _router_weights(3, n_m, d).cuda()
    layer = Mglu(d, h, n_m, act="swish", dtype="bf16")
    G = layer.router_topk(x, Wr, K)
    y = layer.forward_routed(x, Wt, packed, G, K)
    torch.cuda.synchronize()
    assert layer.last_path() == "mma" and int((G != 0).sum()) == K
    ref = _oracle_routed(inp, n_m, 1, G.cpu().numpy().astype(np.float64))
    assert normwise_err(y.float().cpu().numpy().astype(np.float64), ref) <= TIGHT["bf16"]


def test_routed_errors():
    from paper_2506_23225_b200.mglu import Mglu, MgluError, MGLU_ERR_INVALID_ARG
    d, h, n_m = 512, 256, 4
    layer = Mglu(d, h, n_m, dtype="bf16")
    x = torch.zeros(1, d, dtype=torch.bfloat16, device="cuda")
    Wr = torch.zeros(n_m, d, dtype=torch.bfloat16, device="cuda")
    for K in (0, n_m + 1):
        with pytest.raises(MgluError) as e:
            layer.router_topk(x, Wr, K)
        assert e.value.status == MGLU_ERR_INVALID_ARG
    Wt = torch.zeros(h, d, dtype=torch.bfloat16, device="cuda")
    packed = torch.zeros(h * d * n_m // 8, dtype=torch.uint8, device="cuda")
    with pytest.raises(MgluError) as e:
        layer.forward_routed(x, Wt, packed, torch.zeros(1, n_m, device="cuda"), n_m + 1)
    assert e.value.status == MGLU_ERR_INVALID_ARG


@pytest.mark.parametrize("B", [40, 300])
def test_routed_forward_large_batch_auto(B):
    """Prefill-sized routed batches through AUTO (stream-K GEMV / tcgen05 tile GEMM: every mask
    evaluated, weighted in the epilogue)."""
    from oracle import topk_gate
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
    d, h, n_m, K = 1024, 512, 4, 2
    inp = make_inputs(1000 + B, B=B, d=d, h=h, n_m=n_m, dtype="bf16")
    x, Wt = to_device(inp, "bf16")
    packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
    G = topk_gate(np.random.default_rng(B).standard_normal((B, n_m)), K).astype(np.float32)
    layer = Mglu(d, h, n_m, act="swish", dtype="bf16")
    y = layer.forward_routed(x, Wt, packed, torch.from_numpy(G).cuda(), K)
    torch.cuda.synchronize()
    assert layer.last_path() == ("tcdec" if B <= 16 else "tcgen05")
    ref = _oracle_routed(inp, n_m, 1, G.astype(np.float64))
    assert normwise_err(y.float().cpu().numpy().astype(np.float64), ref) <= TIGHT["bf16"]
