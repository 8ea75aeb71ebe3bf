"""Out-of-bounds and concurrency checks of our own (compute-sanitizer is closed on the GPU pool:
runs under it left GPUs needing a reset; its round-2 logs are in profiles/r02/sanitizer_run1.log).

* Guard bands: every output (y, Alg. 1's z, the router's G) is written into the middle of a larger
  buffer pre-filled with a sentinel byte pattern; after the call the bands on both sides must be
  untouched and every inside element written, on every path and at ragged shapes (h % 128 != 0,
  the row split's two box heights, a token count that is not a tile multiple).
* Inputs are read-only: x, Wt and the codes are bit-identical after the calls.
* The stream-K GEMV on three concurrent streams, one handle each (tools/sanitize_case.py), gives
  the single-stream result bit for bit (its last-arriver protocol never waits on another CTA)."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SENT = 0x7F    # bytes 0x7F7F: a bf16 NaN / an fp32 3.4e38 -- never a result of these inputs


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_23225_b200.build import build
    build()


def _guarded(n, dtype, pad=4096):
    """(buffer, view of n elements starting after `pad` bytes of sentinel)"""
    es = torch.tensor([], dtype=dtype).element_size()
    raw = torch.full((2 * pad + n * es,), SENT, dtype=torch.uint8, device="cuda")
    return raw, raw[pad:pad + n * es].view(dtype)


def _check_bands(raw, n, dtype, pad=4096):
    es = torch.tensor([], dtype=dtype).element_size()
    assert bool((raw[:pad] == SENT).all()), "write before the output"
    assert bool((raw[pad + n * es:] == SENT).all()), "write past the output"
    inside = raw[pad:pad + n * es].view(-1, es)
    assert not bool((inside == SENT).all(dim=1).any()), "output element never written"


CASES = [  # (path, d, h, n_m, B)
    ("mma", 512, 300, 4, 3), ("mma", 1024, 1000, 1, 7),
    ("tcdec", 512, 300, 4, 9), ("tcdec", 1024, 9601, 4, 5), ("tcdec", 256, 19000, 8, 30),
    ("tcgen05", 512, 300, 4, 40), ("tcgen05", 256, 700, 8, 130),
    ("simt", 512, 300, 3, 2), ("simt", 256, 200, 16, 3),
]


@pytest.mark.parametrize("path,d,h,n_m,B", CASES)
def test_outputs_stay_in_bounds(path, d, h, n_m, B):
    from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_device
    g = torch.Generator(device="cuda").manual_seed(d + h + B)
    bits = (torch.rand(n_m, h, d, device="cuda", generator=g) > 0.5).to(torch.uint8)
    packed = mglu_pack_masks_device(bits)
    Wt = (torch.randn(h, d, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    x = torch.randn(B, d, device="cuda", generator=g).to(torch.bfloat16)
    x0, W0, p0 = x.clone(), Wt.clone(), packed.clone()
    layer = Mglu(d, h, n_m, act="swish", dtype="bf16", path=path)
    raw, y = _guarded(B * h, torch.bfloat16)
    layer.forward(x, Wt, packed, out=y.view(B, h))
    torch.cuda.synchronize()
    assert layer.last_path() == path
    _check_bands(raw, B * h, torch.bfloat16)
    if path != "mma" or n_m <= 4:
        z = layer.forward_partials(x, Wt, packed)
        assert z.shape == (B, 2 * n_m, h) and bool(torch.isfinite(z).all())
    if n_m in (1, 2, 4, 8):
        Wr = (torch.randn(n_m, d, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
        K = min(2, n_m)
        G = layer.router_topk(x, Wr, K)
        raw2, y2 = _guarded(B * h, torch.bfloat16)
        layer.forward_routed(x, Wt, packed, G, K, out=y2.view(B, h))
        torch.cuda.synchronize()
        _check_bands(raw2, B * h, torch.bfloat16)
    assert torch.equal(x, x0) and torch.equal(Wt, W0) and torch.equal(packed, p0), "an input was written"
    layer.close()


def test_concurrent_streams_case():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_case.py")],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0 and "sanitize case ok" in r.stdout, (r.stdout + r.stderr)[-3000:]
