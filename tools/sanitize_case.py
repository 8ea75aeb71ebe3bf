"""Tiny invocations of every kernel for compute-sanitizer (tests/test_gpu_sanitizer.py runs this
under memcheck / racecheck / synccheck).  Also runs the stream-K GEMV on three concurrent streams
(one handle each) so the inter-CTA protocol is exercised under concurrency."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_device, mglu_unpack_masks_device  # noqa: E402


def main():
    g = torch.Generator(device="cuda").manual_seed(0)
    d, h = 512, 300
    for n_m in (1, 4, 8):
        bits = (torch.rand(n_m, h, d, device="cuda", generator=g) > 0.5).to(torch.uint8)
        packed = mglu_pack_masks_device(bits)
        assert torch.equal(mglu_unpack_masks_device(packed, n_m, h, d), bits)
        Wt = (torch.randn(h, d, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
        for path, B in (("mma", 3), ("tcdec", 9), ("tcrow", 12), ("tcgen05", 40), ("simt", 2)):
            if path == "mma" and n_m >= 4 and B > 4:
                continue
            x = torch.randn(B, d, device="cuda", generator=g).to(torch.bfloat16)
            layer = Mglu(d, h, n_m, act="swish", dtype="bf16", path=path)
            y = layer.forward(x, Wt, packed)
            z = layer.forward_partials(x, Wt, packed)
            Wr = (torch.randn(n_m, d, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
            G = layer.router_topk(x, Wr, min(2, n_m))
            layer.forward_routed(x, Wt, packed, G, min(2, n_m))
            torch.cuda.synchronize()
            assert torch.isfinite(y.float()).all() and torch.isfinite(z).all()
            layer.close()
    # stream-K on three concurrent streams, one handle each (mglu.h threading contract)
    n_m, B, d, h = 4, 12, 1024, 1000
    bits = (torch.rand(n_m, h, d, device="cuda", generator=g) > 0.5).to(torch.uint8)
    packed = mglu_pack_masks_device(bits)
    Wt = (torch.randn(h, d, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    x = torch.randn(B, d, device="cuda", generator=g).to(torch.bfloat16)
    ref = Mglu(d, h, n_m, path="tcdec").forward(x, Wt, packed)
    streams = [torch.cuda.Stream() for _ in range(3)]
    layers = [Mglu(d, h, n_m, path="tcdec") for _ in range(3)]
    outs = [torch.empty_like(ref) for _ in range(3)]
    torch.cuda.synchronize()
    for rep in range(4):
        for s, l, o in zip(streams, layers, outs):
            with torch.cuda.stream(s):
                l.forward(x, Wt, packed, out=o, stream=s)
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o, ref)
    # f32 tiny config (SIMT)
    x32 = torch.randn(1, 64, device="cuda", generator=g)
    W32 = torch.randn(128, 64, device="cuda", generator=g)
    b1 = (torch.rand(1, 128, 64, device="cuda", generator=g) > 0.5).to(torch.uint8)
    Mglu(64, 128, 1, dtype="f32").forward(x32, W32, mglu_pack_masks_device(b1))
    torch.cuda.synchronize()
    print("sanitize case ok")


if __name__ == "__main__":
    main()
