"""Multi-process column-shard path on CPU (gloo, world_size 2 and 3): the host logic of SURVEY
8(e) -- shard bounds, code byte ranges as pointer offsets, and the all-gather that reassembles
[B][h] -- checked end to end with the CPU oracle standing in for the per-rank kernel (the GPU
kernel's own shard parity is tests/test_gpu_shard.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_23225_b200.shard import code_bytes_per_row, gather_columns, shard_bounds, shard_layer


def test_shard_bounds_partition():
    for h in (1, 7, 128, 300, 14336, 28672, 11008):
        for G in (1, 2, 3, 4, 6, 8):
            for align in (1, 8, 128):
                b = [shard_bounds(h, G, r, align=align) for r in range(G)]
                assert b[0][0] == 0 and b[-1][1] == h
                assert all(b[r][1] == b[r + 1][0] for r in range(G - 1))
                assert all(lo % align == 0 for lo, _ in b)          # shards start on a granule
                sizes = [hi - lo for lo, hi in b]
                assert max(sizes) - min(sizes) <= align
    # default granule: whole 128-row tiles for every rank but possibly the last
    for h in (11008, 14336, 28672):
        for G in (3, 6, 8):
            b = [shard_bounds(h, G, r) for r in range(G)]
            assert all((hi - lo) % 128 == 0 for lo, hi in b[:-1])
    # the BASELINE configs shard into whole 128-row tcgen05 tiles
    for h, G in ((14336, 8), (28672, 8), (28672, 4), (28672, 2)):
        assert all((hi - lo) % 128 == 0 for lo, hi in (shard_bounds(h, G, r) for r in range(G)))


def test_code_rows_are_pointer_offsets():
    """Packing a row slice of the masks gives exactly the byte slice of the packed layer."""
    from oracle import pack_np
    from synth import make_inputs
    inp = make_inputs(3, B=1, d=96, h=10, n_m=4)
    full = pack_np(inp["bits"])
    rb = code_bytes_per_row(96, 4)
    for G in (2, 3):
        for r in range(G):
            lo, hi = shard_bounds(10, G, r, align=1)
            np.testing.assert_array_equal(pack_np(inp["bits"][:, lo:hi]), full[lo * rb:hi * rb])
    Wt = torch.arange(10 * 96, dtype=torch.float32).reshape(10, 96)
    p = torch.from_numpy(full.copy())
    W1, p1 = shard_layer(Wt, p, 4, 3, 1, align=1)
    lo, hi = shard_bounds(10, 3, 1, align=1)
    assert W1.data_ptr() == Wt[lo].data_ptr() and p1.data_ptr() == p[lo * rb].data_ptr()


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import COracle, decode_bf16
        from synth import make_inputs
        d, h, n_m, B = 64, 300, 2, 3   # granules of 128 rows: a ragged last shard
        inp = make_inputs(11, B=B, d=d, h=h, n_m=n_m)
        o = COracle()
        packed = torch.from_numpy(o.pack(inp["bits"]))
        Wt = torch.from_numpy(decode_bf16(inp["Wt"]))
        x = decode_bf16(inp["x"])
        W_loc, p_loc = shard_layer(Wt, packed, n_m, world, rank)
        lo, hi = shard_bounds(h, world, rank)
        # the per-rank "kernel": the oracle on this rank's rows only (its own unpacker reads the
        # code slice as a self-contained [hi-lo][d] layer)
        y_loc = o.forward(x, W_loc.numpy(), np.arange(hi - lo), p_loc.numpy(), n_m, 1)
        y = gather_columns(torch.from_numpy(np.ascontiguousarray(y_loc)), h)
        ref = o.forward(x, Wt.numpy(), np.arange(h), packed.numpy(), n_m, 1)
        np.save(os.path.join(out_dir, f"r{rank}.npy"), np.stack([y.numpy(), ref]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gather_reassembles_full_output(tmp_path, world):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        y, ref = np.load(tmp_path / f"r{r}.npy")
        # columns are independent: the gathered shards equal the unsharded oracle exactly
        np.testing.assert_array_equal(y, ref)


def _ffn_worker(rank, world, port, out_dir):
    """Row f1 on CPU: rank-local oracle up-projection on the column shard, dense partial on the
    W_o row shard, gloo all-reduce -- equals the unsharded FFN oracle."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import ACT_SWISH, decode_bf16, dense_np, ffn_forward_np, mglu_forward_np
        from paper_2506_23225_b200.shard import shard_down
        from synth import make_inputs
        d, h, n_m, B = 64, 300, 2, 2
        inp = make_inputs(21, B=B, d=d, h=h, n_m=n_m)
        x, Wt = decode_bf16(inp["x"]), decode_bf16(inp["Wt"])
        Wo = torch.from_numpy(np.random.default_rng(4).standard_normal((d, h)))
        lo, hi = shard_bounds(h, world, rank)
        y_g = mglu_forward_np(x, Wt[lo:hi], inp["bits"][:, lo:hi], ACT_SWISH)
        part = torch.from_numpy(dense_np(y_g, shard_down(Wo, world, rank).numpy()))
        dist.all_reduce(part, op=dist.ReduceOp.SUM)
        ref = ffn_forward_np(x, Wt, inp["bits"], Wo.numpy(), ACT_SWISH)
        np.save(os.path.join(out_dir, f"f{rank}.npy"), np.stack([part.numpy(), ref]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ffn_row_parallel_all_reduce(tmp_path, world):
    mp.spawn(_ffn_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        out, ref = np.load(tmp_path / f"f{r}.npy")
        np.testing.assert_allclose(out, ref, rtol=1e-12, atol=1e-12)
