"""Multi-process column shard with the CUDA kernels per rank: world size 2 processes
on the one GPU this box has (process group over gloo -- NCCL refuses two ranks on one device),
each rank running Mglu on its 128-row-aligned shard of the layer through the C ABI, the h-sliced
outputs all-gathered and compared on every rank with the unsharded layer: bit-identical on the
tcgen05 tile path, within the bf16 bound on the decode path.  Also bench.py itself under
torchrun (2 ranks, gloo): it must print one JSON line whose gather_check passed."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests.helpers import TIGHT, make_inputs, normwise_err, to_device

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_23225_b200.build import build
    build()


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir, path, B):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2506_23225_b200.mglu import Mglu, mglu_pack_masks_host
        from paper_2506_23225_b200.shard import gather_columns, shard_bounds, shard_layer
        d, h, n_m = 2048, 1000, 4
        inp = make_inputs(123, B=B, d=d, h=h, n_m=n_m, dtype="bf16")      # same seed on every rank
        x, Wt = to_device(inp, "bf16")
        packed = torch.from_numpy(mglu_pack_masks_host(inp["bits"])).cuda()
        W_r, p_r = shard_layer(Wt, packed, n_m, world, rank)
        lo, hi = shard_bounds(h, world, rank)
        y_r = Mglu(d, hi - lo, n_m, path=path).forward(x, W_r, p_r)         # the CUDA kernel, this rank's rows
        torch.cuda.synchronize()
        y = gather_columns(y_r.cpu(), h)                                     # gloo all-gather of the slices
        full = Mglu(d, h, n_m, path=path).forward(x, Wt, packed).cpu()
        torch.save({"y": y, "full": full}, os.path.join(out_dir, f"r{rank}.pt"))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("path,B", [("tcgen05", 40), ("mma", 2), ("tcdec", 8)])
def test_two_process_shards(tmp_path, path, B):
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path), path, B), nprocs=2, join=True)
    for r in range(2):
        res = torch.load(tmp_path / f"r{r}.pt")
        if path == "tcgen05":
            assert torch.equal(res["y"], res["full"])
        else:
            err = normwise_err(res["y"].float().numpy().astype(np.float64), res["full"].float().numpy().astype(np.float64))
            assert err <= TIGHT["bf16"], err


def test_bench_under_torchrun_two_ranks():
    env = dict(os.environ, MGLU_DIST_BACKEND="gloo", OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--steps", "5", "--warmup", "3", "--no-comparator", "--layers", "2"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0 and len(lines) == 1, r.stdout[-2000:] + r.stderr[-3000:]
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["scaling"] == "strong"
    gc = out["gather_check"]
    assert gc["max_abs_diff"] <= 0.05 and "all_gather" in gc["collective"], gc
