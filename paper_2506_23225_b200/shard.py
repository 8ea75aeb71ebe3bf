"""Column (h) sharding of one MGLU up-projection layer across the ranks of a process group.

Eq. 3 is evaluated independently for every output column j: t_j, s_i,j and v_i,j
read only row j of Wt and row j of the packed codes.  A layer therefore shards along h with no
exchange on the hot path (north_star): rank g of G owns the contiguous rows
[lo_g, hi_g) of Wt and of the packed codes -- in the pair-split bit-plane layout (R3)
row j owns bytes [j*d*n_m/8, (j+1)*d*n_m/8), so a shard is a pointer offset into both tensors --
and runs an ordinary ``Mglu(d, hi_g - lo_g, n_m)`` handle on its rows.  x is replicated.

The one collective is ``gather_columns``: an all-gather of the h-sliced outputs into [B][h], used
only to check the full output (an FFN's row-parallel down-projection would consume the slices
directly).  Unequal shards (h % G != 0) are padded to the largest slice for the
all-gather and trimmed afterwards.

This module is host logic only (index arithmetic, views and torch.distributed calls); every
arithmetic step of the forward pass runs in libmglu's kernels.
"""
from __future__ import annotations

import torch


SHARD_ALIGN = 128   # rows per shard granule: whole tcgen05 M-tiles / HMMA row tiles on every rank


def shard_bounds(h: int, world: int, rank: int, align: int = SHARD_ALIGN) -> tuple[int, int]:
    """Rows [lo, hi) of rank `rank`: contiguous, in rank order, made of whole `align`-row granules
    (granule counts differ by at most one; only the last rank's last granule may be ragged), so
    every shard keeps the kernels' whole-tile shapes and a row-parallel W_o shard stays
    128-aligned (h_g % 128 == 0 whenever h % 128 == 0)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if align < 1:
        raise ValueError("align must be >= 1")
    n = (h + align - 1) // align
    lo, hi = rank * n // world * align, (rank + 1) * n // world * align
    return min(lo, h), min(hi, h)


def code_bytes_per_row(d: int, n_m: int) -> int:
    """Bytes of packed codes per Wt row: d * n_m / 8 (d % 32 == 0, reading R3)."""
    if d % 32:
        raise ValueError("d must be a multiple of 32")
    return d * n_m // 8


def shard_layer(Wt: torch.Tensor, packed: torch.Tensor, n_m: int, world: int, rank: int,
                align: int = SHARD_ALIGN):
    """Views of this rank's rows of Wt [h][d] and of the packed codes (no copy)."""
    h, d = Wt.shape
    lo, hi = shard_bounds(h, world, rank, align)
    rb = code_bytes_per_row(d, n_m)
    if packed.numel() != h * rb:
        raise ValueError("packed codes size mismatch")
    return Wt[lo:hi], packed[lo * rb:hi * rb]


def gather_columns(y_local: torch.Tensor, h: int, group=None, align: int = SHARD_ALIGN) -> torch.Tensor:
    """All-gather the column slices y_g [B][hi_g - lo_g] of every rank into y [B][h]."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    B = y_local.shape[0]
    width = max(max(shard_bounds(h, world, r, align)[1] - shard_bounds(h, world, r, align)[0] for r in range(world)), 1)
    buf = torch.zeros((B, width), dtype=y_local.dtype, device=y_local.device)
    buf[:, :y_local.shape[1]] = y_local
    parts = [torch.empty((B, width), dtype=y_local.dtype, device=y_local.device) for _ in range(world)]
    dist.all_gather(parts, buf.contiguous(), group=group)        # NCCL over NVLink, or gloo on CPU
    cols = []
    for r in range(world):
        lo, hi = shard_bounds(h, world, r, align)
        cols.append(parts[r][:, :hi - lo])
    return torch.cat(cols, dim=1)


# ------------------------------------------------------------------ FFN block
def shard_down(Wo: torch.Tensor, world: int, rank: int) -> torch.Tensor:
    """Row-parallel (reduction-dim) shard of the down-projection Wo [d][h]: this rank's h-columns
    [lo, hi) -- the rows of the up-projection it owns -- as a contiguous [d][hi - lo] copy (done
    once at load time, as tensor-parallel frameworks store it)."""
    lo, hi = shard_bounds(Wo.shape[1], world, rank)
    return Wo[:, lo:hi].contiguous()


def ffn_forward_tp(up, down, x: torch.Tensor, Wt_g: torch.Tensor, packed_g: torch.Tensor,
                   Wo_g: torch.Tensor, group=None) -> torch.Tensor:
    """One rank's SwiMGLU FFN block under tensor parallelism: the column-sharded up-projection
    y_g = MGLU_g(x) [B][h_g] (no exchange), the row-sharded down-projection partial y_g Wo_g^T
    [B][d] (an n_m = 0 dense handle; each rank's partial is rounded to bf16 by that handle's
    output, then widened), then ONE all-reduce (sum, in fp32) of the partials over the group -- the
    step's only collective (NCCL over NVLink on GPUs, gloo on CPU).  `up` / `down` are Mglu handles
    of shapes (d, h_g, n_m) and (h_g, d, 0); the dense handle needs h_g % 128 == 0 (shard_bounds
    gives that for h % (128 G) == 0, e.g. the Llama shapes at G in {1, 2, 4, 8})."""
    import torch.distributed as dist
    y_g = up.forward(x, Wt_g, packed_g)
    part = down.forward(y_g, Wo_g, None).float()
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(part, op=dist.ReduceOp.SUM, group=group)
    return part
