"""(batch x head) sharding across the GPUs of one node.

The (b, h) slices of the chunkwise mLSTM are fully independent
(test_tiled.cpp:223-262 asserts bitwise slice independence), so multi-GPU runs
shard the flattened slice index into contiguous ranges, one per rank, with no
collective on the data path. The only collective is an optional final
all-gather of H / gradients (NCCL over NVLink on the GPU box, gloo in the CPU
tests), timed separately from the kernels.
"""
from __future__ import annotations

from typing import Callable, Sequence

import torch
import torch.distributed as dist


def shard_range(n_slices: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, end) of the flattened (b*NH + h) index for `rank`.
    Balanced: the first n_slices % world ranks get one extra slice."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n_slices, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def slice_view(x: torch.Tensor, start: int, end: int) -> torch.Tensor:
    """Rows [start, end) of the flattened (B*NH) leading index of a
    [B, NH, ...] tensor, as a [1, end-start, ...] view (n_batch=1, n_head=end-start)."""
    flat = x.reshape(x.shape[0] * x.shape[1], *x.shape[2:])
    return flat[start:end].unsqueeze(0)


def gather_slices(parts: torch.Tensor, n_slices: int, group=None) -> torch.Tensor:
    """All-gather per-rank [1, n_local, ...] shards into [n_slices, ...] (final gather)."""
    world = dist.get_world_size(group)
    sizes = [shard_range(n_slices, world, r) for r in range(world)]
    local = parts.reshape(parts.shape[1], *parts.shape[2:]).contiguous()
    maxn = max(e - s for s, e in sizes)
    pad = torch.zeros((maxn, *local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[: e - s] for b, (s, e) in zip(bufs, sizes)], dim=0)


def run_sharded(compute: Callable[..., Sequence[torch.Tensor]], tensors: Sequence[torch.Tensor],
                n_batch: int, n_head: int, group=None, gather: bool = True):
    """Run `compute(*shard_views)` on this rank's (b, h) slices and optionally
    all-gather every returned [1, n_local, ...] tensor into [B, NH, ...]."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n = n_batch * n_head
    s, e = shard_range(n, world, rank)
    outs = compute(*[slice_view(t, s, e) for t in tensors])
    if not gather or world == 1:
        return outs
    return [gather_slices(o, n, group).reshape(n_batch, n_head, *o.shape[2:]) for o in outs]
