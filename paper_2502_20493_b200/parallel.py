"""Batch sharding across GPUs (one process per GPU) and the on-request output gather.

The unified transpose convolution is an independent map over samples (SPEC.md:253 of the
reference; disjoint writes, read-only weights), so the multi-GPU path is pure data
parallelism: each rank runs the contiguous batch shard `shard_range(batch, world, rank)`
with its own device copy of the segregated weights. Nothing is exchanged on the hot path.
Because per-sample arithmetic is identical, outputs are bitwise independent of the number
of GPUs.

`gather_batch` / `gather_to` assemble the full output only when a caller asks for it
(NCCL all-gather / gather over NVLink on GPUs, gloo on CPU). They are never part of a
timed step.
"""

from __future__ import annotations


def shard_range(batch: int, world: int, rank: int) -> tuple[int, int]:
    """[start, stop) of `rank`'s contiguous shard; sizes differ by at most one sample."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"invalid rank {rank} of world {world}")
    if batch < 0:
        raise ValueError(f"batch must be >= 0, got {batch}")
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard_batch(x, world: int, rank: int):
    """The local shard (a view) of a full (B, ...) batch."""
    start, stop = shard_range(x.shape[0], world, rank)
    return x[start:stop]


def _group_info(group):
    import torch.distributed as dist
    return dist.get_world_size(group), dist.get_rank(group)


def gather_batch(y_local, batch: int, group=None):
    """All-gather the per-rank output shards into the full (batch, ...) tensor on every rank.

    Shards may be uneven (shard_range); they are padded to the largest shard for the
    collective and trimmed afterwards, preserving the global sample order."""
    import torch
    import torch.distributed as dist
    world, rank = _group_info(group)
    sizes = [shard_range(batch, world, r) for r in range(world)]
    if y_local.shape[0] != sizes[rank][1] - sizes[rank][0]:
        raise ValueError(f"rank {rank} holds {y_local.shape[0]} samples, expected "
                         f"{sizes[rank][1] - sizes[rank][0]}")
    cap = max(stop - start for start, stop in sizes)
    buf = torch.zeros((cap,) + tuple(y_local.shape[1:]), dtype=y_local.dtype, device=y_local.device)
    buf[:y_local.shape[0]] = y_local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf.contiguous(), group=group)
    return torch.cat([parts[r][:stop - start] for r, (start, stop) in enumerate(sizes)], dim=0)


def gather_to(y_local, batch: int, dst: int = 0, group=None):
    """Gather the full output on rank `dst` only (returns None elsewhere)."""
    full = gather_batch(y_local, batch, group)
    _, rank = _group_info(group)
    return full if rank == dst else None


def sharded_forward(layer, x_full, group=None, gather: bool = False):
    """Run `layer` (a PreparedLayer) on this rank's shard of the full batch `x_full`.

    Returns the local output shard, or the gathered full output when `gather=True`."""
    world, rank = _group_info(group)
    y = layer.forward(shard_batch(x_full, world, rank).contiguous())
    return gather_batch(y, x_full.shape[0], group) if gather else y
