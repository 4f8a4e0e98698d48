"""Batch / output-channel sharding across GPUs (one process per GPU) and the on-request gather.

The unified transpose convolution is an independent map over samples and output channels
(SPEC.md:253,255-256 of the reference: batch = map over samples; the iteration space is
batch x output channel with disjoint writes and read-only weights; the reference itself tiles
output channels in fixed blocks, engines.py:48-51,294-306). So the multi-GPU path is pure data
parallelism with no exchange on the hot path:

  * batch sharding (the default): rank r runs the contiguous batch shard shard_range(B, G, r)
    with its own device copy of the segregated weights;
  * output-channel sharding (small batches, where the weights dominate the bytes, e.g. the
    l2 layers at B <= 8): rank r prepares only its slice of the bank's output channels and
    computes y[:, co0:co1] for the whole batch.

Per-sample / per-channel arithmetic is identical to one GPU, so outputs are bitwise independent
of the number of GPUs. The full output is assembled only when a caller asks for it, outside any
timed step: `gather_batch` writes every rank's shard straight into the caller-visible output
(one all_gather_into_tensor when the shards are even, one broadcast per rank otherwise -- no
padded staging copy), `gather_channels` does the same along the channel dimension.
"""

from __future__ import annotations


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """[start, stop) of `rank`'s contiguous shard of `total` items; sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"invalid rank {rank} of world {world}")
    if total < 0:
        raise ValueError(f"batch must be >= 0, got {total}")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard_batch(x, world: int, rank: int):
    """The local shard (a view) of a full (B, ...) batch."""
    start, stop = shard_range(x.shape[0], world, rank)
    return x[start:stop]


def _group_info(group):
    import torch.distributed as dist
    return dist.get_world_size(group), dist.get_rank(group)


def gather_batch(y_local, batch: int, group=None, out=None):
    """The full (batch, ...) output on every rank, assembled from the per-rank batch shards.

    Even shards: one all_gather_into_tensor directly into `out`. Uneven shards: one broadcast
    per rank into its slice of `out`. Either way nothing beyond `out` itself is allocated."""
    import torch
    import torch.distributed as dist
    world, rank = _group_info(group)
    spans = [shard_range(batch, world, r) for r in range(world)]
    if y_local.shape[0] != spans[rank][1] - spans[rank][0]:
        raise ValueError(f"rank {rank} holds {y_local.shape[0]} samples, expected "
                         f"{spans[rank][1] - spans[rank][0]}")
    if out is None:
        out = torch.empty((batch,) + tuple(y_local.shape[1:]), dtype=y_local.dtype, device=y_local.device)
    y_local = y_local.contiguous()
    if batch % world == 0 and hasattr(dist, "all_gather_into_tensor"):
        dist.all_gather_into_tensor(out, y_local, group=group)
        return out
    out[spans[rank][0]:spans[rank][1]].copy_(y_local)
    for r, (start, stop) in enumerate(spans):
        if stop > start:
            dist.broadcast(out[start:stop], src=dist.get_global_rank(group, r) if group is not None else r,
                           group=group)
    return out


def gather_to(y_local, batch: int, dst: int = 0, group=None):
    """The full output on rank `dst` only (None elsewhere): one point-to-point receive per peer
    shard, written into its slice of the output."""
    import torch
    import torch.distributed as dist
    world, rank = _group_info(group)
    spans = [shard_range(batch, world, r) for r in range(world)]
    gdst = dist.get_global_rank(group, dst) if group is not None else dst
    if rank != dst:
        dist.send(y_local.contiguous(), dst=gdst, group=group)
        return None
    out = torch.empty((batch,) + tuple(y_local.shape[1:]), dtype=y_local.dtype, device=y_local.device)
    for r, (start, stop) in enumerate(spans):
        if r == rank:
            out[start:stop].copy_(y_local)
        elif stop > start:
            src = dist.get_global_rank(group, r) if group is not None else r
            dist.recv(out[start:stop], src=src, group=group)
    return out


def sharded_forward(layer, x_full, group=None, gather: bool = False):
    """Run `layer` (a PreparedLayer) on this rank's batch shard of the full batch `x_full`.

    Returns the local output shard, or the gathered full output when `gather=True`."""
    world, rank = _group_info(group)
    y = layer.forward(shard_batch(x_full, world, rank).contiguous())
    return gather_batch(y, x_full.shape[0], group) if gather else y


# ------------------------------------------------------------------- output-channel sharding

def prepare_channel_shard(bank, pad: int, world: int, rank: int, compute: str | None = None):
    """This rank's PreparedLayer over output channels [co0, co1) of `bank` (c_in, c_out, n, n),
    and that range. Every rank then runs the whole batch on its channel slice."""
    from .engines import prepare_layer
    c_out = int(bank.shape[1])
    co0, co1 = shard_range(c_out, world, rank)
    if co1 <= co0:
        raise ValueError(f"rank {rank} of {world} gets no output channel of {c_out}")
    return prepare_layer(bank[:, co0:co1], pad, compute=compute), (co0, co1)


def gather_channels(y_local, c_out: int, group=None, out=None):
    """The full (B, c_out, H, W) output on every rank from per-rank channel slices
    (B, co1 - co0, H, W): each rank broadcasts its slice into the strided channel window of
    `out` (a contiguous staging copy of the slice is the only extra buffer)."""
    import torch
    import torch.distributed as dist
    world, rank = _group_info(group)
    spans = [shard_range(c_out, world, r) for r in range(world)]
    b = y_local.shape[0]
    if out is None:
        out = torch.empty((b, c_out) + tuple(y_local.shape[2:]), dtype=y_local.dtype, device=y_local.device)
    for r, (co0, co1) in enumerate(spans):
        buf = y_local.contiguous() if r == rank else torch.empty(
            (b, co1 - co0) + tuple(y_local.shape[2:]), dtype=y_local.dtype, device=y_local.device)
        src = dist.get_global_rank(group, r) if group is not None else r
        dist.broadcast(buf, src=src, group=group)
        out[:, co0:co1].copy_(buf)
    return out
