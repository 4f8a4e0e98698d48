"""Multi-process (gloo, world_size 2, CPU) tests of the batch-sharding plumbing."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_20493_b200.parallel import gather_batch, gather_to, shard_batch, shard_range


def test_shard_range_partitions():
    for batch in (0, 1, 5, 64, 4096, 4097):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(batch, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == batch
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class _FakeLayer:
    """Stand-in for PreparedLayer on CPU: a per-sample deterministic map."""

    def forward(self, x):
        return x * 2.0 + torch.arange(x.shape[1], dtype=x.dtype).view(1, -1, 1, 1)


def _worker(rank, world, port, batch, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(0)
        x_full = torch.rand((batch, 3, 4, 5), generator=g)
        layer = _FakeLayer()
        y_local = layer.forward(shard_batch(x_full, world, rank).contiguous())
        full = gather_batch(y_local, batch)
        assert torch.equal(full, layer.forward(x_full)), "gathered output differs from single-process"
        only0 = gather_to(y_local, batch, dst=0)
        assert (only0 is not None) == (rank == 0)
        if rank == 0:
            torch.save(full, out_path)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("batch", [7, 8])
def test_gloo_world2_shard_and_gather(tmp_path, batch):
    out = str(tmp_path / "full.pt")
    mp.spawn(_worker, args=(2, _free_port(), batch, out), nprocs=2, join=True)
    full = torch.load(out)
    assert full.shape[0] == batch


def _channel_worker(rank, world, port, c_out, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2502_20493_b200.parallel import gather_channels
        g = torch.Generator().manual_seed(1)
        y_full = torch.rand((3, c_out, 4, 5), generator=g)
        co0, co1 = shard_range(c_out, world, rank)
        full = gather_channels(y_full[:, co0:co1], c_out)
        assert torch.equal(full, y_full)
        if rank == 0:
            torch.save(full, out_path)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("c_out", [5, 6])
def test_gloo_world2_channel_gather(tmp_path, c_out):
    out = str(tmp_path / "full.pt")
    mp.spawn(_channel_worker, args=(2, _free_port(), c_out, out), nprocs=2, join=True)
    assert torch.load(out).shape[1] == c_out
