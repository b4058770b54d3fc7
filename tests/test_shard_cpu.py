"""Host logic of the observation-sharded C5' path (paper_2003_08011_b200/
shard.py) on CPU: shard ranges and the size-then-payload broadcast over a
2-rank gloo group.  The device side (pack / unpack / bitwise shard
concatenation, and the same broadcast with CUDA tensors) is
tests/test_gpu_shard.py."""
import multiprocessing as mp
import os
import socket

import pytest

from paper_2003_08011_b200.shard import SHARD_ALIGN, shard_range


@pytest.mark.parametrize("N", [0, 1, 127, 128, 129, 1000, 100_000, 1_250_000, 10_000_000])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 7, 8])
def test_shard_ranges_partition_the_observations(N, world):
    ranges = [shard_range(N, world, r) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == N
    for (a0, a1), (b0, b1) in zip(ranges, ranges[1:]):
        assert a1 == b0 and a0 <= a1
    # every boundary except N sits on a kernel tile
    assert all(s % SHARD_ALIGN == 0 or s == N for s, _ in ranges)
    sizes = [b - a for a, b in ranges]
    assert max(sizes) - min(sizes) < 2 * SHARD_ALIGN  # balanced to a tile (+ the partial last tile)


def test_shard_range_rejects_bad_rank():
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)
    with pytest.raises(ValueError):
        shard_range(10, 0, 0)


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2003_08011_b200.shard import broadcast_bytes, shard_digest, wrap64
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    payload = None
    if rank == 1:  # a non-zero source
        g = torch.Generator().manual_seed(7)
        payload = torch.randint(0, 256, (100_003,), dtype=torch.uint8, generator=g)
    got = broadcast_bytes(payload, src=1)
    # each rank digests its shard of a common float tensor; the sum of the
    # shard digests is the whole tensor's digest
    x = torch.arange(1000, dtype=torch.float32).reshape(100, 10).T.contiguous().T  # column-major
    a, b = shard_range(100, world, rank, align=8)
    d = torch.tensor([shard_digest(x[a:b])], dtype=torch.int64)
    dist.all_reduce(d)
    q.put((rank, got.numel(), int(got.to(torch.int64).sum()), wrap64(int(d.item())), shard_digest(x)))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_gloo_broadcast_bytes_and_digests():
    import torch
    g = torch.Generator().manual_seed(7)
    want = torch.randint(0, 256, (100_003,), dtype=torch.uint8, generator=g)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, n, s, dsum, dfull in res:
        assert n == want.numel() and s == int(want.to(torch.int64).sum())
        assert dsum == dfull  # shard digests add up to the single-rank digest
