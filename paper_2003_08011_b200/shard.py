"""Observation-sharded surveillance across the GPUs of one box (SURVEY 8(e),
BASELINE configs[4] "sharded across 8 x B200").

The reference's estimate is independent per observation (mset.cpp:174-199:
every column of S = sim(D_norm, x_norm), W = G+ S and D W depends only on
its own observation), so the N observations split into contiguous shards,
one per rank, with no collective inside the surveillance loop.  The model
is trained ONCE (rank `src`), packed into one device buffer
(cs_model_pack_device) and broadcast over NCCL -- NVLink / NVSwitch on a
B200 box -- then unpacked on every rank.  The kernels' tiling restarts at
each shard's first observation and no observation's result depends on
another's, so the concatenated shard outputs are bitwise the single-GPU
outputs (the analogue of the reference's worker-count invariance,
test_backends.cpp:80-88; tests/test_gpu_shard.py).

Host logic (shard ranges, the size-then-payload broadcast) is plain
torch.distributed and runs on gloo in tests/test_shard_cpu.py.
"""
from __future__ import annotations

from typing import Optional, Tuple

SHARD_ALIGN = 128  # the surveillance kernels' observation tile


def shard_range(N: int, world: int, rank: int, align: int = SHARD_ALIGN) -> Tuple[int, int]:
    """[start, stop) of rank's contiguous shard of N observations.  Shards
    are balanced in units of `align` observations (the kernels' tile), so
    at most the last shard carries a partial tile; every observation is in
    exactly one shard."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"shard_range: rank {rank} outside world {world}")
    if N < 0:
        raise ValueError("shard_range: N must be >= 0")
    units = (N + align - 1) // align
    base, extra = divmod(units, world)
    u0 = rank * base + min(rank, extra)
    u1 = u0 + base + (1 if rank < extra else 0)
    return min(u0 * align, N), min(u1 * align, N)


def broadcast_bytes(payload, src: int = 0, group=None, device=None):
    """Broadcast a 1-D uint8 tensor of unknown length from `src`: the length
    first (one int64), then the payload.  `payload` is ignored on non-source
    ranks; they receive into a fresh tensor on `device` (the source's tensor
    is returned as is on the source).  NCCL needs CUDA tensors, gloo CPU
    ones: pass `device` accordingly."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    dev = payload.device if (rank == src and payload is not None) else torch.device(device or "cpu")
    n = torch.tensor([payload.numel() if rank == src else 0], dtype=torch.int64, device=dev)
    dist.broadcast(n, src=_global(src, group), group=group)
    if rank != src:
        payload = torch.empty(int(n.item()), dtype=torch.uint8, device=dev)
    dist.broadcast(payload, src=_global(src, group), group=group)
    return payload


def _global(src: int, group) -> int:
    import torch.distributed as dist
    return src if group is None else dist.get_global_rank(group, src)


def broadcast_model(model, backend, src: int = 0, group=None):
    """Train-once / use-everywhere: rank `src` packs its trained model into
    one device buffer and broadcasts it; every other rank unpacks it on
    `backend.device`.  Returns (model, wire_bytes).  On `src` the model
    passed in is returned unchanged."""
    import torch
    import torch.distributed as dist
    from .mset import pack_model, unpack_model
    rank = dist.get_rank(group)
    dev = torch.device("cuda", backend.device)
    wire = pack_model(model) if rank == src else None
    wire = broadcast_bytes(wire, src=src, group=group, device=dev)
    nbytes = wire.numel()
    if rank != src:
        model = unpack_model(wire, backend)
    del wire
    return model, nbytes


def estimate_shard(model, obs, start: int, stop: int, est=None, resid=None, stream=None):
    """Surveil observations [start, stop) of a column-major N x n tensor in
    place (views; no copies): the per-rank step of the sharded estimate."""
    from .mset import estimate_device
    if stop <= start:
        return
    view = lambda t: None if t is None else t[start:stop]  # noqa: E731
    estimate_device(model, obs[start:stop], view(est), view(resid), stream)


def shard_digest(t, chunk: Optional[int] = None) -> int:
    """Order-independent exact digest of a float tensor's bits (sum of the
    32-bit words as int64, wrapping): equal digests for bitwise-equal
    outputs regardless of how the observations were sharded."""
    import torch
    if not t.is_contiguous() and t.dim() == 2 and t.T.is_contiguous():
        t = t.T  # column-major: the same words, no copy
    words = t.contiguous().view(torch.int32) if t.dtype == torch.float32 else t.contiguous().view(torch.int64)
    return wrap64(int(words.sum(dtype=torch.int64).item()))


def wrap64(x: int) -> int:
    """x modulo 2^64 as a signed int64 (digests add with wrap-around, so the
    sum of shard digests equals the digest of the whole)."""
    x &= (1 << 64) - 1
    return x - (1 << 64) if x >= (1 << 63) else x
