"""Observation-sharded surveillance (BASELINE configs[4]):
the packed model wire round-trips bitwise, and shard-by-shard estimates
concatenate to the single-GPU estimates bit for bit -- the analogue of the
reference's worker-count invariance (test_backends.cpp:80-88) -- on both
FP32 tcgen05 paths (fused n <= ~130, two-GEMM above) and the FP64 path.
The last test runs the real broadcast_model over a 2-process group (gloo
carrying CUDA tensors: one GPU per call here, NCCL refuses two ranks on one
device) with rank 0 training once."""
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def p():
    import torch  # noqa: F401
    import paper_2003_08011_b200 as p
    p.context(0)
    return p


def _data(p, n, rows, N, seed=20260810):
    X = p.synthesize(p.SignalSpec.uniform(n, rows, 0.5, 0.3, 1.0, 0.5, 4.0, seed)).data
    obs = p.synthesize(p.SignalSpec.uniform(n, N, 0.5, 0.3, 1.0, 0.5, 4.0, seed + 1)).data
    return X, obs


def _dev(obs, dtype):
    import torch
    return torch.tensor(np.ascontiguousarray(obs.T), dtype=dtype, device="cuda:0").T


CASES = [  # (n, m, precision, io): fused tcgen05, two-GEMM tcgen05, FP64 exact
    (100, 1000, "fp32", "f32"),
    (300, 600, "fp32", "f32"),
    (20, 100, "fp64", "f64"),
]


@pytest.mark.parametrize("n,m,precision,io", CASES)
def test_model_wire_round_trip_is_bitwise(p, n, m, precision, io):
    import torch
    X, obs = _data(p, n, 4 * m, 5000)
    B = p.BackendId("b200", 0, precision)
    model = p.train(X, m, p.KernelConfig(), B)
    wire = p.pack_model(model)
    copy = p.unpack_model(wire, B)
    a, b = model.export(), copy.export()
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    assert (copy.rank, copy.kernel, copy.precision) == (model.rank, model.kernel, model.precision)
    dt = torch.float32 if io == "f32" else torch.float64
    x = _dev(obs, dt)
    e1, r1 = torch.empty_like(x.T).T, torch.empty_like(x.T).T
    e2, r2 = torch.empty_like(x.T).T, torch.empty_like(x.T).T
    p.estimate_device(model, x, e1, r1)
    p.estimate_device(copy, x, e2, r2)
    torch.cuda.synchronize()
    assert torch.equal(e1, e2) and torch.equal(r1, r2)


def test_model_wire_rejects_garbage(p):
    import torch
    from paper_2003_08011_b200.errors import ConfigError, IoError
    junk = torch.zeros(4096, dtype=torch.uint8, device="cuda:0")
    with pytest.raises(IoError):
        p.unpack_model(junk, p.BackendId("b200", 0, "fp32"))
    X, _ = _data(p, 10, 200, 10)
    model = p.train(X, 50, p.KernelConfig(), p.BackendId("b200", 0, "fp32"))
    wire = p.pack_model(model)
    with pytest.raises(ConfigError):
        p.unpack_model(wire[:2048], p.BackendId("b200", 0, "fp32"))


@pytest.mark.parametrize("n,m,precision,io", CASES)
@pytest.mark.parametrize("N", [100_000, 50_001])
def test_sharded_estimates_equal_single_gpu_bitwise(p, n, m, precision, io, N):
    import torch
    from paper_2003_08011_b200.shard import estimate_shard, shard_digest, shard_range, wrap64
    if n >= 300 and N != 100_000:
        pytest.skip("one ragged case per path is enough for the large-n kernel")
    X, obs = _data(p, n, 4 * m, N)
    B = p.BackendId("b200", 0, precision)
    model = p.train(X, m, p.KernelConfig(), B)
    dt = torch.float32 if io == "f32" else torch.float64
    x = _dev(obs, dt)
    e_full, r_full = torch.empty_like(x.T).T, torch.empty_like(x.T).T
    p.estimate_device(model, x, e_full, r_full)
    replica = p.unpack_model(p.pack_model(model), B)  # what a non-source rank holds
    for world in (2, 3, 8):
        e, r = torch.full_like(x.T, float("nan")).T, torch.full_like(x.T, float("nan")).T
        digests = 0
        for rank in range(world):
            a, b = shard_range(N, world, rank)
            estimate_shard(model if rank == 0 else replica, x, a, b, e, r)
            digests += shard_digest(e[a:b])
        torch.cuda.synchronize()
        assert torch.equal(e, e_full), f"world={world}: sharded estimates differ"
        assert torch.equal(r, r_full), f"world={world}: sharded residuals differ"
        assert wrap64(digests) == shard_digest(e_full)


# ------------------------------------------------ 2-process broadcast_model
def _worker(rank, world, port, q, n, m, N):
    import torch
    import torch.distributed as dist
    import paper_2003_08011_b200 as p
    from paper_2003_08011_b200.shard import broadcast_model, estimate_shard, shard_range
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    B = p.BackendId("b200", 0, "fp32")
    X, obs = _data(p, n, 4 * m, N)
    model = p.train(X, m, p.KernelConfig(), B) if rank == 0 else None  # train once
    model, nbytes = broadcast_model(model, B, src=0)
    x = _dev(obs, torch.float32)
    e, r = torch.empty_like(x.T).T, torch.empty_like(x.T).T
    a, b = shard_range(N, world, rank)
    estimate_shard(model, x, a, b, e, r)
    torch.cuda.synchronize()
    q.put((rank, a, b, nbytes, e[a:b].cpu().numpy(), r[a:b].cpu().numpy(), model.export()["gram_pinv"]))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(600)
def test_two_process_broadcast_model_sharded_estimate(p):
    import torch
    n, m, N = 100, 1000, 30_000
    X, obs = _data(p, n, 4 * m, N)
    B = p.BackendId("b200", 0, "fp32")
    ref = p.train(X, m, p.KernelConfig(), B)
    x = _dev(obs, torch.float32)
    e_full, r_full = torch.empty_like(x.T).T, torch.empty_like(x.T).T
    p.estimate_device(ref, x, e_full, r_full)
    torch.cuda.synchronize()
    e_full, r_full = e_full.cpu().numpy(), r_full.cpu().numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, n, m, N)) for r in range(2)]
    for pr in procs:
        pr.start()
    got = [q.get(timeout=400) for _ in range(2)]
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    e, r = np.full_like(e_full, np.nan), np.full_like(r_full, np.nan)
    for rank, a, b, nbytes, es, rs, pinv in got:
        e[a:b], r[a:b] = es, rs
        assert np.array_equal(pinv, ref.export()["gram_pinv"])  # train is deterministic
    assert got[0][3] == got[1][3] > 0
    assert np.array_equal(e, e_full) and np.array_equal(r, r_full)
