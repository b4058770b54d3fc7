"""Sweep driver logic on CPU: grid walk, admissibility, aggregates, validation
(ports of test_sweep.cpp), LPT placement, and the multi-rank gather +
reassembly over a world_size-2 gloo group (no GPU: units are faked)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2003_08011_b200 import errors
from paper_2003_08011_b200.sweep import (CellCoords, CostCell, Phase, SweepConfig, SweepGrid,
                                         generate_cells, plan_units, predicted_cost, run_sweep)


def test_generate_cells_applies_training_constraint():
    # test_sweep.cpp:30-46
    cells = generate_cells(SweepGrid([32, 64], [1024], [32, 64, 128]))
    assert len(cells) == 6
    adm = {(c.n_signals, c.n_memory) for c, ok in cells if ok}
    exc = {(c.n_signals, c.n_memory) for c, ok in cells if not ok}
    assert adm == {(32, 64), (32, 128), (64, 128)}
    assert exc == {(32, 32), (64, 32), (64, 64)}


def test_generate_cells_order():
    # test_sweep.cpp:48-59
    cells = generate_cells(SweepGrid([1, 2], [10, 20], [4, 8]))
    assert [c for c, _ in cells][:5] == [CellCoords(1, 10, 4), CellCoords(1, 20, 4), CellCoords(1, 10, 8),
                                         CellCoords(1, 20, 8), CellCoords(2, 10, 4)]


def test_powers_of_two_grid_and_boundary():
    # test_sweep.cpp:61-78 / acceptance criterion 3
    g = SweepGrid([32 << k for k in range(6)], [1024], [128 << k for k in range(7)])
    cells = generate_cells(g)
    assert len(cells) == 42
    assert all(ok == (c.n_memory >= 2 * c.n_signals) for c, ok in cells)
    assert generate_cells(SweepGrid([1], [8], [2]))[0][1]


def test_grid_and_config_validation():
    # test_sweep.cpp:80-89, :223-238
    with pytest.raises(errors.ConfigError):
        SweepGrid([], [8], [2]).validate()
    with pytest.raises(errors.ConfigError):
        SweepGrid([4, 4], [8], [2]).validate()
    with pytest.raises(errors.ConfigError):
        SweepGrid([4, 2], [8], [2]).validate()
    g = SweepGrid([2], [32], [4, 8])
    for bad in (dict(replicates=0), dict(backends=[]), dict(estimator="neural-net")):
        with pytest.raises(errors.ConfigError):
            SweepConfig(g, **bad).validate()
    cfg = SweepConfig(g)
    cfg.signal_template.kurtosis = 1.0
    with pytest.raises(errors.ConfigError):
        cfg.validate()


def test_aggregate_arithmetic():
    # test_sweep.cpp:205-221
    c = CostCell(CellCoords(1, 1, 2), Phase.train, None, samples=[3.0, 1.0, 2.0])
    c.recompute_aggregates()
    assert c.median == 2.0 and abs(c.mean - 2.0) < 1e-12 and abs(c.stddev - 1.0) < 1e-12
    c.samples = [4.0, 1.0, 2.0, 3.0]
    c.recompute_aggregates()
    assert c.median == 2.5
    c.samples = [5.0]
    c.recompute_aggregates()
    assert c.median == 5.0 and c.stddev == 0.0


def test_lpt_plan_covers_every_unit_once_and_balances():
    cells = [c for c, ok in generate_cells(SweepGrid([10, 20, 50, 100, 200, 500, 1000],
                                                     [10_000, 100_000, 1_000_000],
                                                     [100, 200, 500, 1000, 2000, 4000])) if ok]
    assert len(cells) == 96
    units = [(i, c, r) for i, c in enumerate(cells) for r in range(5)]
    one = sum(predicted_cost(c) * 6 for c in cells)  # 5 replicates + 1 warm-up per cell
    for world in (1, 2, 4, 8):
        plan = plan_units(units, world)
        flat = sorted(u[:1] + u[2:] for p in plan for u in p)
        assert flat == sorted(u[:1] + u[2:] for u in units)
        # the work each rank really runs: its units plus one warm-up per (cell, rank)
        loads = [sum(predicted_cost(u[1]) for u in p) + sum(predicted_cost(cells[i]) for i in {u[0] for u in p})
                 for p in plan]
        assert one / world / max(loads) > 0.95  # near-linear 1 -> 8, warm-ups included
        assert plan == plan_units(units, world)  # deterministic


def _fake_unit(coords, replicate, config, device, warm):
    # deterministic stand-in for the timed unit (pure function of the unit)
    rec = {"coords": (coords.n_signals, coords.n_observations, coords.n_memory),
           "replicate": replicate, "seed": 1000 * coords.n_memory + replicate,
           "train": [1e-3 * coords.n_memory + replicate],
           "surveil": [1e-6 * coords.n_observations + replicate], "error": None,
           "error_kind": None}
    if coords.n_signals == 3 and replicate == 1:
        rec["error"], rec["error_kind"] = "no real Fleishman solution", "MomentInfeasible"
    return rec


def _sweep_config():
    return SweepConfig(SweepGrid([1, 2, 3], [16, 32], [2, 4, 8]), replicates=3, warmups=0)


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s = run_sweep(_sweep_config(), world=world, rank=rank, unit_runner=_fake_unit)
    if rank == 0:
        q.put([(c.coords, c.phase.value, c.samples, c.data_seeds, c.excluded, c.reason) for c in s.cells])
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_gloo_sweep_matches_single_rank():
    single = run_sweep(_sweep_config(), unit_runner=_fake_unit)
    want = [(c.coords, c.phase.value, c.samples, c.data_seeds, c.excluded, c.reason) for c in single.cells]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    got = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert got == want
    # grid order, exclusions and per-replicate sample order survive placement
    reasons = {r for *_, ex, r in got if ex}
    assert reasons == {"m<2n", "no real Fleishman solution"}
    assert len(got) == 18 * 2  # 18 grid cells x 2 phases x 1 backend


# ------------------------------------------------------- host backend kinds
def test_backend_id_label_parse_validate():
    # test_backends.cpp:159-171 plus the b200 kind
    from paper_2003_08011_b200 import BackendId
    assert BackendId.reference().label() == "reference"
    o = BackendId.optimized(4, 32)
    assert o.label() == "optimized[tile=32/workers=4]"
    assert BackendId.parse(o.label()) == o
    assert BackendId.parse("reference") == BackendId.reference()
    assert BackendId.parse("b200[device=1/precision=fp32]") == BackendId("b200", 1, "fp32")
    for bad in ("optimized[tile=4/workers=2]", "optimized[tile=64/workers=-1]", "gpu"):
        with pytest.raises(errors.ConfigError):
            BackendId.parse(bad)
    from paper_2003_08011_b200.surfaces import backend_from_json, backend_to_json
    for b in (BackendId.reference(), o, BackendId("b200", 0, "fp64")):
        assert backend_from_json(backend_to_json(b)) == b


def test_host_backend_requires_registration_and_matches_oracle(oracle):
    import numpy as np
    from oracle import host_backend
    from paper_2003_08011_b200 import BackendId, KernelConfig, algorithm_by_name
    algo = algorithm_by_name("mset2")
    X = oracle.synthesize_uniform(4, 80, 0.5, 0.3, 1.0, 0.5, 4.0, 7)
    obs = oracle.synthesize_uniform(4, 50, 0.5, 0.3, 1.0, 0.5, 4.0, 8)
    host_backend.unregister()
    with pytest.raises(errors.ConfigError):
        algo.train(X, 20, KernelConfig(), BackendId.optimized(2))
    host_backend.register()
    try:
        for b in (BackendId.reference(), BackendId.optimized(2, 16)):
            model = algo.train(X, 20, KernelConfig(), b)
            r = algo.estimate(model, obs, b)
            ref = oracle.train(X, 20)
            want_e, want_r = oracle.estimate(ref, obs)
            assert np.abs(r.estimates - want_e).max() <= 1e-10 * np.abs(want_e).max()
            assert np.array_equal(r.residuals, obs - r.estimates)
        # a host model on the b200 backend (and vice versa) is a ConfigError
        # (estimator.cpp:17-23)
        with pytest.raises(errors.ConfigError):
            algo.estimate(model, obs, BackendId("b200", 0, "fp64"))
    finally:
        host_backend.unregister()


def test_sweep_config_echo_in_metadata():
    from paper_2003_08011_b200.sweep import sweep_config_to_json
    s = run_sweep(_sweep_config(), unit_runner=_fake_unit)
    echo = s.metadata["config"]
    assert echo == sweep_config_to_json(_sweep_config())
    assert echo["grid"]["memory_counts"] == [2, 4, 8] and echo["replicates"] == 3
    assert echo["backends"] == [{"kind": "b200", "device": 0, "precision": "fp32"}]


def _boom_unit(coords, replicate, config, device, warm):
    import torch.distributed as dist
    if dist.get_rank() == 1:
        raise MemoryError("simulated device OOM")
    return _fake_unit(coords, replicate, config, device, warm)


def _fatal_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        run_sweep(_sweep_config(), world=world, rank=rank, unit_runner=_boom_unit)
        q.put((rank, "returned"))
    except RuntimeError as e:
        q.put((rank, str(e)))
    dist.destroy_process_group()


def test_non_error_failure_aborts_every_rank_without_hanging():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fatal_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
    assert set(got) == {0, 1}
    assert all("simulated device OOM" in v for v in got.values()), got
