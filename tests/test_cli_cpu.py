"""Strict sweep configuration and the sweep / speedup command line (ports of
the reference's config.cpp contract and tools/main.cpp exit codes and
outputs; the b200 backend kind is this library's extension).  CPU only: the
sweep runs that would train on a GPU are replaced where noted."""
import json
import os

import pytest

from paper_2003_08011_b200 import cli, sweep as sweep_mod
from paper_2003_08011_b200.config import backend_from_json, load_json_file, parse_sweep_config
from paper_2003_08011_b200.errors import ConfigError, IoError
from paper_2003_08011_b200.mset import BackendId, KernelKind
from paper_2003_08011_b200.surfaces import export_surface_json, import_surface_json
from paper_2003_08011_b200.sweep import CellCoords, CostCell, CostSurface, Phase

GRID = {"signal_counts": [2], "observation_counts": [64], "memory_counts": [8]}


def test_defaults_match_the_reference():
    c = parse_sweep_config({"grid": GRID})
    assert (c.replicates, c.warmups, c.master_seed, c.timer, c.estimator) == (5, 1, 0, "wall_monotonic", "mset2")
    assert c.grid.training_observation_factor == 4
    assert c.kernel.kind == KernelKind.inverse_distance and c.kernel.bandwidth is None
    assert c.backends == [BackendId("b200", 0, "fp32")]


def test_full_config_round_trip():
    j = {"grid": dict(GRID, training_observation_factor=3), "replicates": 2, "warmups": 0,
         "backends": ["reference", {"kind": "optimized", "tile_size": 32, "worker_count": 3},
                      {"kind": "b200", "device": 0, "precision": "fp64"}, "b200"],
         "kernel": {"kind": "gaussian", "bandwidth": 1.5},
         "signals": {"ar_coefficient": 0.5, "cross_correlation": 0.3, "variance": 1.0, "skewness": 0.5,
                     "kurtosis": 4.0},
         "master_seed": 20260810, "timer": "process_cpu", "estimator": "mean"}
    c = parse_sweep_config(j)
    assert [b.label() for b in c.backends] == ["reference", "optimized[tile=32/workers=3]",
                                               "b200[device=0/precision=fp64]", "b200[device=0/precision=fp64]"]
    assert c.kernel.kind == KernelKind.gaussian and c.kernel.bandwidth == 1.5
    assert c.signal_template.kurtosis == 4.0 and c.master_seed == 20260810
    echo = sweep_mod.sweep_config_to_json(c)
    assert parse_sweep_config(echo) == c


@pytest.mark.parametrize("j,msg", [
    ({"grid": GRID, "replicate": 3}, 'sweep config: unknown key "replicate"'),
    ({"grid": dict(GRID, extra=1)}, 'grid: unknown key "extra"'),
    ({}, 'sweep config: missing "grid"'),
    ({"grid": dict(GRID, signal_counts=[2.5])}, 'grid: bad value for "signal_counts"'),
    ({"grid": GRID, "replicates": "5"}, 'sweep config: bad value for "replicates"'),
    ({"grid": GRID, "backends": "b200"}, 'sweep config: "backends" must be an array'),
    ({"grid": GRID, "backends": [{"kind": "tpu"}]}, 'backend: unknown kind "tpu"'),
    ({"grid": GRID, "backends": [{"kind": "b200", "tile_size": 8}]}, 'backend: unknown key "tile_size"'),
    ({"grid": GRID, "backends": [{"kind": "b200", "precision": "fp16"}]}, "unknown precision"),
    ({"grid": GRID, "kernel": {"kind": "cosine"}}, 'kernel: unknown kind "cosine"'),
    ({"grid": GRID, "kernel": {"bandwidth": -1.0}}, "bandwidth must be > 0"),
    ({"grid": GRID, "signals": {"phi": 0.5}}, 'signals: unknown key "phi"'),
    ({"grid": GRID, "timer": "cycles"}, "unknown timer: cycles"),
    ({"grid": GRID, "estimator": "svm"}, "svm"),
    ({"grid": GRID, "master_seed": -1}, 'sweep config: bad value for "master_seed"'),
    ({"grid": dict(GRID, memory_counts=[8, 8])}, "strictly ascending"),
])
def test_config_errors(j, msg):
    with pytest.raises(ConfigError, match=msg.replace("[", r"\[").replace("(", r"\(")):
        parse_sweep_config(j)


def test_threads_env_override(monkeypatch):
    j = {"grid": GRID, "backends": ["reference", {"kind": "optimized", "worker_count": 2}, "b200"]}
    monkeypatch.setenv("CONTAINERSTRESS_THREADS", "6")
    c = parse_sweep_config(j)
    assert [b.worker_count for b in c.backends if b.kind == "optimized"] == [6]
    assert c.threads_override_note == "env:CONTAINERSTRESS_THREADS=6"
    monkeypatch.setenv("CONTAINERSTRESS_THREADS", "0")
    with pytest.raises(ConfigError, match="CONTAINERSTRESS_THREADS must be a positive integer"):
        parse_sweep_config(j)


def test_load_json_file_errors(tmp_path):
    with pytest.raises(IoError, match="cannot open"):
        load_json_file(str(tmp_path / "missing.json"))
    bad = tmp_path / "bad.json"
    bad.write_text("{")
    with pytest.raises(ConfigError):
        load_json_file(str(bad))


def test_backend_json_forms():
    assert backend_from_json("b200") == BackendId("b200", 0, "fp64")
    assert backend_from_json({"kind": "b200", "device": 1, "precision": "fp32"}) == BackendId("b200", 1, "fp32")
    assert backend_from_json({"kind": "reference"}) == BackendId.reference()


# ---------------------------------------------------------------- the CLI
def _write(tmp_path, j):
    p = tmp_path / "sweep.json"
    p.write_text(json.dumps(j))
    return str(p)


def test_sweep_config_error_exit_2(tmp_path, capsys):
    out = tmp_path / "out"
    assert cli.main(["sweep", "--config", _write(tmp_path, {"grid": GRID, "bogus": 1}), "--out", str(out)]) == 2
    assert 'unknown key "bogus"' in capsys.readouterr().err
    assert not out.exists()  # nothing written before the config is valid (main.cpp:157-160)


def test_argument_error_exit_2():
    assert cli.main(["sweep", "--out", "x"]) == 2
    assert cli.main(["frobnicate"]) == 2


def test_sweep_empty_grid_exit_4(tmp_path, capsys):
    j = {"grid": {"signal_counts": [10], "observation_counts": [64], "memory_counts": [8]}}
    out = tmp_path / "out"
    assert cli.main(["sweep", "--config", _write(tmp_path, j), "--out", str(out)]) == 4
    assert "no grid cell satisfies m >= 2n" in capsys.readouterr().err
    man = json.loads((out / "manifest.json").read_text())
    assert man["command"] == "sweep" and man["exit_status"] == 4


def _fake_unit(coords, replicate, config, device, warm):
    # run_unit's record layout with made-up timings (no GPU work)
    nb = len(config.backends)
    return {"coords": (coords.n_signals, coords.n_observations, coords.n_memory), "replicate": replicate,
            "seed": sweep_mod.cell_data_seed(config.master_seed, coords, replicate),
            "train": [1e-3 * coords.n_memory * (b + 1) for b in range(nb)],
            "surveil": [1e-5 * coords.n_observations * (b + 1) for b in range(nb)], "error": None,
            "error_kind": None}


def test_sweep_outputs_and_speedup(tmp_path, monkeypatch, capsys):
    """Full command flow with the per-unit GPU work replaced: the three
    output files, the manifest, the summary table, then `speedup` between
    the two backends of the surface."""
    monkeypatch.setattr(sweep_mod, "run_unit", _fake_unit)
    j = {"grid": {"signal_counts": [2, 10], "observation_counts": [64], "memory_counts": [8, 32]},
         "replicates": 2, "backends": ["b200", {"kind": "b200", "device": 0, "precision": "fp32"}]}
    out = tmp_path / "out"
    assert cli.main(["sweep", "--config", _write(tmp_path, j), "--out", str(out), "--seed", "7"]) == 0
    for f in ("cost_train.csv", "cost_surveil.csv", "surface.json", "manifest.json"):
        assert (out / f).exists(), f
    surface = import_surface_json(str(out / "surface.json"))
    assert surface.metadata["config"]["master_seed"] == 7
    text = capsys.readouterr().out
    assert "median_min_s" in text and "b200[device=0/precision=fp32]" in text
    sp = tmp_path / "sp"
    assert cli.main(["speedup", "--surface", str(out / "surface.json"), "--ref",
                     "b200[device=0/precision=fp64]", "--opt", "b200[device=0/precision=fp32]",
                     "--out", str(sp)]) == 0
    assert (sp / "speedup_train.csv").exists() and (sp / "speedup_surveil.csv").exists()
    assert "holes" in capsys.readouterr().out


def test_sweep_runtime_failure_keeps_partial_output(tmp_path, monkeypatch, capsys):
    def boom(*a, **k):
        raise MemoryError("device out of memory")
    monkeypatch.setattr(sweep_mod, "run_unit", boom)
    out = tmp_path / "out"
    assert cli.main(["sweep", "--config", _write(tmp_path, {"grid": GRID, "replicates": 1}), "--out", str(out)]) == 5
    assert "sweep aborted" in capsys.readouterr().err
    surface = import_surface_json(str(out / "surface.json"))
    assert surface.metadata["partial"] is True
    assert json.loads((out / "manifest.json").read_text())["exit_status"] == 5


def _surface(tmp_path, backends):
    cells = []
    for b, s in backends:
        for ph in (Phase.train, Phase.surveil):
            c = CostCell(CellCoords(2, 64, 8), ph, b)
            c.samples = [s, s, s]
            c.recompute_aggregates()
            cells.append(c)
    path = str(tmp_path / "surface.json")
    export_surface_json(CostSurface(cells, {}), path)
    return path


def test_speedup_resolves_bare_kinds(tmp_path, capsys):
    path = _surface(tmp_path, [(BackendId.reference(), 10.0), (BackendId("b200", 0, "fp32"), 0.01)])
    assert cli.main(["speedup", "--surface", path, "--ref", "reference", "--opt", "b200",
                     "--out", str(tmp_path / "o")]) == 0
    assert "2 cells, 0 holes (reference vs b200[device=0/precision=fp32])" in capsys.readouterr().out
    rows = (tmp_path / "o" / "speedup_train.csv").read_text().splitlines()
    assert len(rows) == 2 and "1000" in rows[1]


def test_speedup_unknown_and_ambiguous_backends(tmp_path, capsys):
    path = _surface(tmp_path, [(BackendId("b200", 0, "fp64"), 1.0), (BackendId("b200", 0, "fp32"), 0.5)])
    assert cli.main(["speedup", "--surface", path, "--ref", "b200", "--opt", "b200", "--out",
                     str(tmp_path / "o")]) == 2
    assert "ambiguous" in capsys.readouterr().err
    assert cli.main(["speedup", "--surface", path, "--ref", "optimized", "--opt", "b200[device=0/precision=fp32]",
                     "--out", str(tmp_path / "o2")]) == 2
    assert "not present in this surface" in capsys.readouterr().err
    assert os.path.exists(tmp_path / "o2") is False


def _cli_rank(rank, world, port, cfg_path, out_dir, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK="0", CSB_DIST_BACKEND="gloo")
    from paper_2003_08011_b200 import cli as c, sweep as sm
    sm.run_unit = _fake_unit
    q.put((rank, c.main(["sweep", "--config", cfg_path, "--out", out_dir])))


def test_cli_sweep_two_ranks_gloo(tmp_path):
    """`torchrun -m paper_2003_08011_b200 sweep` with world size 2 (gloo, no
    GPU work): rank 0 writes the same surface as a single-rank run."""
    import socket
    import torch.multiprocessing as mp
    j = {"grid": {"signal_counts": [2, 4], "observation_counts": [64, 128], "memory_counts": [8, 16]},
         "replicates": 3, "backends": ["b200"], "master_seed": 5}
    cfg = _write(tmp_path, j)
    import paper_2003_08011_b200.sweep as sm
    orig = sm.run_unit
    sm.run_unit = _fake_unit
    try:
        assert cli.main(["sweep", "--config", cfg, "--out", str(tmp_path / "one")]) == 0
    finally:
        sm.run_unit = orig
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_cli_rank, args=(r, 2, port, cfg, str(tmp_path / "two"), q)) for r in range(2)]
    for pr in procs:
        pr.start()
    codes = dict(q.get(timeout=180) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    assert codes == {0: 0, 1: 0}
    one = json.loads((tmp_path / "one" / "surface.json").read_text())
    two = json.loads((tmp_path / "two" / "surface.json").read_text())
    assert one["cells"] == two["cells"]
