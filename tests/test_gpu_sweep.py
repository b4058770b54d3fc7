"""GPU tests of the device data feed and the Monte Carlo sweep driver
(ports of test_sweep.cpp run_cell / run_sweep cases with the B200 backend)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def p():
    import torch  # noqa: F401
    import paper_2003_08011_b200 as p
    p.context(0)
    p.symmetric_eig(np.eye(2), p.BackendId())
    return p


@pytest.mark.parametrize("args", [(1, 5000, 0.0, 0.0, 1.0, 0.0, 3.0, 7),
                                  (5, 3000, 0.5, 0.3, 1.0, 0.5, 4.0, 123),
                                  (64, 20000, 0.8, 0.9, 2.0, 1.0, 5.0, 99),
                                  (3, 2500, -0.4, 0.2, 1.0, -0.5, 4.0, 5)])
def test_device_synthesis_matches_host(p, args):
    host = p.synthesize(p.SignalSpec.uniform(*args)).data
    dev = p.synthesize_device(p.SignalSpec.uniform(*args)).cpu().numpy()
    assert dev.shape == host.shape
    # same recipe; libm, the AR(1) scan and the closed-form Cholesky differ
    # from the sequential host feed only in the last bits
    assert np.abs(dev - host).max() <= 1e-9 * np.abs(host).max()


def test_device_synthesis_long_chunks(p):
    # n x N large enough for the longest chunk length (1024) and a ragged
    # last chunk; the shapes above run 32-128 sample chunks
    args = (80, 1_000_000, 0.5, 0.3, 1.0, 0.5, 4.0, 20260810)
    host = p.synthesize(p.SignalSpec.uniform(*args)).data
    dev = p.synthesize_device(p.SignalSpec.uniform(*args)).cpu().numpy()
    assert np.abs(dev - host).max() <= 1e-9 * np.abs(host).max()


def test_device_synthesis_fp32_output(p):
    import torch
    for args in [(7, 3000, 0.5, 0.3, 1.0, 0.5, 4.0, 5), (100, 100_000, 0.5, 0.3, 1.0, 0.5, 4.0, 6)]:
        spec = p.SignalSpec.uniform(*args)
        a = p.synthesize_device(spec).float()
        b = p.synthesize_device(spec, dtype=torch.float32)
        assert b.dtype == torch.float32 and b.shape == a.shape and b.stride() == a.stride()
        assert torch.equal(a, b)


def test_device_synthesis_statistics(p):
    x = p.synthesize_device(p.SignalSpec.uniform(2, 200000, 0.8, 0.9, 1.0, 0.0, 3.0, 11)).cpu().numpy()
    assert 0.85 < np.corrcoef(x[:, 0], x[:, 1])[0, 1] < 0.95
    c = x[:, 0] - x[:, 0].mean()
    assert 0.75 < (c[:-1] * c[1:]).sum() / (c * c).sum() < 0.85


def test_train_device_matches_host_train(p, oracle):
    X = oracle.synthesize_uniform(20, 400, 0.5, 0.3, 1.0, 0.5, 4.0, 3)
    import torch
    d = torch.tensor(X.T.copy(), device="cuda").T
    a = p.train_device(d, 100, p.KernelConfig(), p.BackendId()).export()
    b = p.train(X, 100, p.KernelConfig(), p.BackendId()).export()
    assert a["source_indices"].tolist() == b["source_indices"].tolist()
    assert np.array_equal(a["gram_pinv"], b["gram_pinv"])


def test_run_cell_samples_and_seeds(p):
    from paper_2003_08011_b200.sweep import CellCoords, SweepConfig, SweepGrid, run_cell
    from paper_2003_08011_b200 import BackendId
    cfg = SweepConfig(SweepGrid([2], [32], [4, 8]), replicates=3, warmups=1, master_seed=1234,
                      backends=[BackendId("b200", 0, "fp32"), BackendId("b200", 0, "fp64")])
    cells = run_cell(CellCoords(2, 32, 4), cfg)
    assert len(cells) == 4
    for c in cells:
        assert not c.excluded and len(c.samples) == 3 and all(s > 0 for s in c.samples)
        assert c.data_seeds == cells[0].data_seeds
    again = run_cell(CellCoords(2, 32, 4), cfg)
    assert again[0].data_seeds == cells[0].data_seeds


def test_run_sweep_holes_and_runtime_exclusion(p):
    from paper_2003_08011_b200.sweep import SweepConfig, SweepGrid, run_sweep
    cfg = SweepConfig(SweepGrid([2], [32], [2, 4]), replicates=2, warmups=0, master_seed=1234)
    calls = []
    s = run_sweep(cfg, lambda i, tot, c, r: calls.append(tot))
    assert calls == [2, 2] and len(s.cells) == 4
    assert [c.reason for c in s.cells if c.excluded] == ["m<2n", "m<2n"]
    cfg.signal_template.skewness, cfg.signal_template.kurtosis = 2.0, 6.0
    s = run_sweep(cfg)
    assert all(c.excluded for c in s.cells)
    assert all("Fleishman" in c.reason for c in s.cells if c.coords.n_memory == 4)


def test_sweep_large_cell_runs(p):
    # one C4-grid corner cell end to end on the device (n=100, N=1e5, m=1000)
    from paper_2003_08011_b200.sweep import CellCoords, SweepConfig, SweepGrid, run_cell
    cfg = SweepConfig(SweepGrid([100], [100_000], [1000]), replicates=1, warmups=0, master_seed=20260810)
    cfg.signal_template.ar_coefficient, cfg.signal_template.cross_correlation = 0.5, 0.3
    cfg.signal_template.skewness, cfg.signal_template.kurtosis = 0.5, 4.0
    cells = run_cell(CellCoords(100, 100_000, 1000), cfg)
    assert not any(c.excluded for c in cells)


def test_sweep_surface_files_and_speedup(p, tmp_path):
    # acceptance.cpp:368-414 analogue: a two-backend sweep's cost CSV and
    # surface JSON re-export byte-identically; the speedup surface of the
    # FP64 path over the tcgen05 FP32 path has the grid's holes
    from paper_2003_08011_b200 import BackendId
    from paper_2003_08011_b200.surfaces import (cells_for_phase, export_cost_csv, export_speedup_csv,
                                                export_surface_json, import_cost_csv, import_surface_json,
                                                speedup)
    from paper_2003_08011_b200.sweep import Phase, SweepConfig, SweepGrid, run_sweep
    f64, f32 = BackendId("b200", 0, "fp64"), BackendId("b200", 0, "fp32")
    cfg = SweepConfig(SweepGrid([2, 8], [2000], [8, 64]), replicates=2, warmups=1, master_seed=20260810,
                      backends=[f64, f32])
    s = run_sweep(cfg)
    c1, c2 = tmp_path / "c1.csv", tmp_path / "c2.csv"
    export_cost_csv(cells_for_phase(s, Phase.train), str(c1))
    export_cost_csv(import_cost_csv(str(c1)), str(c2))
    assert c1.read_bytes() == c2.read_bytes()
    j1, j2 = tmp_path / "s1.json", tmp_path / "s2.json"
    export_surface_json(s, str(j1))
    export_surface_json(import_surface_json(str(j1)), str(j2))
    assert j1.read_bytes() == j2.read_bytes()
    sp = speedup(s, f64, f32)
    holes = [c for c in sp.cells if c.hole]
    assert len(holes) == 2 and all(c.reason == "m<2n" for c in holes)  # (8, 2000, 8) train + surveil
    assert all(c.speedup > 0 for c in sp.cells if not c.hole)
    export_speedup_csv(sp, Phase.surveil, str(tmp_path / "sp.csv"))


def test_sweep_gpu_vs_host_speedup_surface(p, tmp_path):
    # sweep.cpp:206-227: every backend of a replicate runs inside one
    # run_cell, so host and GPU cells share the surface and speedup()
    # (surfaces.cpp:100-145) gives the GPU-vs-host ratio directly.  The host
    # backend is the CPU oracle registered as the reference's "optimized"
    # kind (baseline leg; the library itself never computes on the CPU).
    from oracle import host_backend
    from paper_2003_08011_b200 import BackendId
    from paper_2003_08011_b200.surfaces import export_speedup_csv, export_surface_json, import_surface_json, speedup
    from paper_2003_08011_b200.sweep import Phase, SweepConfig, SweepGrid, run_sweep
    host_backend.register()
    try:
        cpu, gpu = BackendId.optimized(4, 64), BackendId("b200", 0, "fp32")
        cfg = SweepConfig(SweepGrid([10, 20], [2000], [40, 100]), replicates=2, warmups=1,
                          master_seed=20260810, backends=[cpu, gpu])
        s = run_sweep(cfg)
        assert len(s.cells) == 4 * 2 * 2
        assert not any(c.excluded for c in s.cells)
        sp = speedup(s, cpu, gpu)
        # surveillance is faster on the B200 in every cell; training of these
        # tiny models (m <= 100, 4m rows) may not be (launch latency)
        assert all(c.speedup > 1.0 for c in sp.cells if not c.hole and c.phase == Phase.surveil)
        assert all(c.speedup > 0.0 for c in sp.cells if not c.hole)
        export_speedup_csv(sp, Phase.surveil, str(tmp_path / "sp.csv"))
        export_surface_json(s, str(tmp_path / "s.json"))
        back = import_surface_json(str(tmp_path / "s.json"))
        assert {c.backend for c in back.cells} == {cpu, gpu}
    finally:
        host_backend.unregister()


def test_cli_sweep_then_speedup(p, tmp_path, capsys):
    """python -m paper_2003_08011_b200 sweep / speedup (tools/main.cpp:142-275)
    end to end on the GPU: a 2 x 2 grid with one inadmissible cell, FP64 and
    FP32 B200 backends, then the FP64 / FP32 speedup surface."""
    import json
    from paper_2003_08011_b200 import cli
    cfg = {"grid": {"signal_counts": [4, 40], "observation_counts": [3000], "memory_counts": [40, 64]},
           "replicates": 2, "warmups": 1, "master_seed": 20260810,
           "backends": [{"kind": "b200", "device": 0, "precision": "fp64"},
                        {"kind": "b200", "device": 0, "precision": "fp32"}],
           "signals": {"ar_coefficient": 0.5, "cross_correlation": 0.3, "skewness": 0.5, "kurtosis": 4.0}}
    path = tmp_path / "c.json"
    path.write_text(json.dumps(cfg))
    out = tmp_path / "sweep"
    assert cli.main(["sweep", "--config", str(path), "--out", str(out)]) == 0
    captured = capsys.readouterr()
    assert "excluded (m<2n)" in captured.err  # n = 40, m = 40, 64: m < 2n
    assert "b200[device=0/precision=fp32]" in captured.out
    surface = p.surfaces.import_surface_json(str(out / "surface.json"))
    live = [c for c in surface.cells if not c.excluded]
    assert len(live) == 2 * 2 * 2 and all(len(c.samples) == 2 and c.median > 0 for c in live)
    man = json.loads((out / "manifest.json").read_text())
    assert man["exit_status"] == 0 and "surface.json" in man["artifacts"]
    sp = tmp_path / "sp"
    assert cli.main(["speedup", "--surface", str(out / "surface.json"), "--ref",
                     "b200[device=0/precision=fp64]", "--opt", "b200[device=0/precision=fp32]",
                     "--out", str(sp)]) == 0
    rows = (sp / "speedup_surveil.csv").read_text().splitlines()
    assert len(rows) == 1 + 4  # header + every grid cell (holes included)
