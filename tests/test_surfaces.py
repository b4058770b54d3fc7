"""Speedup surface and cost / speedup CSV files (ports of test_surfaces.cpp
81-109, 253-285, 332-359 with the b200 backends standing in for the
reference's reference / optimized kinds).  CPU only."""
import math

import pytest

from paper_2003_08011_b200.errors import IoError
from paper_2003_08011_b200.mset import BackendId
from paper_2003_08011_b200.surfaces import (UnknownBackend, export_cost_csv, export_speedup_csv,
                                            import_cost_csv, speedup)
from paper_2003_08011_b200.sweep import CellCoords, CostCell, CostSurface, Phase

REF = BackendId("b200", 0, "fp64")
OPT = BackendId("b200", 0, "fp32")


def make_cell(n, N, m, phase, backend, seconds):
    c = CostCell(CellCoords(n, N, m), phase, backend)
    c.samples = [seconds, seconds, seconds]
    c.recompute_aggregates()
    return c


def make_excluded(n, N, m, phase, backend, reason):
    return CostCell(CellCoords(n, N, m), phase, backend, excluded=True, reason=reason)


def test_recompute_aggregates_reference_order():
    c = CostCell(CellCoords(2, 64, 8), Phase.train, REF)
    c.samples = [1.0, 2.0, 3.0, 4.0]
    c.recompute_aggregates()
    assert (c.mean, c.median) == (2.5, 2.5)
    assert c.stddev == math.sqrt(5.0 / 3.0)
    # plain left-to-right sum (sweep.cpp:83-86): 1e16 + 1 rounds to 1e16
    c.samples = [1e16, 1.0, -1e16]
    c.recompute_aggregates()
    assert c.mean == 0.0


def test_speedup_self_ratio_definition_and_holes():
    slow = make_cell(2, 64, 8, Phase.train, REF, 0.0)
    slow.samples = [10.0, 10.0, 10.0]
    slow.recompute_aggregates()
    fast = make_cell(2, 64, 8, Phase.train, OPT, 0.0)
    fast.samples = [0.1, 0.1, 0.1]
    fast.recompute_aggregates()
    surface = CostSurface([slow, fast, make_excluded(8, 64, 8, Phase.train, REF, "m<2n"),
                           make_excluded(8, 64, 8, Phase.train, OPT, "m<2n")], {})
    for cell in speedup(surface, REF, REF).cells:
        if not cell.hole:
            assert cell.speedup == 1.0
    sp = speedup(surface, REF, OPT)
    assert len(sp.cells) == 2
    assert not sp.cells[0].hole and sp.cells[0].speedup == pytest.approx(100.0)
    assert sp.cells[1].hole and sp.cells[1].reason == "m<2n"
    with pytest.raises(UnknownBackend):
        speedup(surface, REF, BackendId("b200", 7, "fp32"))


def test_speedup_one_sided_holes():
    surface = CostSurface([make_cell(2, 64, 8, Phase.train, REF, 1.0),
                           make_excluded(2, 64, 8, Phase.train, OPT, "EigFailure"),
                           make_cell(2, 64, 16, Phase.train, REF, 1.0),
                           make_cell(4, 64, 16, Phase.train, OPT, 1.0)], {})
    cells = speedup(surface, REF, OPT).cells
    assert cells[0].hole and cells[0].reason == OPT.label() + ": EigFailure"
    assert cells[1].hole and cells[1].reason == "missing " + OPT.label()
    assert cells[2].hole and cells[2].reason == "missing " + REF.label()


def test_cost_csv_export_import_export_byte_identical(tmp_path):
    cells = [make_cell(2, 64, 8, Phase.train, REF, 0.125), make_cell(2, 64, 8, Phase.train, OPT, 0.03125),
             make_excluded(8, 64, 8, Phase.train, REF, "m<2n")]
    cells[0].samples = [0.1, 0.2, 0.30000001]  # non-representable decimals
    cells[0].recompute_aggregates()
    p1, p2 = tmp_path / "a.csv", tmp_path / "b.csv"
    export_cost_csv(cells, str(p1))
    imported = import_cost_csv(str(p1))
    assert len(imported) == len(cells)
    assert imported[0].samples == cells[0].samples and imported[0].median == cells[0].median
    assert imported[2].excluded and imported[2].reason == "m<2n"
    assert imported[1].backend == OPT
    export_cost_csv(imported, str(p2))
    assert p1.read_bytes() == p2.read_bytes()
    text = p1.read_text()
    assert text.startswith("phase,backend,n_signals,n_observations,n_memory,excluded,"
                           "reason,median_s,mean_s,std_s,samples\n")
    assert "true,m<2n,,,," in text


def test_cost_csv_import_errors(tmp_path):
    bad = tmp_path / "bad.csv"
    bad.write_text("phase,backend\n")
    with pytest.raises(IoError):
        import_cost_csv(str(bad))
    p = tmp_path / "c.csv"
    export_cost_csv([make_cell(2, 64, 8, Phase.train, REF, 0.5)], str(p))
    lines = p.read_text().split("\n")
    p.write_text("\n".join([lines[0], lines[1].replace(",0.5,0.5,0,", ",0.25,0.5,0,")]) + "\n")
    with pytest.raises(IoError, match="aggregates do not match"):
        import_cost_csv(str(p))
    p.write_text("\n".join([lines[0], lines[1] + ",extra"]) + "\n")
    with pytest.raises(IoError, match="expected 11 fields"):
        import_cost_csv(str(p))


def test_speedup_csv_export(tmp_path):
    surface = CostSurface([make_cell(2, 64, 8, Phase.train, REF, 1.0), make_cell(2, 64, 8, Phase.train, OPT, 0.5),
                           make_cell(2, 64, 8, Phase.surveil, REF, 2.0),
                           make_cell(2, 64, 8, Phase.surveil, OPT, 0.5)], {})
    path = tmp_path / "speedup_train.csv"
    export_speedup_csv(speedup(surface, REF, OPT), Phase.train, str(path))
    text = path.read_text()
    assert text.startswith("phase,backend_ref,backend_opt,n_signals,n_observations,"
                           "n_memory,hole,reason,speedup\n")
    assert f"train,{REF.label()},{OPT.label()},2,64,8,false,,2\n" in text
    assert "surveil," not in text


def test_surface_json_round_trip_byte_identical(tmp_path):
    from paper_2003_08011_b200.surfaces import export_surface_json, import_surface_json
    cells = [make_cell(2, 64, 8, Phase.train, REF, 0.125), make_cell(2, 64, 8, Phase.surveil, OPT, 1e-05),
             make_excluded(8, 64, 8, Phase.train, REF, "m<2n")]
    cells[0].samples = [0.1, 0.2, 0.30000001]
    cells[0].data_seeds = [2**64 - 1, 12345, 0]
    cells[0].recompute_aggregates()
    meta = {"generator": "containerstress-b200 0.1.0", "host_description": "x86_64 / Linux",
            "hardware_threads": 16, "timer": "wall_monotonic", "rng_algorithm": "splitmix64",
            "world_size": 2, "placement": "LPT", "started_at": "2026-10-17T00:00:00Z",
            "finished_at": "2026-10-17T00:00:01Z", "backend_capabilities": ["fp64 path", "fp32 path"]}
    s1, s2 = tmp_path / "s1.json", tmp_path / "s2.json"
    export_surface_json(CostSurface(cells, meta), str(s1))
    back = import_surface_json(str(s1))
    assert [c.samples for c in back.cells] == [c.samples for c in cells]
    assert back.cells[0].data_seeds == cells[0].data_seeds
    assert back.cells[0].median == cells[0].median and back.cells[2].excluded
    assert back.cells[1].backend == OPT
    export_surface_json(back, str(s2))
    assert s1.read_bytes() == s2.read_bytes()
    text = s1.read_text()
    assert '"format": "containerstress-surface"' in text and '"version": 1' in text
    bad = tmp_path / "bad.json"
    bad.write_text(text.replace("containerstress-surface", "other"))
    with pytest.raises(IoError):
        import_surface_json(str(bad))
