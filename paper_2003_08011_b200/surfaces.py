"""Cost-surface consumers of the sweep: the GPU-vs-host speedup surface and
the cost / speedup CSV files (surfaces.cpp:100-145, 341-407, 520-537).

`speedup(surface, ref, opt)` pairs every (cell, phase) of a surface that
holds both backends and divides the reference backend's median by the
optimised one's; cells where either side is missing or excluded become
holes carrying the reference's reason texts.  The CSV writers format
doubles with "%.17g" (surfaces.cpp:21-25), so `import_cost_csv` of an
exported file reproduces the cells exactly and re-checks their aggregates
(surfaces.cpp:366-407).
"""
from dataclasses import dataclass, field
from typing import List, Optional

from .errors import ConfigError, IoError
from .mset import BackendId
from .sweep import CellCoords, CostCell, CostSurface, Phase

COST_CSV_HEADER = ("phase,backend,n_signals,n_observations,n_memory,excluded,reason,"
                   "median_s,mean_s,std_s,samples")  # surfaces.cpp:310-312
SPEEDUP_CSV_HEADER = ("phase,backend_ref,backend_opt,n_signals,n_observations,n_memory,"
                      "hole,reason,speedup")  # surfaces.cpp:524-525


class UnknownBackend(ConfigError):
    """surfaces.cpp:97, 108-111 (UnknownBackend)."""


@dataclass
class SpeedupCell:
    """surfaces.hpp SpeedupCell."""
    coords: CellCoords
    phase: Phase
    hole: bool = False
    reason: str = ""
    speedup: float = 0.0


@dataclass
class SpeedupSurface:
    reference_backend: BackendId
    optimized_backend: BackendId
    cells: List[SpeedupCell] = field(default_factory=list)


def _fmt(v: float) -> str:
    return "%.17g" % v  # surfaces.cpp:21-25


def surface_backends(surface: CostSurface) -> List[BackendId]:
    """surfaces.cpp:64-71: distinct backends in first-seen order."""
    out: List[BackendId] = []
    for c in surface.cells:
        if c.backend not in out:
            out.append(c.backend)
    return out


def speedup(surface: CostSurface, ref: BackendId, opt: BackendId) -> SpeedupSurface:
    """surfaces.cpp:100-145."""
    present = surface_backends(surface)
    if ref not in present:
        raise UnknownBackend(f"reference backend {ref.label()} not present in surface")
    if opt not in present:
        raise UnknownBackend(f"optimized backend {opt.label()} not present in surface")
    out = SpeedupSurface(ref, opt)
    seen = []
    for cell in surface.cells:
        key = (cell.coords, cell.phase)
        if key in seen:
            continue
        seen.append(key)
        rc: Optional[CostCell] = surface.find(cell.coords, cell.phase, ref)
        oc: Optional[CostCell] = surface.find(cell.coords, cell.phase, opt)
        sp = SpeedupCell(cell.coords, cell.phase)
        if rc is None or oc is None:
            sp.hole = True
            sp.reason = "missing " + (ref.label() if rc is None else opt.label())
        elif rc.excluded and oc.excluded:
            sp.hole = True
            sp.reason = rc.reason
        elif rc.excluded or oc.excluded:
            bad = rc if rc.excluded else oc
            sp.hole = True
            sp.reason = bad.backend.label() + ": " + bad.reason
        else:
            sp.speedup = rc.median / oc.median
        out.cells.append(sp)
    return out


def cells_for_phase(surface: CostSurface, phase: Phase) -> List[CostCell]:
    """surfaces.cpp:409-416."""
    return [c for c in surface.cells if c.phase == phase]


def export_cost_csv(cells: List[CostCell], path: str) -> None:
    """surfaces.cpp:341-364."""
    try:
        with open(path, "w", newline="") as f:
            f.write(COST_CSV_HEADER + "\n")
            for c in cells:
                row = (f"{c.phase.value},{c.backend.label()},{c.coords.n_signals},"
                       f"{c.coords.n_observations},{c.coords.n_memory},"
                       f"{'true' if c.excluded else 'false'},{c.reason},")
                if not c.excluded:
                    row += f"{_fmt(c.median)},{_fmt(c.mean)},{_fmt(c.stddev)},"
                    row += ";".join(_fmt(s) for s in c.samples)
                else:
                    row += ",,,"
                f.write(row + "\n")
    except OSError as e:
        raise IoError(f"export_cost_csv: cannot open {path}") from e


def _parse_double(s: str, context: str) -> float:
    try:
        return float(s)
    except ValueError:
        raise IoError(f"{context}: bad number \"{s}\"") from None


def _parse_index(s: str, context: str) -> int:
    try:
        return int(s)
    except ValueError:
        raise IoError(f"{context}: bad integer \"{s}\"") from None


def import_cost_csv(path: str) -> List[CostCell]:
    """surfaces.cpp:366-407: exact round trip of export_cost_csv; the stored
    aggregates must equal the ones recomputed from the samples."""
    try:
        lines = open(path, newline="").read().split("\n")
    except OSError:
        raise IoError(f"import_cost_csv: cannot open {path}") from None
    if not lines or lines[0] != COST_CSV_HEADER:
        raise IoError(f"import_cost_csv: bad header in {path}")
    cells: List[CostCell] = []
    for lineno, line in enumerate(lines[1:], start=2):
        if not line:
            continue
        context = f"{path}:{lineno}"
        fields = line.split(",")
        if len(fields) != 11:
            raise IoError(f"{context}: expected 11 fields, got {len(fields)}")
        if fields[0] not in ("train", "surveil"):
            raise ConfigError("unknown phase: " + fields[0])
        if fields[5] not in ("true", "false"):
            raise IoError(f"{context}: bad excluded flag")
        cell = CostCell(CellCoords(_parse_index(fields[2], context), _parse_index(fields[3], context),
                                   _parse_index(fields[4], context)),
                        Phase(fields[0]), BackendId.parse(fields[1]))
        cell.excluded = fields[5] == "true"
        cell.reason = fields[6]
        if not cell.excluded:
            cell.samples = [_parse_double(s, context) for s in fields[10].split(";") if s]
            cell.recompute_aggregates()
            if (cell.median != _parse_double(fields[7], context) or cell.mean != _parse_double(fields[8], context)
                    or cell.stddev != _parse_double(fields[9], context)):
                raise IoError(f"{context}: aggregates do not match samples")
        cells.append(cell)
    return cells


def export_speedup_csv(surface: SpeedupSurface, phase: Phase, path: str) -> None:
    """surfaces.cpp:520-537."""
    try:
        with open(path, "w", newline="") as f:
            f.write(SPEEDUP_CSV_HEADER + "\n")
            for c in surface.cells:
                if c.phase != phase:
                    continue
                row = (f"{c.phase.value},{surface.reference_backend.label()},"
                       f"{surface.optimized_backend.label()},{c.coords.n_signals},"
                       f"{c.coords.n_observations},{c.coords.n_memory},"
                       f"{'true' if c.hole else 'false'},{c.reason},")
                if not c.hole:
                    row += _fmt(c.speedup)
                f.write(row + "\n")
    except OSError as e:
        raise IoError(f"export_speedup_csv: cannot open {path}") from e


# ------------------------------------------------------------ surface JSON
SURFACE_FORMAT = "containerstress-surface"  # surfaces.cpp:442-443


def backend_to_json(b: BackendId):
    """config.cpp:172-177, extended with the b200 kind."""
    if b.kind == "reference":
        return "reference"
    if b.kind == "optimized":
        return {"kind": "optimized", "tile_size": b.tile_size, "worker_count": b.worker_count}
    return {"kind": b.kind, "device": b.device, "precision": b.precision}


def backend_from_json(j) -> BackendId:
    """config.cpp:159-170 (string token or object), plus the b200 kind."""
    if isinstance(j, str):
        return BackendId.parse(j)
    if not isinstance(j, dict):
        raise ConfigError(f"unknown backend id: {j!r}")
    if j.get("kind") == "reference":
        return BackendId.reference()
    if j.get("kind") == "optimized":
        return BackendId.optimized(int(j.get("worker_count", 0)), int(j.get("tile_size", 64)))
    if j.get("kind") != "b200":
        raise ConfigError(f"unknown backend id: {j!r}")
    b = BackendId("b200", int(j["device"]), str(j["precision"]))
    b.validate()
    return b


def _metadata_json(surface: CostSurface) -> dict:
    m = dict(surface.metadata)
    caps = m.get("backend_capabilities", [])
    if caps and not isinstance(caps[0], dict):  # run_sweep form: descriptions in backend order
        caps = [{"backend": backend_to_json(b), "deterministic_summation": True, "description": d}
                for b, d in zip(surface_backends(surface), caps)]
    known = {"generator", "host_description", "host", "hardware_threads", "timer", "rng_algorithm", "started_at",
             "finished_at", "threads_override", "partial", "config", "backend_capabilities"}
    config = dict(m.get("config", {}))
    config.update({k: v for k, v in m.items() if k not in known})  # world_size, placement, ...
    return {"generator": m.get("generator", ""), "host": m.get("host", m.get("host_description", "")),
            "hardware_threads": int(m.get("hardware_threads") or 0), "timer": m.get("timer", ""),
            "rng_algorithm": m.get("rng_algorithm", ""), "started_at": m.get("started_at", ""),
            "finished_at": m.get("finished_at", ""), "threads_override": m.get("threads_override", ""),
            "partial": bool(m.get("partial", False)), "config": config, "backend_capabilities": caps}


def surface_to_json(surface: CostSurface) -> dict:
    """surfaces.cpp:418-459."""
    cells = []
    for c in surface.cells:
        jc = {"phase": c.phase.value, "backend": backend_to_json(c.backend), "n_signals": c.coords.n_signals,
              "n_observations": c.coords.n_observations, "n_memory": c.coords.n_memory,
              "excluded": c.excluded, "reason": c.reason, "samples": list(c.samples),
              "data_seeds": list(c.data_seeds)}
        if c.samples:
            jc["median_s"], jc["mean_s"], jc["std_s"] = c.median, c.mean, c.stddev
        cells.append(jc)
    return {"format": SURFACE_FORMAT, "version": 1, "metadata": _metadata_json(surface), "cells": cells}


def surface_from_json(j: dict) -> CostSurface:
    """surfaces.cpp:461-507 (aggregates recomputed from the samples)."""
    try:
        if j["format"] != SURFACE_FORMAT:
            raise IoError("surface: unexpected format tag")
        if j["version"] != 1:
            raise IoError("surface: unsupported version")
        meta = dict(j["metadata"])
        meta["backend_capabilities"] = [
            {"backend": backend_to_json(backend_from_json(c["backend"])),
             "deterministic_summation": bool(c["deterministic_summation"]), "description": str(c["description"])}
            for c in meta["backend_capabilities"]]
        cells = []
        for jc in j["cells"]:
            if jc["phase"] not in ("train", "surveil"):
                raise ConfigError("unknown phase: " + str(jc["phase"]))
            c = CostCell(CellCoords(int(jc["n_signals"]), int(jc["n_observations"]), int(jc["n_memory"])),
                         Phase(jc["phase"]), backend_from_json(jc["backend"]))
            c.excluded = bool(jc["excluded"])
            c.reason = str(jc["reason"])
            c.samples = [float(x) for x in jc["samples"]]
            c.data_seeds = [int(x) for x in jc["data_seeds"]]
            c.recompute_aggregates()
            cells.append(c)
        return CostSurface(cells, meta)
    except (KeyError, TypeError, ValueError) as e:
        raise IoError(f"surface: malformed JSON: {e}") from None


def export_surface_json(surface: CostSurface, path: str) -> None:
    """surfaces.cpp:509-514: nlohmann dump(2) layout (sorted keys, two-space
    indent, shortest round-trip doubles) plus a trailing newline."""
    import json
    try:
        with open(path, "w", encoding="utf-8", newline="") as f:
            f.write(json.dumps(surface_to_json(surface), indent=2, sort_keys=True, ensure_ascii=False) + "\n")
    except OSError as e:
        raise IoError(f"export_surface_json: cannot open {path}") from e


def import_surface_json(path: str) -> CostSurface:
    import json
    try:
        with open(path, encoding="utf-8") as f:
            j = json.load(f)
    except OSError:
        raise IoError(f"import_surface_json: cannot open {path}") from None
    except ValueError as e:
        raise IoError(f"surface: malformed JSON: {e}") from None
    return surface_from_json(j)
