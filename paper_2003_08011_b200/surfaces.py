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
