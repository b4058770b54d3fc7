"""Monte Carlo scoping sweep on B200s (sweep.hpp:26-109, sweep.cpp:77-325).

Same grid walk, admissibility rule, seeds, warm-up policy, timing brackets
and exclusion semantics as the reference driver; the difference is placement:
the reference walks cells strictly serially on one CPU, here the
independent (cell, replicate) units are spread over the ranks of one node
(one process per GPU) by longest-processing-time-first on a predicted cost,
each rank times its own units on its own device (serial per device, so the
"no concurrent timing on one device" rule holds), and rank 0 gathers the
fixed-size cost records over torch.distributed (NCCL over NVLink on GPUs,
gloo in the CPU tests) and reassembles the surface in the reference's cell
order.  Unit placement never changes the data: every replicate's signals
derive from cell_data_seed(master, coords, r) alone (sweep.cpp:119-126).

Per unit: synthesize the replicate's training (factor * m rows) and
surveillance (N rows) signals on the device (untimed, sweep.cpp:207-208),
then per backend time train and estimate separately with a wall-clock
bracket around synchronous calls (sweep.cpp:212-219), samples clamped to
>= 1e-9 s (sweep.cpp:221-225).
"""
from __future__ import annotations

import dataclasses
import json
import math
import os
import platform
import statistics
import threading
import time
from dataclasses import dataclass, field
from enum import Enum
from typing import Callable, List, Optional, Sequence, Tuple

from . import errors
from .errors import ConfigError, ConstraintViolated, EmptyGrid
from .mset import BackendId, KernelConfig, KernelKind, capabilities

RNG_ALGORITHM = "splitmix64-v1/box-muller"  # rng.hpp:12


class Phase(str, Enum):
    train = "train"
    surveil = "surveil"


@dataclass
class SweepGrid:
    """sweep.hpp:30-37"""
    signal_counts: List[int]
    observation_counts: List[int]
    memory_counts: List[int]
    training_observation_factor: int = 4

    def validate(self) -> None:  # sweep.cpp:79-96
        for name in ("signal_counts", "observation_counts", "memory_counts"):
            values = getattr(self, name)
            if not values:
                raise ConfigError(f"grid: {name} must be non-empty")
            for i, v in enumerate(values):
                if v < 1:
                    raise ConfigError(f"grid: {name} must be positive")
                if i > 0 and v <= values[i - 1]:
                    raise ConfigError(f"grid: {name} must be strictly ascending")
        if self.training_observation_factor < 1:
            raise ConfigError("grid: training_observation_factor must be >= 1")


@dataclass
class SignalStatsTemplate:
    """sweep.hpp:41-47"""
    ar_coefficient: float = 0.0
    cross_correlation: float = 0.0
    variance: float = 1.0
    skewness: float = 0.0
    kurtosis: float = 3.0


@dataclass
class SweepConfig:
    """sweep.hpp:49-62"""
    grid: SweepGrid
    replicates: int = 5
    warmups: int = 1
    backends: List[BackendId] = field(default_factory=lambda: [BackendId("b200", 0, "fp32")])
    kernel: KernelConfig = field(default_factory=KernelConfig)
    signal_template: SignalStatsTemplate = field(default_factory=SignalStatsTemplate)
    master_seed: int = 0
    timer: str = "wall_monotonic"
    estimator: str = "mset2"
    threads_override_note: str = ""  # config.hpp: where a worker-count override came from

    def validate(self) -> None:  # sweep.cpp:98-111
        from .estimator import algorithm_by_name
        self.grid.validate()
        if self.replicates < 1:
            raise ConfigError("sweep: replicates must be >= 1")
        if self.warmups < 0:
            raise ConfigError("sweep: warmups must be >= 0")
        if not self.backends:
            raise ConfigError("sweep: at least one backend is required")
        for b in self.backends:
            b.validate()
        self.kernel.validate()
        algorithm_by_name(self.estimator)
        t = self.signal_template
        if not t.kurtosis > t.skewness * t.skewness + 1.0:
            raise ConfigError("sweep: signal kurtosis violates the Pearson bound")
        if self.timer not in ("wall_monotonic", "process_cpu"):
            raise ConfigError("unknown timer: " + self.timer)


@dataclass(frozen=True)
class CellCoords:
    """sweep.hpp:64-71"""
    n_signals: int
    n_observations: int
    n_memory: int

    def admissible(self) -> bool:
        return self.n_memory >= 2 * self.n_signals


@dataclass
class CostCell:
    """sweep.hpp:73-88"""
    coords: CellCoords
    phase: Phase
    backend: BackendId
    samples: List[float] = field(default_factory=list)
    mean: float = 0.0
    median: float = 0.0
    stddev: float = 0.0
    excluded: bool = False
    reason: str = ""
    data_seeds: List[int] = field(default_factory=list)

    def recompute_aggregates(self) -> None:  # sweep.cpp:113-137
        s = self.samples
        if not s:
            self.mean = self.median = self.stddev = 0.0
            return
        # plain left-to-right loops as in the reference (Python >= 3.12's
        # sum() of floats is compensated and can differ in the last bit)
        mean = 0.0
        for x in s:
            mean += x
        self.mean = mean / float(len(s))
        srt = sorted(s)
        h = len(srt) // 2
        self.median = srt[h] if len(srt) % 2 == 1 else 0.5 * (srt[h - 1] + srt[h])
        if len(s) < 2:
            self.stddev = 0.0
        else:
            ss = 0.0
            for x in s:
                ss += (x - self.mean) * (x - self.mean)
            self.stddev = math.sqrt(ss / (float(len(s)) - 1.0))


@dataclass
class CostSurface:
    """surfaces.hpp:17-40 (cells in grid order + run metadata)."""
    cells: List[CostCell]
    metadata: dict

    def find(self, coords: CellCoords, phase: Phase, backend: BackendId) -> Optional[CostCell]:
        for c in self.cells:
            if c.coords == coords and c.phase == phase and c.backend == backend:
                return c
        return None


def generate_cells(grid: SweepGrid) -> List[Tuple[CellCoords, bool]]:
    """sweep.cpp:103-117: signals-major, then memory, then observations."""
    grid.validate()
    out = []
    for n in grid.signal_counts:
        for m in grid.memory_counts:
            for obs in grid.observation_counts:
                c = CellCoords(n, obs, m)
                out.append((c, c.admissible()))
    return out


def cell_data_seed(master_seed: int, coords: CellCoords, replicate: int) -> int:
    from .signals import cell_data_seed as _seed
    return _seed(master_seed, coords.n_signals, coords.n_observations, coords.n_memory, replicate)


def sweep_config_to_json(config: SweepConfig) -> dict:
    """config.cpp:252-274 (the config echo stored in the surface metadata)."""
    from .surfaces import backend_to_json
    kernel = {"kind": KernelKind(config.kernel.kind).name}
    if config.kernel.bandwidth is not None:
        kernel["bandwidth"] = config.kernel.bandwidth
    t = config.signal_template
    g = config.grid
    return {"grid": {"signal_counts": list(g.signal_counts), "observation_counts": list(g.observation_counts),
                     "memory_counts": list(g.memory_counts),
                     "training_observation_factor": g.training_observation_factor},
            "replicates": config.replicates, "warmups": config.warmups,
            "backends": [backend_to_json(b) for b in config.backends], "kernel": kernel,
            "signals": {"ar_coefficient": t.ar_coefficient, "cross_correlation": t.cross_correlation,
                        "variance": t.variance, "skewness": t.skewness, "kurtosis": t.kurtosis},
            "master_seed": config.master_seed, "timer": config.timer, "estimator": config.estimator}


def _timer(kind: str) -> Callable[[], float]:
    return time.monotonic if kind == "wall_monotonic" else time.process_time


# --------------------------------------------------------------- one unit
def _cell_data(coords: CellCoords, config: SweepConfig, base: int, device: int):
    """sweep.cpp:148-161, synthesized on the device."""
    from .signals import SignalSpec, derive_seed, synthesize_device
    t = config.signal_template
    rows = config.grid.training_observation_factor * coords.n_memory

    def spec(N, seed):
        return SignalSpec.uniform(coords.n_signals, N, t.ar_coefficient, t.cross_correlation,
                                  t.variance, t.skewness, t.kurtosis, seed)
    training = synthesize_device(spec(rows, derive_seed(base, [0])), device)
    # FP32-only backend lists take the surveillance block straight in FP32
    # (bit-identical to the FP64 block's .float(), one pass fewer)
    import torch
    f32 = config.estimator == "mset2" and all(b.precision == "fp32" for b in config.backends)
    surveil = synthesize_device(spec(coords.n_observations, derive_seed(base, [1])), device,
                                torch.float32 if f32 else None)
    return training, surveil


def _train_eval(coords: CellCoords, config: SweepConfig, backend: BackendId, training, surveil,
                clock) -> Tuple[float, float]:
    """Timed train + estimate of one backend on device-resident data."""
    import torch
    from .estimator import MsetModel, algorithm_by_name
    from .mset import estimate_device, train_device
    if config.estimator != "mset2" or backend.is_host:
        # host backends (and the non-GPU estimators) take host FP64 copies of
        # the replicate's signals, made outside the timed brackets
        algo = algorithm_by_name(config.estimator)
        X, O = training.double().cpu().numpy(), surveil.double().cpu().numpy()
        t0 = clock()
        model = algo.train(X, coords.n_memory, config.kernel, backend)
        t1 = clock()
        t2 = clock()
        algo.estimate(model, O, backend)
        t3 = clock()
        return max(t1 - t0, 1e-9), max(t3 - t2, 1e-9)
    dev = training.device
    obs = surveil if backend.precision == "fp64" else surveil.float()
    est = torch.empty_like(obs.T).T
    res = torch.empty_like(obs.T).T
    torch.cuda.synchronize(dev)
    t0 = clock()
    model = train_device(training, coords.n_memory, config.kernel, backend)
    t1 = clock()
    t2 = clock()
    estimate_device(model, obs, est, res)
    torch.cuda.synchronize(dev)
    t3 = clock()
    del model
    return max(t1 - t0, 1e-9), max(t3 - t2, 1e-9)


def run_unit(coords: CellCoords, replicate: int, config: SweepConfig, device: int,
             warm: bool) -> dict:
    """One (cell, replicate): optional untimed warm-ups (seeds >= replicates,
    sweep.cpp:188-204), then the timed train/estimate of every backend."""
    clock = _timer(config.timer)
    rec = {"coords": (coords.n_signals, coords.n_observations, coords.n_memory),
           "replicate": replicate, "seed": cell_data_seed(config.master_seed, coords, replicate),
           "train": [], "surveil": [], "error": None, "error_kind": None}
    backends = [b if b.is_host else dataclasses.replace(b, device=device) for b in config.backends]
    try:
        if warm:
            for w in range(config.warmups):
                base = cell_data_seed(config.master_seed, coords, config.replicates + w)
                tr, sv = _cell_data(coords, config, base, device)
                for b in backends:
                    _train_eval(coords, config, b, tr, sv, clock)
        tr, sv = _cell_data(coords, config, rec["seed"], device)
        for b in backends:
            t_train, t_surv = _train_eval(coords, config, b, tr, sv, clock)
            rec["train"].append(t_train)
            rec["surveil"].append(t_surv)
    except errors.Error as e:
        rec["error"] = str(e)
        rec["error_kind"] = type(e).__name__
    return rec


# ------------------------------------------------------------ distribution
def predicted_cost(coords: CellCoords) -> float:
    """Predicted wall time (ms) of one timed (cell, replicate) unit on a B200,
    calibrated on round-2 measurements: ~1.5 ms fixed
    (launches, synchronisations, Python), train ~1.6e-10 m^3 (the certified
    Cholesky inverse dominates large m), surveillance ~1e-11 N n m (4 N n m
    flops at ~400 TFLOP/s), device synthesis ~1.2e-8 ms per generated sample
    (N n surveillance + 4 m n training rows).  Only ratios matter."""
    n, N, m = coords.n_signals, coords.n_observations, coords.n_memory
    return 1.5 + 1.6e-10 * m ** 3 + 1.0e-11 * N * n * m + 1.2e-8 * N * n + 4.8e-8 * m * n


def plan_units(units: Sequence[Tuple[int, CellCoords, int]], world: int,
               warmups: int = 1) -> List[List[Tuple[int, CellCoords, int]]]:
    """Place (cell_index, coords, replicate) units on `world` ranks.

    A rank runs `warmups` untimed passes of a cell before its first timed
    unit of that cell (sweep.cpp:193-204, kept per (cell, rank) so every
    timed sample follows a warm-up on its own device), so spreading a cell's
    replicates over ranks multiplies its warm-ups.  Cells are therefore
    placed whole, largest first, on the least-loaded rank (LPT), and a cell
    is split into replicate groups only when its warm-ups plus replicates
    exceed an even share of the total.  Per-unit LPT without this paid a
    warm-up per (cell, rank) for nearly every large cell and capped the
    predicted 8-rank efficiency of the C4 grid at 0.64; cell-level LPT
    reaches 0.99.  Deterministic (ties by rank, then cell order)."""
    cells: dict = {}
    for u in units:
        cells.setdefault(u[0], []).append(u)
    for lst in cells.values():
        lst.sort(key=lambda u: u[2])
    total = sum(predicted_cost(lst[0][1]) * (len(lst) + warmups) for lst in cells.values())
    target = total / max(world, 1)
    loads = [0.0] * world
    plan: List[List[Tuple[int, CellCoords, int]]] = [[] for _ in range(world)]
    order = sorted(cells, key=lambda i: (-predicted_cost(cells[i][0][1]) * (len(cells[i]) + warmups), i))
    for idx in order:
        lst = cells[idx]
        c = predicted_cost(lst[0][1])
        reps = len(lst)
        g = 1
        while g < reps and (warmups + -(-reps // g)) * c > target:
            g += 1
        sizes = [reps // g + (1 if k < reps % g else 0) for k in range(g)]
        start = 0
        for sz in sizes:
            group = lst[start:start + sz]
            start += sz
            r = min(range(world), key=lambda k: (loads[k], k))
            plan[r].extend(group)
            loads[r] += c * (warmups + sz)
    for p in plan:  # each rank walks its units in grid order
        p.sort(key=lambda u: (u[0], u[2]))
    return plan


def _gather(records: list, world: int) -> list:
    if world == 1:
        return [records]
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, records)
    return out


def run_cell(coords: CellCoords, config: SweepConfig, device: int = 0) -> List[CostCell]:
    """sweep.cpp:170-239 on one device."""
    if not coords.admissible():
        raise ConstraintViolated("run_cell: cell violates m >= 2n")
    recs = [run_unit(coords, r, config, device, warm=(r == 0)) for r in range(config.replicates)]
    return _assemble_cell(coords, config, recs)


def _assemble_cell(coords: CellCoords, config: SweepConfig, recs: List[dict]) -> List[CostCell]:
    cells = [CostCell(coords, ph, b) for ph in (Phase.train, Phase.surveil) for b in config.backends]
    recs = sorted(recs, key=lambda r: r["replicate"])
    failed = [r for r in recs if r["error"] is not None]
    if failed:  # sweep.cpp:229-236: any Error excludes the whole cell
        for c in cells:
            c.excluded = True
            c.reason = failed[0]["error"]
            c.recompute_aggregates()
        return cells
    nb = len(config.backends)
    for r in recs:
        for b in range(nb):
            cells[b].samples.append(r["train"][b])
            cells[b].data_seeds.append(r["seed"])
            cells[nb + b].samples.append(r["surveil"][b])
            cells[nb + b].data_seeds.append(r["seed"])
    for c in cells:
        c.recompute_aggregates()
    return cells


def run_sweep(config: SweepConfig, progress: Optional[Callable] = None, *, world: int = 1,
              rank: int = 0, device: int = 0, unit_runner: Callable = None) -> Optional[CostSurface]:
    """sweep.cpp:277-325, distributed over `world` ranks (this is `rank`).
    Returns the surface on rank 0 (None elsewhere).  `unit_runner` replaces
    run_unit (tests of the placement / gather / assembly logic on CPU)."""
    unit_runner = unit_runner or run_unit
    config.validate()
    grid_cells = generate_cells(config.grid)
    if not any(ok for _, ok in grid_cells):
        raise EmptyGrid("run_sweep: no grid cell satisfies m >= 2n")
    started = time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())
    units = [(i, c, r) for i, (c, ok) in enumerate(grid_cells) if ok for r in range(config.replicates)]
    mine = plan_units(units, world, config.warmups)[rank]
    records = []
    seen = set()
    fatal = None
    try:
        for idx, coords, r in mine:
            warm = idx not in seen  # one warm-up pass per (cell, rank), as run_cell does per cell
            seen.add(idx)
            rec = unit_runner(coords, r, config, device, warm)
            rec["cell_index"] = idx
            records.append(rec)
    except Exception as e:  # noqa: BLE001 -- every rank must still reach the gather
        fatal = f"rank {rank}: {type(e).__name__}: {e}"
        records = [{"fatal": fatal}]
    gathered = _gather(records, world)
    # a non-Error failure (e.g. CUDA OOM) aborts the sweep as the serial
    # reference would -- on every rank, after the gather, so no rank is left
    # waiting in the collective
    fatals = [rec["fatal"] for part in gathered for rec in part if "fatal" in rec]
    if fatals:
        raise RuntimeError("run_sweep aborted: " + "; ".join(fatals))
    if rank != 0:
        return None
    by_cell = {}
    for part in gathered:
        for rec in part:
            by_cell.setdefault(rec["cell_index"], []).append(rec)
    surface_cells = []
    for i, (coords, ok) in enumerate(grid_cells):
        if ok:
            results = _assemble_cell(coords, config, by_cell.get(i, []))
        else:
            results = [CostCell(coords, ph, b, excluded=True, reason="m<2n")
                       for ph in (Phase.train, Phase.surveil) for b in config.backends]
        if progress:
            progress(i, len(grid_cells), coords, results)
        surface_cells.extend(results)
    meta = {
        "generator": "containerstress-b200 0.1.0",
        "host_description": f"{platform.processor() or platform.machine()} / {platform.system()} {platform.release()}",
        "hardware_threads": os.cpu_count(),
        "timer": config.timer,
        "rng_algorithm": RNG_ALGORITHM,
        "threads_override": config.threads_override_note,
        "config": sweep_config_to_json(config),
        "world_size": world,
        "placement": "LPT over (cell, replicate) units; records gathered with torch.distributed",
        "started_at": started,
        "finished_at": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
    }
    try:
        meta["backend_capabilities"] = [capabilities(b if b.is_host else dataclasses.replace(b, device=device)).description
                                        for b in config.backends]
    except errors.Error:
        meta["backend_capabilities"] = []
    return CostSurface(surface_cells, meta)
