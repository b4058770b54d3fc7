"""Command line for GPU sweeps (reference: proj/tools/main.cpp:118-278).

    python -m paper_2003_08011_b200 sweep --config C.json --out DIR
           [--backend b200,reference,...] [--threads K] [--seed S]
    python -m paper_2003_08011_b200 speedup --surface DIR/surface.json
           --ref LABEL --opt LABEL --out DIR

Same outputs, messages and exit codes as the reference's ``cmd_sweep`` /
``cmd_speedup``: cost_train.csv, cost_surveil.csv, surface.json (sweep),
speedup_train.csv, speedup_surveil.csv (speedup) and a manifest.json in
the output directory; exit 0 success, 2 configuration error, 4 empty grid,
5 runtime failure after partial output (main.cpp:205-231: the cells
reported so far are written with ``metadata.partial = true``; the records
of a multi-rank sweep only reach rank 0 at the final gather, so a failure
before it leaves an empty partial surface).  The
reference's ``synth`` command (signal files, moment reports) is outside
this library's scope.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from typing import List, Optional

from . import errors
from .config import load_json_file, override_worker_count, parse_sweep_config
from .mset import BackendId
from .surfaces import (cells_for_phase, export_cost_csv, export_speedup_csv, export_surface_json,
                       import_surface_json, speedup, surface_backends, UnknownBackend)
from .sweep import CostSurface, Phase, run_sweep, sweep_config_to_json

OK, CONFIG_ERROR, INFEASIBLE, EMPTY_GRID, RUNTIME_FAILURE = 0, 2, 3, 4, 5  # main.cpp:27-36


def _now() -> str:
    return time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())


def _write_text_atomic(path: str, text: str) -> None:
    """main.cpp:49-59"""
    tmp = path + ".tmp"
    try:
        with open(tmp, "w") as f:
            f.write(text)
    except OSError:
        raise errors.IoError("cannot open " + tmp) from None
    os.replace(tmp, path)


class _Manifest:
    """main.cpp:61-78"""

    def __init__(self, command: str):
        self.command, self.out_dir, self.config = command, "", {}
        self.started_at, self.artifacts = _now(), []

    def finish(self, status: int) -> None:
        if not self.out_dir:
            return
        body = {"command": self.command, "config": self.config, "out_dir": self.out_dir,
                "started_at": self.started_at, "finished_at": _now(), "exit_status": status,
                "artifacts": self.artifacts}
        _write_text_atomic(os.path.join(self.out_dir, "manifest.json"), json.dumps(body, indent=2) + "\n")


def _summary(surface: CostSurface, out) -> None:
    """main.cpp:118-140"""
    out.write("phase    backend                          cells   median_min_s   median_max_s\n")
    for phase in (Phase.train, Phase.surveil):
        for b in surface_backends(surface):
            meds = [c.median for c in surface.cells if c.phase == phase and c.backend == b and not c.excluded]
            lo, hi = (min(meds), max(meds)) if meds else (0.0, 0.0)
            out.write(f"{phase.value:<8} {b.label():<32} {len(meds):5d}   {lo:12.6g}   {hi:12.6g}\n")


def cmd_sweep(config_path: str, out_dir: str, backend_csv: str = "", threads: Optional[int] = None,
              seed: Optional[int] = None, *, world: int = 1, rank: int = 0, device: int = 0) -> int:
    """main.cpp:142-232 (the sweep itself may span `world` ranks, sweep.run_sweep)."""
    manifest = _Manifest("sweep")
    try:
        config = parse_sweep_config(load_json_file(config_path))
        if backend_csv:
            config.backends = [BackendId.parse(t) for t in backend_csv.split(",")]
        if threads is not None:
            override_worker_count(config, threads, f"cli:--threads={threads}")
        if seed is not None:
            config.master_seed = seed
        config.validate()
        if rank == 0:
            os.makedirs(out_dir, exist_ok=True)
            manifest.out_dir = out_dir
            manifest.config = sweep_config_to_json(config)
    except errors.Error as e:
        sys.stderr.write(f"error: {e}\n")
        return CONFIG_ERROR

    partial: List = []

    def progress(index, total, coords, results):  # main.cpp:164-180
        line = f"[cell {index + 1}/{total}] n={coords.n_signals} obs={coords.n_observations} m={coords.n_memory}"
        if results and results[0].excluded:
            line += f" excluded ({results[0].reason})"
        else:
            for c in results:
                if c.phase == Phase.train:
                    line += f" {c.backend.label()}={c.median:g}s"
        sys.stderr.write(line + "\n")
        partial.extend(results)

    def write_outputs(surface: CostSurface) -> None:  # main.cpp:182-195
        export_cost_csv(cells_for_phase(surface, Phase.train), os.path.join(out_dir, "cost_train.csv"))
        export_cost_csv(cells_for_phase(surface, Phase.surveil), os.path.join(out_dir, "cost_surveil.csv"))
        export_surface_json(surface, os.path.join(out_dir, "surface.json"))
        manifest.artifacts += ["cost_train.csv", "cost_surveil.csv", "surface.json", "manifest.json"]

    try:
        surface = run_sweep(config, progress, world=world, rank=rank, device=device)
        if rank != 0:
            return OK
        write_outputs(surface)
        manifest.finish(OK)
        _summary(surface, sys.stdout)
        return OK
    except errors.EmptyGrid as e:
        sys.stderr.write(f"error: {e}\n")
        manifest.finish(EMPTY_GRID)
        return EMPTY_GRID
    except Exception as e:  # noqa: BLE001 -- main.cpp:205-231: keep what completed
        sys.stderr.write(f"error: sweep aborted: {e}\n")
        if rank != 0:
            return RUNTIME_FAILURE
        meta = {"generator": "containerstress-b200 0.1.0", "timer": config.timer,
                "threads_override": config.threads_override_note, "config": sweep_config_to_json(config),
                "partial": True, "started_at": manifest.started_at, "finished_at": _now()}
        try:
            write_outputs(CostSurface(partial, meta))
        except Exception as inner:  # noqa: BLE001
            sys.stderr.write(f"error: could not write partial output: {inner}\n")
        manifest.finish(RUNTIME_FAILURE)
        return RUNTIME_FAILURE


def resolve_backend(surface: CostSurface, token: str) -> BackendId:
    """surfaces.cpp:81-98: a full label, or a bare kind present exactly once."""
    present = surface_backends(surface)
    for b in present:
        if b.label() == token:
            return b
    if token in ("reference", "optimized", "b200"):
        matches = [b for b in present if b.kind == token]
        if len(matches) == 1:
            return matches[0]
        if len(matches) > 1:
            raise UnknownBackend(f'backend "{token}" is ambiguous in this surface; use a full label')
    raise UnknownBackend(f'backend "{token}" not present in this surface')


def cmd_speedup(surface_path: str, ref_token: str, opt_token: str, out_dir: str) -> int:
    """main.cpp:234-275"""
    manifest = _Manifest("speedup")
    try:
        surface = import_surface_json(surface_path)
        ref = resolve_backend(surface, ref_token)
        opt = resolve_backend(surface, opt_token)
        result = speedup(surface, ref, opt)
        os.makedirs(out_dir, exist_ok=True)
        manifest.out_dir = out_dir
        manifest.config = {"surface": surface_path, "ref": ref.label(), "opt": opt.label()}
        export_speedup_csv(result, Phase.train, os.path.join(out_dir, "speedup_train.csv"))
        export_speedup_csv(result, Phase.surveil, os.path.join(out_dir, "speedup_surveil.csv"))
        manifest.artifacts += ["speedup_train.csv", "speedup_surveil.csv", "manifest.json"]
        manifest.finish(OK)
        holes = sum(1 for c in result.cells if c.hole)
        sys.stdout.write(f"speedup: {len(result.cells) - holes} cells, {holes} holes "
                         f"({ref.label()} vs {opt.label()})\n")
        return OK
    except errors.Error as e:
        sys.stderr.write(f"error: {e}\n")
        manifest.finish(CONFIG_ERROR)
        return CONFIG_ERROR


def main(argv: Optional[List[str]] = None) -> int:
    """main.cpp:279-323 (argument errors exit 2, like CLI11's parse errors there)."""
    ap = argparse.ArgumentParser(prog="python -m paper_2003_08011_b200",
                                 description="Compute-cost scoping benchmarks on B200")
    ap.add_argument("--version", action="version", version="containerstress-b200 0.1.0")
    sub = ap.add_subparsers(dest="command", required=True)
    sw = sub.add_parser("sweep", help="Run a cost sweep")
    sw.add_argument("--config", required=True, help="SweepConfig JSON path")
    sw.add_argument("--out", required=True, help="Output directory")
    sw.add_argument("--backend", default="", help="Comma-separated backend ids overriding the config")
    sw.add_argument("--threads", type=int, help="Worker count override for optimized backends")
    sw.add_argument("--seed", type=int, help="Override the master seed")
    sp = sub.add_parser("speedup", help="Cost ratios between backends")
    sp.add_argument("--surface", required=True, help="surface.json path")
    sp.add_argument("--ref", required=True, help="Reference backend id")
    sp.add_argument("--opt", required=True, help="Optimized backend id")
    sp.add_argument("--out", required=True, help="Output directory")
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return OK if e.code == 0 else CONFIG_ERROR
    if a.command == "sweep":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        device = int(os.environ.get("LOCAL_RANK", "0"))
        if world > 1:  # one process per GPU (torchrun), records gathered at the end
            import torch.distributed as dist
            if not dist.is_initialized():
                # CSB_DIST_BACKEND=gloo: several ranks without GPUs (tests)
                dist.init_process_group(os.environ.get("CSB_DIST_BACKEND", "nccl"))
        return cmd_sweep(a.config, a.out, a.backend, a.threads, a.seed, world=world, rank=rank, device=device)
    return cmd_speedup(a.surface, a.ref, a.opt, a.out)


if __name__ == "__main__":
    sys.exit(main())
