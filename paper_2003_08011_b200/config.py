"""Strict JSON sweep configuration (reference: proj/src/config.cpp:1-286).

Same contract as the reference parser: unknown keys are rejected with
``<context>: unknown key "<k>"`` (config.cpp:12-19), wrong types raise
``ConfigError`` naming the key (config.cpp:21-29), absent keys take the
reference defaults (replicates 5, warmups 1, training factor 4, timer
wall_monotonic, estimator mset2, config.cpp:198-246), and
``CONTAINERSTRESS_THREADS`` overrides the worker count of host backends
(config.cpp:236-244).  The one extension is the backend kind ``b200``
(SURVEY 8b): ``"b200"`` or ``{"kind": "b200", "device": D, "precision":
"fp64" | "fp32"}``; the reference's schema enums gain that kind
(INTEGRATION.md section 5).
"""
from __future__ import annotations

import dataclasses
import json
import os
from typing import Any, List, Set

from .errors import ConfigError, IoError
from .mset import BackendId, KernelConfig, KernelKind
from .sweep import SignalStatsTemplate, SweepConfig, SweepGrid

__all__ = ["load_json_file", "parse_sweep_config", "kernel_from_json", "backend_from_json",
           "override_worker_count"]


def _require_keys(j: Any, allowed: Set[str], context: str) -> None:
    """config.cpp:12-19"""
    if not isinstance(j, dict):
        raise ConfigError(f"{context}: expected a JSON object")
    for key in j:
        if key not in allowed:
            raise ConfigError(f'{context}: unknown key "{key}"')


def _is_int(v: Any) -> bool:
    return isinstance(v, int) and not isinstance(v, bool)


def _is_num(v: Any) -> bool:
    return (isinstance(v, (int, float))) and not isinstance(v, bool)


def _get(j: dict, key: str, kind: str, context: str, fallback: Any = dataclasses.MISSING) -> Any:
    """config.cpp:21-35: typed access with the reference's error shape."""
    if key not in j:
        if fallback is dataclasses.MISSING:
            raise ConfigError(f'{context}: bad value for "{key}": key not found')
        return fallback
    v = j[key]
    ok = {"int": _is_int, "uint": lambda x: _is_int(x) and x >= 0, "num": _is_num,
          "str": lambda x: isinstance(x, str),
          "int_list": lambda x: isinstance(x, list) and all(_is_int(e) for e in x)}[kind](v)
    if not ok:
        raise ConfigError(f'{context}: bad value for "{key}": expected {kind.replace("_", " ")}, got {v!r}')
    return float(v) if kind == "num" else v


def load_json_file(path: str) -> Any:
    """config.cpp:57-65"""
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise IoError("cannot open " + path) from None
    try:
        return json.loads(text)
    except json.JSONDecodeError as e:
        raise ConfigError(f"{path}: {e}") from None


def kernel_from_json(j: Any) -> KernelConfig:
    """config.cpp:126-143"""
    _require_keys(j, {"kind", "bandwidth"}, "kernel")
    kind = _get(j, "kind", "str", "kernel", "inverse_distance")
    if kind not in ("inverse_distance", "gaussian"):
        raise ConfigError(f'kernel: unknown kind "{kind}"')
    bw = j.get("bandwidth")
    cfg = KernelConfig(KernelKind[kind], None if bw is None else _get(j, "bandwidth", "num", "kernel"))
    cfg.validate()
    return cfg


def backend_from_json(j: Any) -> BackendId:
    """config.cpp:159-170, plus the b200 kind."""
    if isinstance(j, str):
        return BackendId.parse(j)
    _require_keys(j, {"kind", "tile_size", "worker_count", "device", "precision"}, "backend")
    kind = _get(j, "kind", "str", "backend")
    if kind == "reference":
        _require_keys(j, {"kind"}, "backend")
        return BackendId.reference()
    if kind == "optimized":
        _require_keys(j, {"kind", "tile_size", "worker_count"}, "backend")
        return BackendId.optimized(_get(j, "worker_count", "int", "backend", 0), _get(j, "tile_size", "int", "backend", 64))
    if kind == "b200":
        _require_keys(j, {"kind", "device", "precision"}, "backend")
        b = BackendId("b200", _get(j, "device", "int", "backend", 0), _get(j, "precision", "str", "backend", "fp64"))
        b.validate()
        return b
    raise ConfigError(f'backend: unknown kind "{kind}"')


def override_worker_count(config: SweepConfig, workers: int, note: str) -> None:
    """config.hpp override_worker_count: every optimized backend gets the
    worker count; the note is echoed into the surface metadata."""
    if workers < 1:
        raise ConfigError("worker count override must be >= 1")
    config.backends = [dataclasses.replace(b, worker_count=workers) if b.kind == "optimized" else b
                       for b in config.backends]
    config.threads_override_note = note


def parse_sweep_config(j: Any) -> SweepConfig:
    """config.cpp:179-250"""
    _require_keys(j, {"grid", "replicates", "warmups", "backends", "kernel", "signals", "master_seed",
                      "timer", "estimator"}, "sweep config")
    if "grid" not in j:
        raise ConfigError('sweep config: missing "grid"')
    g = j["grid"]
    _require_keys(g, {"signal_counts", "observation_counts", "memory_counts", "training_observation_factor"},
                  "grid")
    grid = SweepGrid(_get(g, "signal_counts", "int_list", "grid"), _get(g, "observation_counts", "int_list", "grid"),
                     _get(g, "memory_counts", "int_list", "grid"),
                     _get(g, "training_observation_factor", "int", "grid", 4))
    backends: List[BackendId]
    if "backends" in j:
        if not isinstance(j["backends"], list):
            raise ConfigError('sweep config: "backends" must be an array')
        backends = [backend_from_json(b) for b in j["backends"]]
    else:
        # the reference defaults to its two host kinds (config.cpp:218-220);
        # this library runs the GPU kind by default
        backends = [BackendId("b200", 0, "fp32")]
    template = SignalStatsTemplate()
    if "signals" in j:
        s = j["signals"]
        _require_keys(s, {"ar_coefficient", "cross_correlation", "variance", "skewness", "kurtosis"}, "signals")
        template = SignalStatsTemplate(_get(s, "ar_coefficient", "num", "signals", 0.0),
                                       _get(s, "cross_correlation", "num", "signals", 0.0),
                                       _get(s, "variance", "num", "signals", 1.0),
                                       _get(s, "skewness", "num", "signals", 0.0),
                                       _get(s, "kurtosis", "num", "signals", 3.0))
    timer = _get(j, "timer", "str", "sweep config", "wall_monotonic")
    if timer not in ("wall_monotonic", "process_cpu"):
        raise ConfigError("unknown timer: " + timer)
    config = SweepConfig(grid=grid, replicates=_get(j, "replicates", "int", "sweep config", 5),
                         warmups=_get(j, "warmups", "int", "sweep config", 1), backends=backends,
                         kernel=kernel_from_json(j["kernel"]) if "kernel" in j else KernelConfig(),
                         signal_template=template,
                         master_seed=_get(j, "master_seed", "uint", "sweep config", 0), timer=timer,
                         estimator=_get(j, "estimator", "str", "sweep config", "mset2"))
    env = os.environ.get("CONTAINERSTRESS_THREADS")
    if env is not None:
        try:
            workers = int(env)
        except ValueError:
            workers = 0
        if workers < 1 or env.strip() != env:
            raise ConfigError(f'CONTAINERSTRESS_THREADS must be a positive integer, got "{env}"')
        override_worker_count(config, workers, f"env:CONTAINERSTRESS_THREADS={env}")
    config.validate()
    return config

