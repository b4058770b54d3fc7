#!/usr/bin/env python
"""Benchmark of the B200 MSET2 hot path (BASELINE.json configs[1] = C2).

Workload (per GPU): n = 100 signals, N = 100,000 surveillance observations,
m = 1,000 memory vectors, 4,000 training rows; FP64 train + FP32 (tcgen05
3xFP16) surveillance; inverse-distance kernel, h = sqrt(n); synthetic data
from the reference's synthesis recipe (demo template: phi 0.5, rho 0.3,
var 1, skew 0.5, kurt 4, master seed 20260810).

A step is one surveillance pass over the N observations (estimate +
residual), inputs resident in HBM (FP32 column-major), L2 flushed between
steps (256 MiB write, outside the per-step events).  `value` is
observations/s over all ranks; `e2e` is the same metric through the C-ABI
host-buffer call (pinned FP64 host observations in, FP64 estimates and
residuals out, H2D/D2H inside the timed region).  Train time is reported
alongside (`train`).  Multi-GPU: one process per GPU, independent
observation shards (weak scaling), no data-path collective; barrier +
max-over-ranks timing through torch.distributed.

`--impl reference` times the reference's CPU implementation of the same
path (the oracle restatement, optimized backend, all host threads) on a
bounded observation sample per step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_SIG, N_OBS, N_MEM, TRAIN_FACTOR = 100, 100_000, 1_000, 4
TEMPLATE = dict(phi=0.5, rho=0.3, var=1.0, skew=0.5, kurt=4.0)
MASTER_SEED = 20260810
METRIC = "MSET2 observations estimated/sec"
UNIT = "obs/s"
WORKLOAD = "C2: MSET2 100 signals, 100k observations, 1,000 memory vectors (FP64 train + FP32 surveillance)"
L2_FLUSH_BYTES = 256 << 20
CPU_SAMPLE_OBS = 8192


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_info():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return model, os.cpu_count() or 1


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def load_traffic():
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        d = json.load(open(path))
        return d.get("mset_estimate_tc_kernel_C2")
    except (OSError, ValueError):
        return None


def load_f16_peak():
    """Dense kind::f16 tcgen05 throughput measured on this pool by
    tools/mma_probe (profiles/mma_probe.json), TFLOP/s at max clock."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "mma_probe.json")))
        return max(r["tflops_at_base_clock"] for r in d["results"] if r["kind"] == "f16")
    except (OSError, ValueError, KeyError):
        return None


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "fallback": True}


def make_data(rank):
    import paper_2003_08011_b200 as p
    base = p.cell_data_seed(MASTER_SEED, N_SIG, N_OBS, N_MEM, rank)
    t = TEMPLATE
    train = p.synthesize(p.SignalSpec.uniform(N_SIG, TRAIN_FACTOR * N_MEM, t["phi"], t["rho"],
                                              t["var"], t["skew"], t["kurt"],
                                              p.derive_seed(base, [0]))).data
    obs = p.synthesize(p.SignalSpec.uniform(N_SIG, N_OBS, t["phi"], t["rho"], t["var"],
                                            t["skew"], t["kurt"], p.derive_seed(base, [1]))).data
    return train, obs


# ----------------------------------------------------------------- reference
def run_reference(args, world, rank):
    """The reference CPU path (oracle restatement, optimized backend with all
    host threads) on a bounded sample of the same workload per step."""
    if rank != 0:
        return
    from oracle import oracle as o
    o.build()
    import numpy as np
    train, obs = make_data(0)
    _, cores = cpu_info()
    model = o.train(train, N_MEM, o.INVERSE_DISTANCE, 0.0, o.OPTIMIZED, 64, cores)
    sample = obs[:CPU_SAMPLE_OBS]
    for _ in range(args.warmup):
        o.estimate(model, sample[:1024], o.OPTIMIZED, 64, cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        o.estimate(model, sample, o.OPTIMIZED, 64, cores)
        times.append(time.perf_counter() - t0)
    step = statistics.mean(times)
    v = CPU_SAMPLE_OBS / step
    model_name, _ = cpu_info()
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference synthesis recipe, demo template)",
        "config": {"workload": WORKLOAD, "n_signals": N_SIG, "n_observations": N_OBS,
                   "n_memory": N_MEM, "sample_observations_per_step": CPU_SAMPLE_OBS},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{CPU_SAMPLE_OBS} of {N_OBS} observations per step, "
                                   f"oracle optimized backend (tile 64, {cores} threads), {model_name}"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_sample(train, obs):
    from oracle import oracle as o
    o.build()
    model_name, cores = cpu_info()
    model = o.train(train, N_MEM, o.INVERSE_DISTANCE, 0.0, o.OPTIMIZED, 64, cores)
    sample = obs[:CPU_SAMPLE_OBS]
    t0 = time.perf_counter()
    o.estimate(model, sample, o.OPTIMIZED, 64, cores)
    t = time.perf_counter() - t0
    t1 = time.perf_counter()
    o.train(train, N_MEM, o.INVERSE_DISTANCE, 0.0, o.OPTIMIZED, 64, cores)
    train_s = time.perf_counter() - t1
    return {"value": CPU_SAMPLE_OBS / t, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{CPU_SAMPLE_OBS} of {N_OBS} observations, oracle optimized backend "
                      f"(tile 64, {cores} threads) on {model_name}",
            "train_ms": train_s * 1e3}


# BASELINE configs[3] / SURVEY 8(d) C4: 7 x 3 x 6 = 126 cells, 96 admissible,
# 5 replicates -> 480 (cell, replicate) units (~11 s on one B200)
SWEEP_GRID = dict(signal_counts=[10, 20, 50, 100, 200, 500, 1000],
                  observation_counts=[10_000, 100_000, 1_000_000],
                  memory_counts=[100, 200, 500, 1000, 2000, 4000])
SWEEP_REPLICATES = 5


def run_bench_sweep(world, rank, local, barrier, max_over_ranks):
    """The reference's Monte Carlo scoping sweep (run_sweep, sweep.cpp:277-325)
    on the C4 grid: (cell, replicate) units LPT-placed over the ranks,
    cost records gathered over torch.distributed.  Reports units/s over the
    whole sweep wall time (device synthesis + timed train/estimate + gather),
    max over ranks."""
    from paper_2003_08011_b200 import BackendId
    from paper_2003_08011_b200.sweep import SweepConfig, SweepGrid, SignalStatsTemplate, run_sweep
    cfg = SweepConfig(SweepGrid(**SWEEP_GRID), replicates=SWEEP_REPLICATES, warmups=1,
                      backends=[BackendId("b200", local, "fp32")], master_seed=MASTER_SEED,
                      signal_template=SignalStatsTemplate(0.5, 0.3, 1.0, 0.5, 4.0))
    barrier()
    t0 = time.perf_counter()
    surface = run_sweep(cfg, world=world, rank=rank, device=local)
    barrier()
    wall = max_over_ranks(time.perf_counter() - t0)
    if rank != 0:
        return None
    units = sum(len(c.samples) for c in surface.cells if c.phase.value == "train")
    cells = sum(1 for c in surface.cells if c.phase.value == "train" and not c.excluded)
    excluded = sum(1 for c in surface.cells if c.phase.value == "train" and c.excluded)
    train_s = sum(sum(c.samples) for c in surface.cells if c.phase.value == "train")
    surv_s = sum(sum(c.samples) for c in surface.cells if c.phase.value == "surveil")
    return {"metric": "MC sweep (cell, replicate) units/s", "value": units / wall, "unit": "units/s",
            "cells_per_s": cells / wall, "units": units, "admissible_cells": cells,
            "excluded_cells": excluded, "wall_s": wall, "timed_train_s": train_s,
            "timed_surveil_s": surv_s, "scaling": "strong", "n_gpus": world,
            "grid": {**SWEEP_GRID, "replicates": SWEEP_REPLICATES, "warmups": 1},
            "note": "full C4 grid (SURVEY 8d); device-side synthesis; wall includes synthesis, "
                    "untimed warm-ups and the gather"}


# ---------------------------------------------------------------------- B200
def run_large(local, n, N, m, workload, passes=5):
    """A large-n configuration on one GPU: train time through the device API
    and device-resident FP32 surveillance on the two-GEMM tcgen05 path.  Data
    from the device synthesiser (same recipe; host synthesis of 1e9+ samples
    is impractical)."""
    import torch
    import paper_2003_08011_b200 as p
    dev = torch.device("cuda", local)
    t = TEMPLATE
    base = p.cell_data_seed(MASTER_SEED, n, N, m, 0)
    spec = lambda rows, seed: p.SignalSpec.uniform(n, rows, t["phi"], t["rho"], t["var"], t["skew"],  # noqa: E731
                                                   t["kurt"], seed)
    X = p.synthesize_device(spec(TRAIN_FACTOR * m, p.derive_seed(base, [0])), local)
    backend = p.BackendId("b200", local, "fp32")
    model = p.train_device(X, m, p.KernelConfig(), backend)  # warm (pool, cuSOLVER modules for this size)
    tt = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fresh = p.train_device(X, m, p.KernelConfig(), backend)
        tt.append(time.perf_counter() - t0)
        model = fresh  # the previous model is freed outside the timed region
    del X
    obs64 = p.synthesize_device(spec(N, p.derive_seed(base, [1])), local)
    obs = obs64.T.float().T          # N x n column-major FP32
    del obs64
    torch.cuda.empty_cache()
    est = torch.empty_like(obs.T).T
    res = torch.empty_like(obs.T).T
    st = torch.cuda.current_stream(dev)
    p.estimate_device(model, obs, est, res, st)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(passes)]
    for a, b in ev:
        a.record(st)
        p.estimate_device(model, obs, est, res, st)
        b.record(st)
    torch.cuda.synchronize()
    ok = bool(torch.isfinite(est).all()) and bool(torch.allclose(res, obs - est))
    ms = statistics.median(a.elapsed_time(b) for a, b in ev)
    flops = 4.0 * n * m * N
    f16 = load_f16_peak() or 2380.0
    del obs, est, res, model
    torch.cuda.empty_cache()
    return {"workload": workload, "n_signals": n, "n_observations": N, "n_memory": m,
            "obs_per_s": N / (ms * 1e-3), "ms_per_pass": ms, "passes": passes,
            "algorithmic_tflops": flops / (ms * 1e-3) / 1e12,
            "frac_3xf16": flops / (ms * 1e-3) / 1e12 / (f16 / 3),
            "frac_3xf16_of_measured_bf16": flops / (ms * 1e-3) / 1e12 / (load_peaks().get("bf16_tflops", 1686.0) / 3),
            "kernels": "pack_obs + obs_sqnorm + gemm3x_f16_kernel<256,EpiSim> + gemm3x_f16_kernel<256,EpiOut> "
                       "per observation block",
            "train_ms": statistics.median(tt) * 1e3, "train_ms_min": min(tt) * 1e3,
            "train_api": "cs_mset_train_device (device FP64 training rows, synchronous)",
            "outputs_checked": ok}


def run_c3(args, local):
    """BASELINE configs[2] (C3: n=1000, N=1M, m=4000, 16k training rows)."""
    return run_large(local, 1000, 1_000_000, 4000,
                     "C3: n=1000, N=1,000,000, m=4,000 (16k training rows), FP32 device-resident I/O")


def run_c5(args, local):
    """BASELINE configs[4] made admissible (m >= 2n, so n=4,000
    with m=8,000) and sharded 8 ways: one GPU's shard of 10M / 8 = 1.25M
    observations (the 8-GPU job is 8 independent shards, no collective)."""
    return run_large(local, 4000, 1_250_000, 8000,
                     "C5': n=4000, m=8000 (32k training rows), 1.25M observations = one of 8 shards "
                     "of 10M, FP32 device-resident I/O", passes=3)


def run_b200(args, world, rank, local):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2003_08011_b200 as p

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    backend = p.BackendId("b200", local, "fp32")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    train, obs = make_data(rank)

    # ---- train (FP64), host API, synchronous: report median of 3
    train_times = []
    model = p.train(train, N_MEM, p.KernelConfig(), backend)  # warm (pool, cuSOLVER modules)
    for _ in range(5):
        t0 = time.perf_counter()
        fresh = p.train(train, N_MEM, p.KernelConfig(), backend)
        train_times.append(time.perf_counter() - t0)
        model = fresh  # the previous model is freed outside the timed region
    train_ms = statistics.median(train_times) * 1e3
    # same call with the eigen_spectrum computed inside train (eigenvalues-only
    # syevd; the default path defers it to the first export)
    os.environ["CSB_EAGER_SPECTRUM"] = "1"
    eager = []
    for _ in range(3):
        t0 = time.perf_counter()
        fresh = p.train(train, N_MEM, p.KernelConfig(), backend)
        eager.append(time.perf_counter() - t0)
        del fresh
    del os.environ["CSB_EAGER_SPECTRUM"]
    train_eager_ms = statistics.median(eager) * 1e3

    # ---- device-resident surveillance
    d_obs = torch.tensor(obs.T.astype(np.float32), device=dev).T          # N x n col-major
    d_est = torch.empty_like(d_obs.T).T
    d_res = torch.empty_like(d_obs.T).T
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(max(args.warmup, 3)):
        p.estimate_device(model, d_obs, d_est, d_res, stream)
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    barrier()
    w0 = time.perf_counter()
    for i in range(args.steps):
        flush.zero_()                      # L2 flush, outside the step events
        starts[i].record(stream)
        p.estimate_device(model, d_obs, d_est, d_res, stream)
        ends[i].record(stream)
    barrier()
    wall = time.perf_counter() - w0
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    mean_ms = statistics.mean(step_ms)
    mean_ms_max = max_over_ranks(mean_ms)

    # ---- end to end through the C-ABI host-buffer call (pinned FP64)
    h_obs = torch.from_numpy(np.asfortranarray(obs).T.copy()).pin_memory()  # n x N rows = signals
    h_est = torch.empty_like(h_obs).pin_memory()
    h_res = torch.empty_like(h_obs).pin_memory()
    obs_np = h_obs.numpy().T          # N x n, column-major view of pinned memory
    est_np = h_est.numpy().T
    res_np = h_res.numpy().T
    from paper_2003_08011_b200 import _lib
    import ctypes as C

    def e2e_call():
        _lib.check(_lib.lib().cs_mset_estimate(
            p.context(local).handle, model.handle, obs_np.ctypes.data_as(_lib.pd), N_OBS, N_SIG,
            est_np.ctypes.data_as(_lib.pd), res_np.ctypes.data_as(_lib.pd)))

    for _ in range(2):
        e2e_call()
    e2e_steps = max(3, min(args.steps, 20))
    barrier()
    e2e_t = []
    for _ in range(e2e_steps):
        t0 = time.perf_counter()
        e2e_call()
        e2e_t.append(time.perf_counter() - t0)
    barrier()
    clocks = sampler.stop()
    e2e_mean = max_over_ranks(statistics.mean(e2e_t))
    # correctness guard on the e2e output: residual identity
    assert np.array_equal(res_np, obs_np - est_np)

    # ---- Monte Carlo scoping sweep (cells/s), strong scaling over ranks
    sweep = None if args.no_sweep else run_bench_sweep(world, rank, local, barrier, max_over_ranks)

    if rank != 0:
        return
    peaks = load_peaks()
    flops_per_obs = 4.0 * N_SIG * N_MEM                       # F = 4nm
    achieved_tflops = flops_per_obs * N_OBS / (mean_ms * 1e-3) / 1e12
    bf16 = peaks.get("bf16_tflops", 1590.0)
    # tensor work actually issued: 3 FP16 products per GEMM incl. padding
    K1, N2 = (N_SIG + 2 + 15) // 16 * 16, (N_SIG + 15) // 16 * 16  # + ||d||^2, ||x||^2 columns
    MT = 64  # tile the library selects for n = 100 (choose_tc_shape: MT 64, 2 ACC + 2 S buffers)
    f16_peak = load_f16_peak() or 2380.0
    m_pad = (N_MEM + MT - 1) // MT * MT
    n_tiles = (N_OBS + 127) // 128
    issued = 3 * 2 * 128 * n_tiles * m_pad * (K1 + N2)
    issued_tflops = issued / (mean_ms * 1e-3) / 1e12
    traffic = load_traffic()
    value = world * N_OBS / (mean_ms_max * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean_ms_max,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference synthesis recipe, demo template phi .5 rho .3 skew .5 kurt 4)",
        "config": {"workload": WORKLOAD, "n_signals": N_SIG, "n_observations_per_gpu": N_OBS,
                   "n_memory": N_MEM, "training_rows": TRAIN_FACTOR * N_MEM,
                   "kernel": "inverse_distance", "bandwidth": "sqrt(n)",
                   "surveillance": "fused tcgen05 3xFP16 (FP32-accurate, exact power-of-two operand scales)", "train": "FP64",
                   "l2": "flushed between steps (256 MiB write outside step events)",
                   "parallelism": f"dp{world} (independent observation shards)"},
        "wall_s_timed_region": wall,
        "gpu_launches": args.steps,
        "train": {"ms": train_ms, "api": "cs_mset_train (host FP64 in, synchronous)",
                  "includes": "H2D + selection + scale + Gram + certified-Cholesky pseudo-inverse (rank == m "
                              "proven by the 1-norm condition bound; eigen route otherwise) + P=Dn G+ + "
                              "operand packing; eigen_spectrum deferred to first export",
                  "ms_with_eigen_spectrum": train_eager_ms},
        "e2e": {"value": world * N_OBS / e2e_mean, "unit": UNIT,
                "h2d_bytes_per_step": N_OBS * N_SIG * 8,
                "d2h_bytes_per_step": 2 * N_OBS * N_SIG * 8,
                "api": "cs_mset_estimate (pinned host FP64 in, estimates + residuals out)"},
        "roofline": {"bound": "tensor", "achieved": achieved_tflops, "peak": bf16, "unit": "TFLOP/s",
                     "frac": achieved_tflops / bf16, "traffic": traffic,
                     "kernel": "mset_estimate_tc_kernel<64,2,2,float,true>",
                     "algorithmic_flops_per_launch": flops_per_obs * N_OBS,
                     "peak_note": "peak = measured dense bf16 (MEASURED_PEAKS.json); the kernel runs "
                                  "tcgen05 kind::f16 (same dense rate) and issues 3 split products per "
                                  "GEMM (3xFP16, FP32-accurate), so its algorithmic ceiling is peak/3; "
                                  "peak_f16_probe = tools/mma_probe at 1965 MHz",
                     "frac_3xf16": achieved_tflops / (bf16 / 3),
                     "peak_f16_probe": f16_peak,
                     "frac_3xf16_of_probe": achieved_tflops / (f16_peak / 3),
                     "issued_f16_tflops": issued_tflops,
                     "tensor_pipe_frac_issued": issued_tflops / f16_peak},
        "clocks": clocks,
    }
    if sweep is not None:
        line["sweep"] = sweep
    if world == 1 and not args.no_c3:
        line["c3"] = run_c3(args, local)
    if world == 1 and not args.no_c5:
        line["c5"] = run_c5(args, local)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_sample(train, obs)
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-c3", action="store_true")
    ap.add_argument("--no-c5", action="store_true")
    args = ap.parse_args()
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    run_b200(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
