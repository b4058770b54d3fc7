#!/usr/bin/env python
"""Benchmark of the B200 MSET2 hot path (BASELINE.json configs[1] = C2).

Workload (per GPU): n = 100 signals, N = 100,000 surveillance observations,
m = 1,000 memory vectors, 4,000 training rows; FP64 train + FP32 (tcgen05
3xFP16) surveillance; inverse-distance kernel, h = sqrt(n); synthetic data
from the reference's synthesis recipe (demo template: phi 0.5, rho 0.3,
var 1, skew 0.5, kurt 4, master seed 20260810, cell_data_seed per rank).

A step is one surveillance pass over the N observations (estimate +
residual).  `value` = observations/s with inputs resident in HBM (FP32
column-major), L2 flushed between steps, CUDA events on the launching
stream, max over ranks.  `e2e` = the same metric through the reference-facing
C-ABI call `cs_mset_estimate` (pinned FP64 host observations in, FP64
estimates + residuals out; H2D and D2H inside the timed region).  Beside the
headline: `train` (FP64 train incl. the eigen spectrum, the reference's
train contract), `c1` (BASELINE configs[0]), `c3` (configs[2], incl. e2e),
`c5` (configs[4] made admissible: rank 0 trains once, NCCL broadcast of
the packed model, 10M observations sharded over the ranks), `sweep` (configs[3]), `sprt`,
`roofline`, `cpu_baseline` (the CPU oracle on this box's host cores).
Multi-GPU: one process per GPU, independent observation shards (weak
scaling), no data-path collective; barrier + max-over-ranks timing.

`--impl reference` times the reference's CPU implementation of the same
path -- the oracle restatement (oracle/, the reference itself cannot be
built: Eigen3 and vendor/ are absent), optimized
backend on all host threads -- over the full C2 workload per step, with
data synthesized by the oracle's own generator; the B200 library is never
loaded in that arm.
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
DATA = "synthetic (reference synthesis recipe, demo template phi .5 rho .3 skew .5 kurt 4)"


def config_dict(world):
    """The workload description -- identical in both arms."""
    return {"workload": WORKLOAD, "n_signals": N_SIG, "n_observations_per_gpu": N_OBS,
            "n_memory": N_MEM, "training_rows": TRAIN_FACTOR * N_MEM,
            "kernel": "inverse_distance", "bandwidth": "sqrt(n)", "train": "FP64",
            "surveillance": "FP32 (tolerance 1e-3 vs the FP64 reference)",
            "l2": "flushed between steps (256 MiB write outside step events)",
            "parallelism": f"dp{world} (independent observation shards)"}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # development only: several ranks on one GPU (CSB_BENCH_DEVICE=0 with
    # CSB_BENCH_DIST_BACKEND=gloo) to exercise the multi-rank plumbing
    if os.environ.get("CSB_BENCH_DEVICE"):
        local = int(os.environ["CSB_BENCH_DEVICE"])
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
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        cores = os.cpu_count() or 1
    return model, cores


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


def _json_file(*parts):
    try:
        return json.load(open(os.path.join(ROOT, *parts)))
    except (OSError, ValueError):
        return None


def load_traffic(key):
    d = _json_file("profiles", "traffic.json") or {}
    return d.get(key)


def load_peaks():
    d = _json_file("MEASURED_PEAKS.json")
    if d:
        return d
    # /opt/skills/guides/B200_PROFILING.md fallback
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "fallback": True}


SUSTAINED_NOTE = ("P_eff = measured dense bf16 SUSTAINED (MEASURED_PEAKS.json bf16_tflops_sustained; the "
                  "passes run back to back for seconds, where the clock settles at ~1.35 GHz) / 3: 3xFP16 "
                  "split products; frac_vs_burst_peak uses the burst figure")


def sustained_p_eff():
    """(sustained, burst) 3xFP16 ceilings: long back-to-back passes (C3, C5')
    are judged against the sustained measured bf16 rate, single short
    launches (the C2 step) against the burst rate (B200_PROFILING.md)."""
    peaks = load_peaks()
    burst = peaks.get("bf16_tflops", 1590.0)
    return peaks.get("bf16_tflops_sustained", burst) / 3, burst / 3


def load_probe_peaks():
    """FP64 (DMMA, DFMA) and MUFU throughputs measured on this pool by
    tools/peaks_probe.cu (profiles/peaks_probe.json)."""
    return _json_file("profiles", "peaks_probe.json") or {}


# ----------------------------------------------------------------- reference
def _oracle_data(o, n, N, m, rank):
    """The same bytes the B200 arm trains and surveils on, from the oracle's
    own generator (bitwise equal to the library's host synthesizer:
    tests/test_abi_cpu.py)."""
    base = o.cell_data_seed(MASTER_SEED, n, N, m, rank)
    t = TEMPLATE
    train = o.synthesize_uniform(n, TRAIN_FACTOR * m, t["phi"], t["rho"], t["var"], t["skew"], t["kurt"],
                                 o.derive_seed(base, [0]))
    obs = o.synthesize_uniform(n, N, t["phi"], t["rho"], t["var"], t["skew"], t["kurt"],
                               o.derive_seed(base, [1]))
    return train, obs


def run_reference(args, world, rank):
    """The reference CPU path (oracle restatement of mset.cpp:139-199 with the
    optimized backend's loop nests, backends.cpp:154-272, all host threads)
    over the full C2 workload per step.  Rank 0 only."""
    if rank != 0:
        return
    from oracle import oracle as o
    o.build()
    model_name, cores = cpu_info()
    train, obs = _oracle_data(o, N_SIG, N_OBS, N_MEM, 0)
    t0 = time.perf_counter()
    model = o.train(train, N_MEM, o.INVERSE_DISTANCE, 0.0, o.OPTIMIZED, 64, cores)
    train_ms = (time.perf_counter() - t0) * 1e3
    for _ in range(args.warmup):   # untimed warm-up on a slice (cache / thread start-up)
        o.estimate(model, obs[:4096], o.OPTIMIZED, 64, cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        o.estimate(model, obs, o.OPTIMIZED, 64, cores)
        times.append(time.perf_counter() - t0)
    step = statistics.mean(times)
    v = N_OBS / step
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": DATA, "config": config_dict(world),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"full C2 workload ({N_OBS} observations) per step; oracle optimized backend "
                                   f"(tile 64, {cores} threads) on {model_name}; warm-ups on 4096 observations"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "train": {"ms": train_ms, "api": "oracle train (optimized backend, tql2 eigensolver)"},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_c2(train, obs):
    """The oracle on the full C2 workload (~4 s of CPU work on 16 cores)."""
    from oracle import oracle as o
    o.build()
    model_name, cores = cpu_info()
    t1 = time.perf_counter()
    model = o.train(train, N_MEM, o.INVERSE_DISTANCE, 0.0, o.OPTIMIZED, 64, cores)
    train_s = time.perf_counter() - t1
    o.estimate(model, obs[:2048], o.OPTIMIZED, 64, cores)
    t0 = time.perf_counter()
    o.estimate(model, obs, o.OPTIMIZED, 64, cores)
    t = time.perf_counter() - t0
    return {"value": N_OBS / t, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"full C2 ({N_OBS} observations, one pass), oracle optimized backend "
                      f"(tile 64, {cores} threads) on {model_name}",
            "train_ms": train_s * 1e3}


def cpu_sample_estimate(D, scale, pinv, rank, obs, label):
    """Oracle surveillance of a bounded observation sample with a given model
    (timing does not depend on the model values)."""
    from oracle import oracle as o
    o.build()
    model_name, cores = cpu_info()
    import math
    m = o.Model(D=D, scale=scale, gram_pinv=pinv, rank=rank, h=math.sqrt(D.shape[0]), kind=o.INVERSE_DISTANCE,
                source_indices=None, eigen_spectrum=None)
    o.estimate(m, obs[:64], o.OPTIMIZED, 64, cores)
    t0 = time.perf_counter()
    o.estimate(m, obs, o.OPTIMIZED, 64, cores)
    t = time.perf_counter() - t0
    return {"value": obs.shape[0] / t, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{label}: {obs.shape[0]} observations, oracle optimized backend (tile 64, {cores} threads) "
                      f"on {model_name}, the B200-trained FP64 model"}


# BASELINE configs[3] / SURVEY 8(d) C4: 7 x 3 x 6 = 126 cells, 96 admissible,
# 5 replicates -> 480 (cell, replicate) units
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
                    "untimed warm-ups and the gather; timed train = certified-Cholesky train with "
                    "eigen_spectrum deferred to first export (the `train.ms` headline above is the "
                    "eager, reference-contract time)"}


def run_host_sweep(local):
    """GPU-vs-host speedup surface on the reduced grid (signals <=
    100, N <= 1e5): the b200 backend and the reference's `optimized` host
    backend (the CPU oracle, registered as the baseline leg) timed inside the
    same run_cell loop (sweep.cpp:206-227), then speedup() (surfaces.cpp:100-145)."""
    from oracle import host_backend
    from paper_2003_08011_b200 import BackendId
    from paper_2003_08011_b200.surfaces import export_speedup_csv, speedup
    from paper_2003_08011_b200.sweep import Phase, SignalStatsTemplate, SweepConfig, SweepGrid, run_sweep
    host_backend.register()
    _, cores = cpu_info()
    cpu, gpu = BackendId.optimized(cores, 64), BackendId("b200", local, "fp32")
    cfg = SweepConfig(SweepGrid([10, 20, 50], [10_000], [100, 200]), replicates=2, warmups=1,
                      backends=[cpu, gpu], master_seed=MASTER_SEED,
                      signal_template=SignalStatsTemplate(0.5, 0.3, 1.0, 0.5, 4.0))
    t0 = time.perf_counter()
    s = run_sweep(cfg, device=local)
    wall = time.perf_counter() - t0
    host_backend.unregister()
    sp = speedup(s, cpu, gpu)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    for ph in (Phase.train, Phase.surveil):
        export_speedup_csv(sp, ph, os.path.join(ROOT, "gpurun_out", f"speedup_{ph.value}.csv"))
    rows = [{"phase": c.phase.value, "n": c.coords.n_signals, "N": c.coords.n_observations,
             "m": c.coords.n_memory, "speedup": c.speedup, "hole": c.hole} for c in sp.cells]
    return {"grid": {"signal_counts": [10, 20, 50], "observation_counts": [10_000], "memory_counts": [100, 200],
                     "replicates": 2}, "reference_backend": cpu.label(), "optimized_backend": gpu.label(),
            "wall_s": wall, "cells": rows,
            "note": "speedup = median(host optimized) / median(b200), per phase (surfaces.cpp:100-145)"}


# ---------------------------------------------------------------------- B200
def _device_pass_timer(p, torch, model, obs, est, res, st, passes, flush=None):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(passes)]
    for a, b in ev:
        if flush is not None:
            flush.zero_()
        a.record(st)
        p.estimate_device(model, obs, est, res, st)
        b.record(st)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev]


def _e2e_timer(p, model, obs_np, local, reps):
    """cs_mset_estimate on pinned host FP64 buffers; returns seconds per call."""
    import numpy as np
    import torch
    from paper_2003_08011_b200 import _lib
    N, n = obs_np.shape
    h_obs = torch.from_numpy(np.ascontiguousarray(obs_np.T)).pin_memory()  # rows = signals
    h_est = torch.empty_like(h_obs).pin_memory()
    h_res = torch.empty_like(h_obs).pin_memory()
    o, e, r = h_obs.numpy().T, h_est.numpy().T, h_res.numpy().T  # N x n column-major views

    def call():
        _lib.check(_lib.lib().cs_mset_estimate(p.context(local).handle, model.handle, o.ctypes.data_as(_lib.pd),
                                               N, n, e.ctypes.data_as(_lib.pd), r.ctypes.data_as(_lib.pd)))
    call()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        call()
        ts.append(time.perf_counter() - t0)
    assert np.array_equal(r, o - e)  # residual identity on the e2e output
    return ts, e


def _train_times(p, fn, reps):
    tt = []
    model = fn()
    for _ in range(reps):
        t0 = time.perf_counter()
        fresh = fn()
        tt.append(time.perf_counter() - t0)
        model = fresh  # the previous model is freed outside the timed region
    return tt, model


def _train_flops(n, m):
    """FP64 train work: Gram 2m^2 n (GEMM form) + Cholesky m^3/3 +
    inverse L^-T L^-1 2m^3/3... counted as 4m^3/3 for the two triangular
    products + P = D_n G+ 2 n m^2."""
    return 2.0 * m * m * n + m ** 3 / 3.0 + 4.0 * m ** 3 / 3.0 + 2.0 * n * m * m


def run_large(local, n, N, m, workload, passes=5, e2e_obs=0, cpu_obs=0):
    """A large-n configuration on one GPU: train time through the device API
    and device-resident FP32 surveillance on the two-GEMM tcgen05 path; data
    from the device synthesiser (same recipe; host synthesis of 1e9+ samples
    is impractical).  Optional: e2e through cs_mset_estimate on the first
    `e2e_obs` observations (host FP64 buffers) and a CPU oracle sample."""
    import torch
    import paper_2003_08011_b200 as p
    dev = torch.device("cuda", local)
    t = TEMPLATE
    base = p.cell_data_seed(MASTER_SEED, n, N, m, 0)
    spec = lambda rows, seed: p.SignalSpec.uniform(n, rows, t["phi"], t["rho"], t["var"], t["skew"],  # noqa: E731
                                                   t["kurt"], seed)
    X = p.synthesize_device(spec(TRAIN_FACTOR * m, p.derive_seed(base, [0])), local)
    backend = p.BackendId("b200", local, "fp32")
    os.environ["CSB_EAGER_SPECTRUM"] = "1"
    tt_eager, model = _train_times(p, lambda: p.train_device(X, m, p.KernelConfig(), backend), 3)
    del os.environ["CSB_EAGER_SPECTRUM"]
    tt, model = _train_times(p, lambda: p.train_device(X, m, p.KernelConfig(), backend), 5)
    del X
    obs64 = p.synthesize_device(spec(N, p.derive_seed(base, [1])), local)
    obs = obs64.T.float().T          # N x n column-major FP32
    host_slice = obs64[:max(e2e_obs, cpu_obs)].cpu().numpy() if (e2e_obs or cpu_obs) else None
    del obs64
    torch.cuda.empty_cache()
    est = torch.empty_like(obs.T).T
    res = torch.empty_like(obs.T).T
    st = torch.cuda.current_stream(dev)
    p.estimate_device(model, obs, est, res, st)
    ms_list = _device_pass_timer(p, torch, model, obs, est, res, st, passes)
    ok = bool(torch.isfinite(est).all()) and bool(torch.allclose(res, obs - est))
    ms = statistics.median(ms_list)
    flops = 4.0 * n * m * N
    p_eff, p_burst = sustained_p_eff()
    tf = flops / (ms * 1e-3) / 1e12
    out = {"workload": workload, "n_signals": n, "n_observations": N, "n_memory": m,
           "obs_per_s": N / (ms * 1e-3), "ms_per_pass": ms, "passes": passes,
           "algorithmic_tflops": tf,
           "roofline": {"bound": "tensor", "achieved": tf, "peak": p_eff, "unit": "TFLOP/s",
                        "frac": tf / p_eff, "frac_vs_burst_peak": tf / p_burst,
                        "peak_note": SUSTAINED_NOTE},
           "kernels": "pack_obs + obs_sqnorm + gemm3x_f16_kernel<256,EpiSim> + gemm3x_f16_kernel<256,EpiOut> "
                      "per observation block",
           "train_ms": statistics.median(tt_eager) * 1e3, "train_ms_min": min(tt_eager) * 1e3,
           "train_ms_spectrum_deferred": statistics.median(tt) * 1e3,
           "train_api": "cs_mset_train_device (device FP64 training rows, synchronous); train_ms includes "
                        "the eigen spectrum (reference contract, mset.cpp:153-154)",
           "outputs_checked": ok}
    fp64 = load_probe_peaks().get("dmma_f64_tflops")
    if fp64:
        tf = _train_flops(n, m) / statistics.median(tt) / 1e12  # tt in seconds
        out["train_roofline"] = {"bound": "fp64 tensor (DMMA)", "achieved": tf, "peak": fp64, "unit": "TFLOP/s",
                                 "frac": tf / fp64, "flops": _train_flops(n, m),
                                 "note": "Gram 2m^2n + Cholesky m^3/3 + inverse 4m^3/3 + P 2nm^2 over the "
                                         "spectrum-deferred train time"}
    if e2e_obs:
        import numpy as np
        ts, _ = _e2e_timer(p, model, np.asfortranarray(host_slice[:e2e_obs]), local, 3)
        e = statistics.median(ts)
        out["e2e"] = {"value": e2e_obs / e, "unit": UNIT, "observations": e2e_obs,
                      "h2d_bytes_per_step": e2e_obs * n * 8, "d2h_bytes_per_step": 2 * e2e_obs * n * 8,
                      "api": "cs_mset_estimate (pinned host FP64 in, estimates + residuals out)"}
    if cpu_obs:
        import numpy as np
        ex = model.export()
        out["cpu_baseline"] = cpu_sample_estimate(ex["D"], ex["signal_scale"], ex["gram_pinv"], model.rank,
                                                  np.asfortranarray(host_slice[:cpu_obs]), workload.split(":")[0])
    del obs, est, res, model
    torch.cuda.empty_cache()
    return out


def run_c3(args, local):
    """BASELINE configs[2] (C3: n=1000, N=1M, m=4000, 16k training rows)."""
    return run_large(local, 1000, 1_000_000, 4000,
                     "C3: n=1000, N=1,000,000, m=4,000 (16k training rows), FP32 device-resident I/O",
                     e2e_obs=250_000, cpu_obs=0 if args.no_cpu_baseline else 1500)


C5_N, C5_n, C5_m, C5_CHUNK = 10_000_000, 4000, 8000, 1_250_000
if os.environ.get("CSB_BENCH_C5_SMALL"):  # development only (multi-rank plumbing on one GPU)
    C5_N, C5_n, C5_m, C5_CHUNK = 2_000_000, 1000, 2000, 250_000


def run_c5(args, world, rank, local, barrier, max_over_ranks):
    """BASELINE configs[4] made admissible (m >= 2n, so n = 4,000
    with m = 8,000), sharded as SURVEY 8(e) specifies: rank 0 trains ONCE,
    the packed device model is broadcast over NCCL (one buffer,
    paper_2003_08011_b200/shard.py), and the 10M observations are split into
    contiguous per-rank shards with no collective inside the surveillance
    loop.  The observation stream is a fixed grid of 8 chunks of 1.25M (each
    synthesized on the device from derive_seed(base, [1, chunk]), outside
    the timed region), so the data -- and, by construction, every output
    bit -- is the same at 1, 2, 4 or 8 GPUs: the line carries an exact
    digest of all estimates (sum of their FP32 words) to show it.  Strong
    scaling: total work fixed at 10M observations."""
    import torch
    import torch.distributed as dist
    import paper_2003_08011_b200 as p
    from paper_2003_08011_b200.shard import broadcast_model, shard_digest, shard_range, wrap64
    dev = torch.device("cuda", local)
    t = TEMPLATE
    n, m = C5_n, C5_m
    base = p.cell_data_seed(MASTER_SEED, n, C5_N, m, 0)
    spec = lambda rows, seed: p.SignalSpec.uniform(n, rows, t["phi"], t["rho"], t["var"], t["skew"],  # noqa: E731
                                                   t["kurt"], seed)
    backend = p.BackendId("b200", local, "fp32")
    out = {"workload": f"C5': n={n}, m={m} ({TRAIN_FACTOR * m // 1000}k training rows), N={C5_N // 1_000_000}M "
                       "observations sharded over the ranks, FP32 device-resident I/O",
           "n_signals": n, "n_memory": m, "n_observations": C5_N, "n_gpus": world, "scaling": "strong",
           "chunks": C5_N // C5_CHUNK}
    model = None
    if rank == 0:
        X = p.synthesize_device(spec(TRAIN_FACTOR * m, p.derive_seed(base, [0])), local)
        os.environ["CSB_EAGER_SPECTRUM"] = "1"
        tt_eager, _ = _train_times(p, lambda: p.train_device(X, m, p.KernelConfig(), backend), 2)
        del os.environ["CSB_EAGER_SPECTRUM"]
        tt, model = _train_times(p, lambda: p.train_device(X, m, p.KernelConfig(), backend), 3)
        del X
        torch.cuda.empty_cache()
        out.update(train_ms=statistics.median(tt_eager) * 1e3, train_ms_min=min(tt_eager) * 1e3,
                   train_ms_spectrum_deferred=statistics.median(tt) * 1e3,
                   train_api="cs_mset_train_device on rank 0 only (device FP64 training rows, synchronous); "
                             "train_ms includes the eigen spectrum (mset.cpp:153-154)")
        fp64 = load_probe_peaks().get("dmma_f64_tflops")
        if fp64:
            tf = _train_flops(n, m) / statistics.median(tt) / 1e12
            out["train_roofline"] = {"bound": "fp64 tensor (DMMA)", "achieved": tf, "peak": fp64,
                                     "unit": "TFLOP/s", "frac": tf / fp64, "flops": _train_flops(n, m),
                                     "note": "Gram 2m^2n + Cholesky m^3/3 + inverse 4m^3/3 + P 2nm^2 over the "
                                             "spectrum-deferred train time"}
    # ---- broadcast of the trained model (one packed device buffer)
    barrier()
    t0 = time.perf_counter()
    if world > 1:
        model, wire_bytes = broadcast_model(model, backend, src=0)
    else:
        wire_bytes = p.pack_model(model).numel()
    barrier()
    bcast_s = time.perf_counter() - t0
    # ---- this rank's chunks of the fixed 8-chunk observation grid
    c0, c1 = shard_range(C5_N // C5_CHUNK, world, rank, align=1)
    ms_total, digest = 0.0, 0
    st = torch.cuda.current_stream(dev)
    obs = est = res = None
    for c in range(c0, c1):
        obs = None
        torch.cuda.empty_cache()
        obs = p.synthesize_device(spec(C5_CHUNK, p.derive_seed(base, [1, c])), local, dtype=torch.float32)
        torch.cuda.empty_cache()
        if est is None:
            est, res = torch.empty_like(obs.T).T, torch.empty_like(obs.T).T
            p.estimate_device(model, obs, est, res, st)  # warm-up (lazy operand setup)
        ms = _device_pass_timer(p, torch, model, obs, est, res, st, 1)[0]
        ms_total += ms
        digest = wrap64(digest + shard_digest(est))
        if c == c0 and not bool(torch.allclose(res, obs - est)):
            raise RuntimeError("C5': residual identity failed")
    del obs, est, res
    torch.cuda.empty_cache()
    ms_max = max_over_ranks(ms_total)
    d = torch.tensor([digest], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(d)
    if rank != 0:
        del model
        return None
    flops = 4.0 * n * m * C5_N
    p_eff, p_burst = sustained_p_eff()
    out.update(obs_per_s=C5_N / (ms_max * 1e-3), ms_estimate_max_over_ranks=ms_max,
               broadcast_ms=bcast_s * 1e3, model_wire_bytes=wire_bytes,
               collective="%s broadcast of the packed model (torch.distributed, %d ranks)" % (
                   dist.get_backend().upper(), world) if world > 1 else "none (1 rank)",
               obs_per_s_incl_train_and_broadcast=C5_N / (out["train_ms_spectrum_deferred"] * 1e-3 + bcast_s
                                                          + ms_max * 1e-3),
               estimates_digest=wrap64(int(d.item())),
               digest_note="sum of the FP32 words of all 10M x 4000 estimates (int64, wrapping): equal at "
                           "every GPU count when the sharded outputs are bitwise equal",
               algorithmic_tflops=flops / (ms_max * 1e-3) / 1e12,
               roofline={"bound": "tensor", "achieved": flops / (ms_max * 1e-3) / 1e12, "peak": p_eff * world,
                         "unit": "TFLOP/s", "frac": flops / (ms_max * 1e-3) / 1e12 / (p_eff * world),
                         "frac_vs_burst_peak": flops / (ms_max * 1e-3) / 1e12 / (p_burst * world),
                         "peak_note": SUSTAINED_NOTE + " (per GPU x n_gpus)"},
               kernels="pack_obs + obs_sqnorm + gemm3x_f16_kernel<256,EpiSim> + gemm3x_f16_kernel<256,EpiOut> "
                       "per observation block")
    del model
    torch.cuda.empty_cache()
    return out


def run_c1(args, local, reps):
    """BASELINE configs[0] (C1: n=20, N=10k, m=100, 400 training rows): the
    MUFU / launch-latency-bound corner."""
    import numpy as np
    import torch
    import paper_2003_08011_b200 as p
    n, N, m = 20, 10_000, 100
    dev = torch.device("cuda", local)
    base = p.cell_data_seed(MASTER_SEED, n, N, m, 0)
    t = TEMPLATE
    mk = lambda rows, s: p.synthesize(p.SignalSpec.uniform(n, rows, t["phi"], t["rho"], t["var"], t["skew"],  # noqa
                                                           t["kurt"], p.derive_seed(base, [s]))).data
    train, obs = mk(TRAIN_FACTOR * m, 0), mk(N, 1)
    backend = p.BackendId("b200", local, "fp32")
    os.environ["CSB_EAGER_SPECTRUM"] = "1"
    tt, model = _train_times(p, lambda: p.train(train, m, p.KernelConfig(), backend), 5)
    del os.environ["CSB_EAGER_SPECTRUM"]
    d_obs = torch.tensor(obs.T.astype(np.float32), device=dev).T
    d_est, d_res = torch.empty_like(d_obs.T).T, torch.empty_like(d_obs.T).T
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream(dev)
    _device_pass_timer(p, torch, model, d_obs, d_est, d_res, st, 3, flush)
    ms = statistics.mean(_device_pass_timer(p, torch, model, d_obs, d_est, d_res, st, reps, flush))
    ts, _ = _e2e_timer(p, model, obs, local, max(3, min(reps, 20)))
    e = statistics.mean(ts)
    peaks = load_peaks()
    gbs = 12.0 * n * N / (ms * 1e-3) / 1e9
    out = {"workload": "C1: n=20, N=10,000, m=100 (400 training rows)", "obs_per_s": N / (ms * 1e-3),
           "ms_per_pass": ms, "train_ms": statistics.median(tt) * 1e3,
           "train_api": "cs_mset_train (host FP64 in), eigen spectrum inside train",
           "e2e": {"value": N / e, "unit": UNIT, "h2d_bytes_per_step": N * n * 8, "d2h_bytes_per_step": 2 * N * n * 8},
           "roofline": {"bound": "hbm", "achieved": gbs, "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                        "frac": gbs / peaks.get("hbm_gbs", 6650.0),
                        "note": "12n bytes/obs (FP32 x in, est + resid out); 79 128-observation tiles < 148 SMs, "
                                "so the launch is latency-bound, not HBM-bound"}}
    if not args.no_cpu_baseline:
        from oracle import oracle as o
        o.build()
        model_name, cores = cpu_info()
        ref = o.train(train, m, o.INVERSE_DISTANCE, 0.0, o.OPTIMIZED, 64, cores)
        o.estimate(ref, obs[:256], o.OPTIMIZED, 64, cores)
        t0 = time.perf_counter()
        reps_cpu = 5
        for _ in range(reps_cpu):
            o.estimate(ref, obs, o.OPTIMIZED, 64, cores)
        tc = (time.perf_counter() - t0) / reps_cpu
        out["cpu_baseline"] = {"value": N / tc, "unit": UNIT, "cores": cores, "kind": "port",
                               "sample": f"full C1, oracle optimized backend ({cores} threads) on {model_name}"}
    return out


def run_sprt_bench(local, n=1000, N=1_000_000, reps=5):
    """SPRT over device-resident FP32 residuals (N x n column-major; the C3
    surveillance output shape): cs_sprt_device = speculate pass (staged,
    coalesced, vectorised residual reads and flag stores) + fix-up pass (warp
    per signal) + the small state / count copies, CUDA events on the stream
    it runs on.  Bytes: FP32 residual in (4 B) + flag byte out (1 B) per
    (observation, signal), against the HBM peak."""
    import numpy as np
    import torch
    import paper_2003_08011_b200 as p
    dev = torch.device("cuda", local)
    g = torch.Generator(device=dev).manual_seed(7)
    resid = torch.randn((n, N), generator=g, device=dev, dtype=torch.float32).T
    det = p.SprtDetector(np.ones(n), backend=p.BackendId("b200", local, "fp32"))
    st = torch.cuda.current_stream(dev)
    det.update_device(resid, stream=st)
    torch.cuda.synchronize()
    ms, walls = [], []
    for _ in range(reps):
        det.state[:] = 0.0
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a.record(st)
        _, counts = det.update_device(resid, stream=st)
        b.record(st)
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - t0)
        ms.append(a.elapsed_time(b))
    t = statistics.median(ms) * 1e-3
    gbs = (4.0 + 1.0) * n * N / t / 1e9
    hbm = load_peaks().get("hbm_gbs", 6650.0)
    return {"n_signals": n, "n_observations": N, "ms": t * 1e3, "wall_ms": statistics.median(walls) * 1e3,
            "flags_per_s": n * N / t, "achieved_gbs": gbs, "peak_gbs": hbm, "frac": gbs / hbm,
            "alarms": int(counts.sum()),
            "kernels": "sprt_speculate_kernel<float,true> + sprt_fixup_kernel<float>",
            "note": "CUDA events around the cs_sprt_device call on its stream (kernels + state/count copies); "
                    "FP32 residuals in (4 B), byte flags out (1 B) per (observation, signal)"}


def run_b200(args, world, rank, local):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2003_08011_b200 as p

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        be = os.environ.get("CSB_BENCH_DIST_BACKEND", "nccl")
        dist.init_process_group(be, device_id=dev if be == "nccl" else None)
    backend = p.BackendId("b200", local, "fp32")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        tt = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    base = p.cell_data_seed(MASTER_SEED, N_SIG, N_OBS, N_MEM, rank)
    t = TEMPLATE
    mk = lambda rows, s: p.synthesize(p.SignalSpec.uniform(N_SIG, rows, t["phi"], t["rho"], t["var"], t["skew"],  # noqa
                                                           t["kurt"], p.derive_seed(base, [s]))).data
    train, obs = mk(TRAIN_FACTOR * N_MEM, 0), mk(N_OBS, 1)

    # ---- train (FP64), host API, synchronous.  Headline = the reference's
    # train contract (eigen_spectrum computed inside train, mset.cpp:153-154);
    # the spectrum-deferred time is reported beside it
    os.environ["CSB_EAGER_SPECTRUM"] = "1"
    eager, _ = _train_times(p, lambda: p.train(train, N_MEM, p.KernelConfig(), backend), 5)
    del os.environ["CSB_EAGER_SPECTRUM"]
    deferred, model = _train_times(p, lambda: p.train(train, N_MEM, p.KernelConfig(), backend), 5)

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
    barrier()
    e2e_t, _ = _e2e_timer(p, model, obs, local, max(3, min(args.steps, 20)))
    barrier()
    clocks = sampler.stop()
    e2e_mean = max_over_ranks(statistics.mean(e2e_t))

    # secondary sections: a failure is recorded in the line instead of losing
    # the headline (the traceback goes to stderr)
    def section(name, fn):
        try:
            return fn()
        except Exception as exc:  # noqa: BLE001
            import traceback
            traceback.print_exc(file=sys.stderr)
            return {"error": f"{name}: {type(exc).__name__}: {exc}"}

    # ---- C5' (configs[4]): train once, broadcast, observation shards
    c5 = None if args.no_c5 else section("c5", lambda: run_c5(args, world, rank, local, barrier, max_over_ranks))

    # ---- Monte Carlo scoping sweep (cells/s), strong scaling over ranks
    sweep = None if args.no_sweep else section(
        "sweep", lambda: run_bench_sweep(world, rank, local, barrier, max_over_ranks))

    if rank != 0:
        return
    peaks = load_peaks()
    flops_per_obs = 4.0 * N_SIG * N_MEM                       # F = 4nm
    achieved_tflops = flops_per_obs * N_OBS / (mean_ms * 1e-3) / 1e12
    bf16 = peaks.get("bf16_tflops", 1590.0)
    p_eff = bf16 / 3.0
    K1, N2 = (N_SIG + 2 + 15) // 16 * 16, (N_SIG + 7) // 8 * 8  # + ||d||^2, ||x||^2 columns; GEMM2 N steps by 8
    MT = 64
    m_pad = (N_MEM + MT - 1) // MT * MT
    n_tiles = (N_OBS + 127) // 128
    issued = 3 * 2 * 128 * n_tiles * m_pad * (K1 + N2)
    issued_tflops = issued / (mean_ms * 1e-3) / 1e12
    value = world * N_OBS / (mean_ms_max * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean_ms_max,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": DATA, "config": config_dict(world),
        "wall_s_timed_region": wall,
        "gpu_launches": args.steps,
        "kernels_per_step": {"mset_estimate_tc_kernel<64,2,2,float,true>": 1},
        "train": {"ms": statistics.median(eager) * 1e3, "ms_min": min(eager) * 1e3,
                  "ms_spectrum_deferred": statistics.median(deferred) * 1e3,
                  "api": "cs_mset_train (host FP64 in, synchronous)",
                  "includes": "H2D + selection + scale + Gram + certified-Cholesky pseudo-inverse (rank == m "
                              "proven by the 1-norm condition bound; eigen route otherwise) + eigen_spectrum "
                              "(eigenvalues-only) + P = Dn G+ + operand packing"},
        "e2e": {"value": world * N_OBS / e2e_mean, "unit": UNIT,
                "h2d_bytes_per_step": N_OBS * N_SIG * 8,
                "d2h_bytes_per_step": 2 * N_OBS * N_SIG * 8,
                "api": "cs_mset_estimate (pinned host FP64 in, estimates + residuals out)"},
        "roofline": {"bound": "tensor", "achieved": achieved_tflops, "peak": p_eff, "unit": "TFLOP/s",
                     "frac": achieved_tflops / p_eff, "traffic": load_traffic("mset_estimate_tc_kernel_C2"),
                     "kernel": "mset_estimate_tc_kernel<64,2,2,float,true>",
                     "algorithmic_flops_per_launch": flops_per_obs * N_OBS,
                     "peak_note": "P_eff (SURVEY 8d) = measured dense bf16 (MEASURED_PEAKS.json, "
                                  f"{bf16} TFLOP/s; kind::f16 runs at the same dense rate) / 3: the kernel "
                                  "issues 3 FP16 split products per GEMM (FP32-accurate 3xFP16)",
                     "issued_f16_tflops": issued_tflops,
                     "tensor_pipe_frac_issued": issued_tflops / bf16},
        "clocks": clocks,
    }
    if sweep is not None:
        line["sweep"] = sweep
    if c5 is not None:
        line["c5"] = c5
    if world == 1:
        if not args.no_c1:
            line["c1"] = section("c1", lambda: run_c1(args, local, args.steps))
        if not args.no_c3:
            line["c3"] = section("c3", lambda: run_c3(args, local))
        if not args.no_sprt:
            line["sprt"] = section("sprt", lambda: run_sprt_bench(local))
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = section("cpu_baseline", lambda: cpu_baseline_c2(train, obs))
            if not args.no_sweep:
                line["host_sweep"] = section("host_sweep", lambda: run_host_sweep(local))
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-c1", action="store_true")
    ap.add_argument("--no-c3", action="store_true")
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--no-sprt", action="store_true")
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
