"""Where the C4 sweep's wall time goes (development tool): wraps the unit
phases (device synthesis, timed train+estimate, FP32 conversion) with device
synchronisation and sums their wall times per (n, N, m) class.
Usage: python tools/sweep_profile.py"""
import collections
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2003_08011_b200 import BackendId  # noqa: E402
from paper_2003_08011_b200 import sweep as sw  # noqa: E402

acc = collections.defaultdict(float)


def wrap(name, fn):
    def inner(*a, **k):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        acc[name] += time.perf_counter() - t
        return r
    return inner


sw._cell_data = wrap("synthesis", sw._cell_data)
sw._train_eval = wrap("train+estimate (incl. FP32 copy, output alloc)", sw._train_eval)
import paper_2003_08011_b200.mset as mset  # noqa: E402
mset.train_device = wrap("  train_device", mset.train_device)
mset.estimate_device = wrap("  estimate_device", mset.estimate_device)
cfg = sw.SweepConfig(sw.SweepGrid(**bench.SWEEP_GRID), replicates=bench.SWEEP_REPLICATES, warmups=1,
                     backends=[BackendId("b200", 0, "fp32")], master_seed=bench.MASTER_SEED,
                     signal_template=sw.SignalStatsTemplate(0.5, 0.3, 1.0, 0.5, 4.0))
sw.run_sweep(cfg, device=0)  # warm
acc.clear()
t0 = time.perf_counter()
sw.run_sweep(cfg, device=0)
wall = time.perf_counter() - t0
print(f"wall {wall:.2f} s")
for k, v in acc.items():
    print(f"  {k:50s} {v:7.2f} s")
