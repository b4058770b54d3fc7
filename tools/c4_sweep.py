"""Full C4 Monte Carlo scoping sweep (7 x 3 x 6 grid, 96
admissible cells) on one GPU; prints wall time and units/s.  Dev tool."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa
from paper_2003_08011_b200 import BackendId
from paper_2003_08011_b200.sweep import SweepConfig, SweepGrid, SignalStatsTemplate, run_sweep
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
grid = SweepGrid(signal_counts=[10, 20, 50, 100, 200, 500, 1000], observation_counts=[10_000, 100_000, 1_000_000],
                 memory_counts=[100, 200, 500, 1000, 2000, 4000])
cfg = SweepConfig(grid, replicates=reps, warmups=1, backends=[BackendId("b200", 0, "fp32")], master_seed=20260810,
                  signal_template=SignalStatsTemplate(0.5, 0.3, 1.0, 0.5, 4.0))
t = time.perf_counter()
s = run_sweep(cfg, world=1, rank=0, device=0)
wall = time.perf_counter() - t
tr = [c for c in s.cells if c.phase.value == "train"]
units = sum(len(c.samples) for c in tr)
print(json.dumps({"wall_s": wall, "units": units, "units_per_s": units / wall,
                  "admissible": sum(not c.excluded for c in tr), "excluded": sum(c.excluded for c in tr),
                  "train_s": sum(sum(c.samples) for c in tr),
                  "surveil_s": sum(sum(c.samples) for c in s.cells if c.phase.value == "surveil")}))
