"""The bench's C2 step loop under a profiler range (development tool): train
the C2 model and warm up outside the range, then 5 steps (L2 flush + one
surveillance pass each) inside cudaProfilerStart/Stop, so that
`ncu --profile-from-start off` lists exactly the launches of the timed steps.
Usage: ncu --profile-from-start off --metrics gpu__time_duration.sum ... python tools/c2_steps.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_08011_b200 as p  # noqa: E402

n, N, m = 100, 100_000, 1000
base = p.cell_data_seed(20260810, n, N, m, 0)
mk = lambda rows, s: p.synthesize(p.SignalSpec.uniform(n, rows, 0.5, 0.3, 1.0, 0.5, 4.0,  # noqa: E731
                                                       p.derive_seed(base, [s]))).data
model = p.train(mk(4 * m, 0), m, p.KernelConfig(), p.BackendId("b200", 0, "fp32"))
dev = torch.device("cuda", 0)
obs = torch.tensor(mk(N, 1).T.astype(np.float32), device=dev).T
est, res = torch.empty_like(obs.T).T, torch.empty_like(obs.T).T
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream(dev)
for _ in range(3):
    p.estimate_device(model, obs, est, res, st)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(5):
    flush.zero_()
    p.estimate_device(model, obs, est, res, st)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
