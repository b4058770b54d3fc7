"""Times large-n surveillance (two-GEMM path) at BASELINE config 3's model
shape.  Development tool.  Usage: python tools/c3_time.py [n m N]"""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_08011_b200 as p  # noqa: E402

n, m, N = (int(a) for a in sys.argv[1:4]) if len(sys.argv) >= 4 else (1000, 4000, 200_000)
dev = torch.device("cuda", 0)
X = p.synthesize(p.SignalSpec.uniform(n, 4 * m, 0.5, 0.3, 1.0, 0.5, 4.0, 1)).data
t = time.perf_counter()
g = p.train(X, m, p.KernelConfig(), p.BackendId("b200", 0, "fp32"))
print(f"train {1e3 * (time.perf_counter() - t):.1f} ms")
t = time.perf_counter()
g = p.train(X, m, p.KernelConfig(), p.BackendId("b200", 0, "fp32"))
print(f"train (warm) {1e3 * (time.perf_counter() - t):.1f} ms")
obs = torch.randn(n, N, device=dev, dtype=torch.float32).T
est = torch.empty_like(obs.T).T
res = torch.empty_like(obs.T).T
st = torch.cuda.current_stream()
for _ in range(2):
    p.estimate_device(g, obs, est, res, st)
ts = []
for _ in range(5):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    p.estimate_device(g, obs, est, res, st)
    b.record(st)
    b.synchronize()
    ts.append(a.elapsed_time(b))
ms = statistics.median(ts)
fl = 4.0 * n * m * N
print(f"n={n} m={m} N={N}: {ms:.2f} ms  {N / ms * 1e3:.3e} obs/s  {fl / ms / 1e9:.1f} TFLOP/s algorithmic "
      f"({fl * 3 / ms / 1e9:.1f} issued tf32)")
