"""One sweep unit's device work at a given shape (development tool, for ncu
launch lists): synthesize the training rows (4m x n) and the surveillance
block (N x n) on the device, then train an FP32 model.
Usage: python tools/feed_train.py [n m N]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402,F401

import paper_2003_08011_b200 as p  # noqa: E402

n, m, N = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (1000, 4000, 1000000)
for rep in range(2):
    X = p.synthesize_device(p.SignalSpec.uniform(n, 4 * m, 0.5, 0.3, 1.0, 0.5, 4.0, 11 + rep))
    O = p.synthesize_device(p.SignalSpec.uniform(n, N, 0.5, 0.3, 1.0, 0.5, 4.0, 12 + rep))
    g = p.train_device(X, m, p.KernelConfig(), p.BackendId("b200", 0, "fp32"))
    print(f"rep {rep}: n={n} m={m} N={N} rank={g.rank}")
    del X, O, g
