"""Eigenvalues-only timing at a few sizes (development tool; own path vs
cuSOLVER is selected by CSB_EIG_OWN).  Usage: python tools/eig_time.py [m ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2003_08011_b200 as p  # noqa: E402

p.context(0)
for m in [int(a) for a in sys.argv[1:]] or [100]:
    rng = np.random.default_rng(1)
    A = rng.standard_normal((m, m))
    A = np.asfortranarray(A @ A.T)
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        p.symmetric_eigvals(A)
        ts.append(time.perf_counter() - t)
    print(m, os.environ.get("CSB_EIG_OWN", "default"), "%.3f ms" % (1e3 * sorted(ts)[2]))
