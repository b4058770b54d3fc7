"""Per-phase train timings (CSB_TRACE=1) for the BASELINE configs (C1-C3)."""
import os, sys, time
os.environ.setdefault("CSB_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: F401,E402
import paper_2003_08011_b200 as p  # noqa: E402

p.symmetric_eig([[1.0, 0.0], [0.0, 1.0]])
for n, m in [(20, 100), (100, 1000), (1000, 4000)] if len(sys.argv) < 2 else [tuple(map(int, a.split(","))) for a in sys.argv[1:]]:
    X = p.synthesize_device(p.SignalSpec.uniform(n, 4 * m, 0.5, 0.3, 1.0, 0.5, 4.0, 7))
    for prec in ("fp64", "fp32", "fp32", "fp32", "fp32"):
        print(f"--- n={n} m={m} {prec}", file=sys.stderr, flush=True)
        t = time.perf_counter()
        g = p.train_device(X, m, p.KernelConfig(), p.BackendId("b200", 0, prec))
        print(f"n={n} m={m} {prec} train {1e3*(time.perf_counter()-t):.1f} ms rank={g.rank}", flush=True)
