"""e2e (host FP64 API) throughput vs pipeline chunk size at C2.  Dev tool."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch  # noqa: E401
import paper_2003_08011_b200 as p
from paper_2003_08011_b200 import _lib
n, m, N = 100, 1000, 100_000
X = p.synthesize(p.SignalSpec.uniform(n, 4 * m, 0.5, 0.3, 1.0, 0.5, 4.0, 1)).data
obs = p.synthesize(p.SignalSpec.uniform(n, N, 0.5, 0.3, 1.0, 0.5, 4.0, 2)).data
g = p.train(X, m, p.KernelConfig(), p.BackendId("b200", 0, "fp32"))
h_obs = torch.from_numpy(np.asfortranarray(obs).T.copy()).pin_memory()
h_est = torch.empty_like(h_obs).pin_memory()
h_res = torch.empty_like(h_obs).pin_memory()
o, e, r = h_obs.numpy().T, h_est.numpy().T, h_res.numpy().T
for cd in [1 << 17, 1 << 18, 3 << 17, 1 << 19, 3 << 18, 1 << 20, 1 << 21]:
    os.environ["CSB_E2E_CHUNK_DOUBLES"] = str(cd)
    f = lambda: _lib.check(_lib.lib().cs_mset_estimate(p.context(0).handle, g.handle, o.ctypes.data_as(_lib.pd), N, n,  # noqa
                                                        e.ctypes.data_as(_lib.pd), r.ctypes.data_as(_lib.pd)))
    f(); f()
    ts = []
    for _ in range(10):
        t = time.perf_counter(); f(); ts.append(time.perf_counter() - t)
    print(f"chunk {cd} doubles ({cd // n} obs): {N / statistics.mean(ts):.3e} obs/s  {statistics.mean(ts)*1e3:.2f} ms")
