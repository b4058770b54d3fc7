"""Times the fused tcgen05 surveillance kernel over several (n, m) shapes.

Device-resident FP32 I/O, CUDA events on the launching stream, L2 flushed
between launches.  Prints one JSON object per shape.  Development tool (not
the bench contract; see bench.py).
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_08011_b200 as p  # noqa: E402

SHAPES = [(20, 100, 200_000), (64, 512, 200_000), (100, 1000, 100_000), (128, 1024, 100_000),
          (32, 2048, 100_000), (100, 4000, 50_000)]


def main():
    shapes = SHAPES
    if len(sys.argv) > 1:
        shapes = [tuple(int(x) for x in s.split(",")) for s in sys.argv[1:]]
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for n, m, N in shapes:
        X = p.synthesize(p.SignalSpec.uniform(n, 4 * m, 0.5, 0.3, 1.0, 0.5, 4.0, 1)).data
        obs = p.synthesize(p.SignalSpec.uniform(n, N, 0.5, 0.3, 1.0, 0.5, 4.0, 2)).data
        g = p.train(X, m, p.KernelConfig(), p.BackendId("b200", 0, "fp32"))
        d_obs = torch.tensor(obs.T.astype(np.float32), device=dev).T
        d_est = torch.empty_like(d_obs.T).T
        d_res = torch.empty_like(d_obs.T).T
        st = torch.cuda.current_stream(dev)
        for _ in range(3):
            p.estimate_device(g, d_obs, d_est, d_res, st)
        times = []
        for _ in range(10):
            mode = os.environ.get("FLUSH", "write")
            if mode == "write":
                flush.zero_()
            elif mode == "read":
                flush.sum(dtype=torch.int32)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(st)
            p.estimate_device(g, d_obs, d_est, d_res, st)
            b.record(st)
            b.synchronize()
            times.append(a.elapsed_time(b))
        ms = statistics.median(times)
        tf = 4.0 * n * m * N / (ms * 1e-3) / 1e12
        print(json.dumps({"n": n, "m": m, "N": N, "ms": ms, "obs_per_s": N / (ms * 1e-3),
                          "algorithmic_tflops": tf}), flush=True)


if __name__ == "__main__":
    main()
